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
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include "es_device.cuh"
#include "es_internal.h"
#include "es_spmm.h"

namespace es {
namespace {

constexpr unsigned kAll = 0xffffffffu;

// 16-B global -> shared copy, zero-filling when src_bytes == 0 (no global read is made): the
// ring is refilled branch-free, slots past the row's end land as zeros.
// (.cg: L2 only -- the .ca form, L1-allocating, measured slower: profiles/r01.md)
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
// the same with an L2 eviction-policy hint (A/B: evict_last on the slab gathers)
__device__ __forceinline__ void cp_async16_zfill_hint(uint32_t dst, const void* src, uint32_t src_bytes,
                                                      uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;"
                 :: "r"(dst), "l"(src), "r"(src_bytes), "l"(pol) : "memory");
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

// ---- device backstops of the workspace contract (include/es_spmm.h: reuse_sampled, nnz)
// A row whose slots would end past the workspace capacity, or a call whose expected sampling
// signature differs from the one the sampling call left in the header, is written as NaN (a
// loud failure, never a truncated sum) and the reason is ORed into the header's status word.
__device__ __forceinline__ bool slab_row_guard(const SlabParams& p, int64_t raw_end, bool sig_bad) {
    const bool over = raw_end > p.cap;
    if ((over || sig_bad) && p.ws_status && (threadIdx.x & 31) == 0)
        atomicOr(p.ws_status, (over ? kWsOverflow : 0) | (sig_bad ? kWsSignature : 0));
    return over || sig_bad;
}

__device__ __forceinline__ void slab_poison_row(const SlabParams& p, int64_t r) {
    const float nan = __int_as_float(0x7fc00000);
    for (int c = threadIdx.x & 31; c < p.w; c += 32) {
        if (p.c_mc) st_multicast(p.c_mc + (p.row_base + r) * p.ldc + p.col0 + c, nan);
        else if (p.n_peers == 0) p.C[r * p.ldc + c] = nan;
        else
            for (int q = 0; q < p.n_peers; ++q) p.c_peers[q][(p.row_base + r) * p.ldc + p.col0 + c] = nan;
    }
}

// Epilogue of one lane's piece: E consecutive elements starting at slice column `col`
// (a5: SUM, or MEAN / divisor with IEEE division, k = 0 -> 0), 16-B stores where C allows.
template <int E>
__device__ __forceinline__ void slab_store_piece(const SlabParams& p, int64_t r, int col, const float* tot,
                                                 int64_t div, uint64_t pol) {
#pragma unroll
    for (int h4 = 0; h4 < E / 4; ++h4) {
        const int c0 = col + 4 * h4;
        const int rem = p.w - c0;
        if (rem <= 0) break;
        float res[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float t = tot[4 * h4 + c];
            res[c] = p.reduce == kMean ? (div > 0 ? __fdiv_rn(t, (float)div) : 0.0f) : t;
        }
        auto put = [&](float* dst) {
            if (p.c_vec && rem >= 4) st_stream4(dst, res, pol);
            else
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < rem) st_stream(dst + c, res[c], pol);
        };
        if (p.c_mc) {                                // fused all-gather through NVLS multicast
            float* dst = p.c_mc + (p.row_base + r) * p.ldc + p.col0 + c0;
            if (p.c_vec && rem >= 4) st_multicast4(dst, res);
            else
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < rem) st_multicast(dst + c, res[c]);
        } else if (p.n_peers == 0) {
            put(p.C + r * p.ldc + c0);
        } else {                                     // fused all-gather: every rank's C (NEXT-1)
            const int64_t off = (p.row_base + r) * p.ldc + p.col0 + c0;
            for (int q = 0; q < p.n_peers; ++q) put(p.c_peers[q] + off);
        }
    }
}

// Stores of 4 results to peer ranks' C or through NVLS multicast (the fused all-gather): out of
// line, so the flow kernel's row epilogue stays small in the instruction stream.
__device__ __noinline__ void slab_store_remote(const SlabParams& p, int64_t r, int c0, int rem, float r0, float r1,
                                               float r2, float r3) {
    const float res[4] = {r0, r1, r2, r3};
    const int64_t off = (p.row_base + r) * p.ldc + p.col0 + c0;
    const uint64_t pol = policy_evict_first();
    if (p.c_mc) {
        if (p.c_vec && rem >= 4) st_multicast4(p.c_mc + off, res);
        else
            for (int c = 0; c < 4 && c < rem; ++c) st_multicast(p.c_mc + off + c, res[c]);
        return;
    }
    for (int q = 0; q < p.n_peers; ++q) {
        if (p.c_vec && rem >= 4) st_stream4(p.c_peers[q] + off, res, pol);
        else
            for (int c = 0; c < 4 && c < rem; ++c) st_stream(p.c_peers[q] + off + c, res[c], pol);
    }
}

// slab_store_piece with the MEAN divisor already converted to float (flow kernel; (float)k_i or
// (float)d_i -- the same value the int64 form converts)
template <int E>
__device__ __forceinline__ void slab_store_piece_f(const SlabParams& p, int64_t r, int col, const float* tot,
                                                   float div, uint64_t pol) {
#pragma unroll
    for (int h4 = 0; h4 < E / 4; ++h4) {
        const int c0 = col + 4 * h4;
        const int rem = p.w - c0;
        if (rem <= 0) break;
        float res[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float t = tot[4 * h4 + c];
            res[c] = p.reduce == kMean ? (div > 0.0f ? __fdiv_rn(t, div) : 0.0f) : t;
        }
        if (p.c_mc || p.n_peers > 0) {
            slab_store_remote(p, r, c0, rem, res[0], res[1], res[2], res[3]);
        } else {
            float* dst = p.C + r * p.ldc + c0;
            if (p.c_vec && rem >= 4) st_stream4(dst, res, pol);
            else
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c < rem) st_stream(dst + c, res[c], pol);
        }
    }
}

// Slots [beg, end) of local row r (k_i of them), the guards applied.  Returns false when the
// warp has nothing to compute (guard tripped: the row was poisoned).
__device__ __forceinline__ bool slab_row_slots(const SlabParams& p, int64_t r, int64_t& beg, int32_t& k) {
    const uint64_t pol = policy_evict_first();
    beg = ld_stream(p.s_rowptr + r, pol) - p.slot_base;
    int64_t end = ld_stream(p.s_rowptr + r + 1, pol) - p.slot_base;
    if (p.direct_s > 0 && end - beg > p.direct_s) end = beg + p.direct_s;   // Bucket: first s of the row
    bool sig_bad = p.ws_sig != nullptr && *p.ws_sig != p.sig;
    if (p.reuse_s > 0 && !sig_bad && end <= p.cap) {              // reused slots: the caller's graph?
        const int64_t d = ld_stream(p.rowptr + r + 1, pol) - ld_stream(p.rowptr + r, pol);
        sig_bad = end - beg != (d < p.reuse_s ? d : (int64_t)p.reuse_s);
    }
    if (slab_row_guard(p, end, sig_bad)) {
        slab_poison_row(p, r);
        return false;
    }
    k = end > beg ? (int32_t)(end - beg) : 0;
    return true;
}

// ---------------------------------------------------------------- register-direct slab kernel
// The default slab kernel.  One warp per row, split into S = 32/G groups of G
// lanes; step u of a 32-slot chunk consumes slots S*u + e (group e = lane / G).  Lane `sub` of
// a group owns the P 32-byte pieces sub + G*q of the 256-byte slab row and gathers each with
// ONE 256-bit load (SASS LDG.E...256) straight into registers: no shared memory, so every B
// byte crosses the L1 data path once (the shared-memory ring wrote it with LDGSTS and read it
// back with LDS: two crossings, the measured limiter of that kernel).  The loads of step u + D
// are issued right after step u is consumed into the D-deep register ring it released; slots
// past k_i (and pieces past the slice) are zero-filled, so they add exactly +0.
// Per element: group e sums slots j = e (mod S) in slot order with 32-slot-chunk partials,
// then an xor tree over the groups -- the order of the shared-memory ring with the same G
// (bitwise; tested), inside the DESIGN.md §6 bound.
template <bool BF16> struct Piece32;
template <> struct Piece32<false> {              // 8 fp32
    static constexpr int kElems = 8;
    __device__ __forceinline__ static void widen(const uint32_t* w, float* out) {
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = __uint_as_float(w[i]);
    }
};
template <> struct Piece32<true> {               // 16 bf16, widened exactly to fp32 (NEXT-4)
    static constexpr int kElems = 16;
    __device__ __forceinline__ static void widen(const uint32_t* w, float* out) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            out[2 * i] = __uint_as_float(w[i] << 16);
            out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
};

// 256-bit gather of one 32-B piece when `on` (CACHE 0: L1::no_allocate; 1: L1-allocating, so hot
// B rows can hit in L1 across the warps of an SM).  The predicate lives inside the asm and the
// registers are in/out operands: a predicated-off load leaves them as they were, so the ring's
// registers are the load's destination (no moves).
template <int CACHE>
__device__ __forceinline__ void ld256(const void* src, uint32_t* w, bool on) {
    if constexpr (CACHE == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
                     "@p ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
                     : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
                       "+r"(w[7])
                     : "l"(src), "r"((int)on));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
                     "@p ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
                     : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3]), "+r"(w[4]), "+r"(w[5]), "+r"(w[6]),
                       "+r"(w[7])
                     : "l"(src), "r"((int)on));
}

template <int G, int P, int D, int W, int MINW, bool BF16, bool FULL, int CACHE>
__global__ void __launch_bounds__(32 * W, MINW / W)
spmm_slab_ldg(const SlabParams p) {
    constexpr int E = Piece32<BF16>::kElems;
    constexpr int S = 32 / G;            // slots per step
    constexpr int U = G;                 // steps per 32-slot chunk
    static_assert((G == 2 || G == 4 || G == 8) && G * P <= 8, "lanes x pieces per slot (8 pieces = 256 B)");
    static_assert(D >= 2 && U % D == 0, "ring depth must divide the steps of a chunk");
    const int lane = threadIdx.x & 31;
    const int e = lane / G, sub = lane % G;
    const int64_t r = (int64_t)blockIdx.x * W + (threadIdx.x >> 5);
    if (r >= p.n_rows) return;
    int64_t beg;
    int32_t k;
    if (!slab_row_slots(p, r, beg, k)) return;
    const char* bl = reinterpret_cast<const char*>(p.B) + sub * 32;
    const uint32_t row_bytes = (uint32_t)(p.ldb * (BF16 ? 2 : 4));

    // Slots past k_i are neither loaded nor accumulated (predicated loads and FMAs: no zero
    // fill, so no register moves); pieces past a narrow slice are not loaded and their
    // accumulators are never stored (the xor tree only combines equal pieces).
    uint32_t buf[D][P][8];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) buf[d][q][i] = 0u;
    auto issue = [&](int d, int32_t col, bool valid) {
        const char* src = bl + (uint64_t)(uint32_t)col * row_bytes;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const bool on = FULL ? valid : (valid && sub + G * q < p.nv);
            ld256<CACHE>(src + q * G * 32, buf[d][q], on);
        }
    };
    auto load_pair = [&](int64_t j, int32_t& c, float& a) {      // slot j of the row (coalesced)
        const uint64_t pol = policy_evict_first();
        c = ld_stream(p.s_colind + beg + j, pol);
        a = p.s_val ? ld_stream(p.s_val + beg + j, pol) : 1.0f;
    };

    int32_t c0 = 0, c1 = 0;
    float a0 = 0.0f, a1 = 0.0f;
    if (lane < k) load_pair(lane, c0, a0);
    if (32 + lane < k) load_pair(32 + lane, c1, a1);
#pragma unroll
    for (int t = 0; t < D; ++t) issue(t, __shfl_sync(kAll, c0, S * t + e), S * t + e < k);
    float part[P][E], tot[P][E];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < E; ++c) { part[q][c] = 0.0f; tot[q][c] = 0.0f; }
    // one 32-slot chunk: full chunks (all slots valid, warp-uniform test) run branch-free; only a
    // row's last, partial chunk predicates its FMAs on the slot being < k
    auto chunk = [&](int32_t j0, auto partial) {
#pragma unroll 1
        for (int u0 = 0; u0 < U; u0 += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {                        // step u = u0 + d, ring slot d
                const int u = u0 + d;
                const float av = __shfl_sync(kAll, a0, S * u + e);
                if (!decltype(partial)::value || j0 + S * u + e < k) {
#pragma unroll
                    for (int q = 0; q < P; ++q) {
                        float x[E];
                        Piece32<BF16>::widen(buf[d][q], x);
#pragma unroll
                        for (int c = 0; c < E; ++c) part[q][c] = fmaf(av, x[c], part[q][c]);
                    }
                }
                const int tn = u + D;                            // refill: step u + D
                const int32_t cn = __shfl_sync(kAll, tn < U ? c0 : c1, (S * tn + e) & 31);
                issue(d, cn, j0 + S * tn + e < k);
            }
        }
    };
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
        if (j0 + 32 <= k) chunk(j0, std::false_type{});
        else chunk(j0, std::true_type{});
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
    const uint64_t pol_a = policy_evict_first();
    int64_t div = k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
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
            if (FULL || piece < p.nv) slab_store_piece<E>(p, r, piece * E, tot[q], div, pol_a);
        }
    }
}

// ---------------------------------------------------------------- shared-memory ring slab kernel
// The round-1 kernel, kept for B rows that are 16-B but not 32-B aligned and for A/B
// measurement (ES_KERNEL_SLAB_SMEM).  Same mapping with 16-B pieces staged through a per-warp
// cp.async ring: lane `sub` owns the P pieces sub + G*q (nv <= G*P <= 16), each LDGSTS
// instruction of a group covers G*16 contiguous bytes.  Ring layout [warps][D][P][S][G]: the
// 8 lanes of a quarter-warp always touch 128 contiguous bytes (conflict-free for every G).
// Per element: group e sums slots j = e (mod S) in slot order (32-slot-chunk partials), then
// an xor tree over the groups (G = 16: spmm_cpasync_hw's order, bitwise).
// LA2: the (col, val) chunk window looks two 32-slot chunks ahead instead of one (the chunk
// loads queue behind the ring's copies in the L1 miss path; one chunk of lead time was the top
// stall of the kernel, profiles/r02.md).
template <int G, int P, int D, int MINB, bool FULL, int W, bool BF16 = false, bool LA2 = false>
__global__ void __launch_bounds__(32 * W, MINB * 8 / W)
spmm_slab(const SlabParams p) {
    constexpr int E = SlabPiece<BF16>::kElems;   // B elements (-> fp32 accumulators) per piece
    constexpr int S = 32 / G;            // slots per step
    constexpr int U = 32 / S;            // steps per 32-slot chunk (= G)
    static_assert((G == 2 || G == 4 || G == 8 || G == 16) && G * P <= 16, "lanes x pieces per slot");
    static_assert(D >= 2 && U % D == 0, "ring depth must divide the steps of a chunk");
    constexpr int kStage = 32 * P;                               // float4 per warp stage
    extern __shared__ __align__(16) float4 slab_ring[];          // [warps][D][P][S][G]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int e = lane / G, sub = lane % G;
    const int64_t r = (int64_t)blockIdx.x * W + warp;
    if (r >= p.n_rows) return;
    int64_t beg;
    int32_t k;
    if (!slab_row_slots(p, r, beg, k)) return;
    const uint32_t my_s = smem_u32(slab_ring + (size_t)warp * D * kStage + e * G + sub);
    const char* bl = reinterpret_cast<const char*>(p.B) + sub * 16;
    const uint32_t row_bytes = (uint32_t)(p.ldb * (BF16 ? 2 : 4));

    // FULL: all 16 pieces of the slice exist (every slice but a narrower last one)
    auto copy = [&](int stage, int32_t col, bool valid) {
        const char* src = bl + (uint64_t)(uint32_t)col * row_bytes;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const bool on = FULL ? valid : (valid && sub + G * q < p.nv);
            cp_async16_zfill(my_s + (stage * kStage + q * 32) * 16, src + q * G * 16, on ? 16u : 0u);
        }
    };
    auto load_pair = [&](int64_t j, int32_t& c, float& a) {      // slot j of the row (coalesced)
        const uint64_t pol = policy_evict_first();
        c = ld_stream(p.s_colind + beg + j, pol);
        a = p.s_val ? ld_stream(p.s_val + beg + j, pol) : 1.0f;
    };

    // (col, val) of the chunk being consumed (c0, a0) and of the next one (c1, a1); slots past
    // k carry (0, 0.0f), so their (zero-filled) pieces add exactly +0.
    int32_t c0 = 0, c1 = 0, c2 = 0;
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f;
    if (lane < k) load_pair(lane, c0, a0);
    if (32 + lane < k) load_pair(32 + lane, c1, a1);
    if (LA2 && 64 + lane < k) load_pair(64 + lane, c2, a2);
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
                    SlabPiece<BF16>::widen(lds128(my_s + (d * kStage + q * 32) * 16), x);
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
        if (LA2) {
            c1 = c2;
            a1 = a2;
            c2 = 0;
            a2 = 0.0f;
            if (j0 + 96 + lane < k) load_pair(j0 + 96 + lane, c2, a2);
        } else {
            c1 = 0;
            a1 = 0.0f;
            if (j0 + 64 + lane < k) load_pair(j0 + 64 + lane, c1, a1);
        }
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
            if (FULL || piece < p.nv) slab_store_piece<E>(p, r, piece * E, tot[q], div, pol_a);
        }
    }
}

// ---------------------------------------------------------------- flow slab kernel (the default)
// The per-row ring kernel above pays, for every (row, slice): the rowptr -> (col, val) -> first
// copies latency chain before its ring is full, the ring's drain at the row's end (refills of
// steps past k_i are zero-fills that still write shared memory), and a 4-row CTA that waits for
// its longest row.  Here a PERSISTENT warp owns a contiguous range of rows balanced by slots
// (flow_search below), and the rows' sampled slots -- padded in the
// workspace to multiples of 4 (column -1, value 0; es_kernels.cu sample_materialize) -- are ONE
// contiguous stream of 4-slot steps.  The cp.async ring therefore runs D steps ahead across row
// boundaries, the (col, val) chunks are 32 consecutive stream slots loaded one chunk ahead, and
// the row metadata (slot ends, divisors) is loaded 32 rows at a time, one batch ahead: a warp
// pays the latency chain once per pass instead of once per row.  Each step belongs to exactly
// one row (the padding), so a row's end is an event of the step stream: after the step that
// completes it, the group partials are combined and stored.
// Per element (bitwise the order of spmm_slab<8, 2, ...>): group e = lane / 8 sums slots
// j = e (mod 4) of the row in slot order, with partials over the row's 32-slot chunks (flushed
// when the stream passes row-local step 8m), then the xor tree over the 4 groups.  Padding
// slots add exactly +0 (zero-filled pieces).
// P = 16-B pieces per lane: a slice of up to 8P pieces (P = 3: 96 fp32 / 192 bf16 elements),
// so F = 602 runs as 7 balanced passes of 21-22 pieces instead of 9 x 16 plus a 7-piece tail.
__device__ __noinline__ void slab_fill_row(const SlabParams& p, int64_t r, float v) {
    for (int c = threadIdx.x & 31; c < p.w; c += 32) {
        if (p.c_mc) st_multicast(p.c_mc + (p.row_base + r) * p.ldc + p.col0 + c, v);
        else if (p.n_peers == 0) p.C[r * p.ldc + c] = v;
        else
            for (int q = 0; q < p.n_peers; ++q) p.c_peers[q][(p.row_base + r) * p.ldc + p.col0 + c] = v;
    }
}

// The row partition of the flow grid: warp w of nw owns rows [i(w), i(w+1)) where i(w) is the
// smallest row index with s_rowptr[i] + kFlowRowCost * i >= total * w / nw (the rows' padded
// slots plus a per-row cost for the epilogue and store, in slot units).  Found by the warp
// itself with a 32-ary search (each round probes 32 rows, one per lane, and keeps the interval
// between the last probe below the target and the first at or above it): ~log32(n) dependent
// loads instead of a partition array in the workspace, so every pass kernel can size its own
// persistent grid.
constexpr int64_t kFlowRowCost = 8;
constexpr int kFlowPad = 16;         // slots: every row of the flow layout is a whole number of 4-step blocks

// Per-warp rare-path state of the flow kernel (shared memory, after the ring).
struct FlowMeta {
    int64_t rb, P0;                 // the warp's first row and first slot
    int32_t nrows, bo, bstart;      // rows; first row of the current batch (from rb); its first step
    int32_t caprel, fetch_t;        // capacity bound (relative to P0); step of the last batch fetch
    uint32_t live, pmask;           // rows of the batch still to stream / to poison at their end
    int32_t endstep[32];            // lane i: row bo + i ends before this stream step
    float divf[32];                 // lane i: its MEAN divisor
    int32_t nse[2][32], nk[2][32];  // raw batches (double-buffered): s_rowptr[r+1] low word, k_i
};
__device__ __forceinline__ int64_t flow_search(const int64_t* __restrict__ s_rowptr, int64_t n, int64_t target,
                                               int lane) {
    int64_t lo = 0, hi = n;          // answer in [lo, hi]; s_rowptr[hi] + c*hi >= target
    while (lo < hi) {
        const int64_t q = lo + (hi - lo) * (lane + 1) / 32;      // lane 31 probes hi
        const bool ge = ld_stream(s_rowptr + q, policy_evict_first()) + kFlowRowCost * q >= target;
        const int f = __ffs(__ballot_sync(kAll, ge)) - 1;       // lane 31 always votes
        const int64_t qf = __shfl_sync(kAll, q, f);
        const int64_t qb = __shfl_sync(kAll, q, f > 0 ? f - 1 : 0);
        lo = f > 0 ? qb + 1 : lo;
        hi = qf;
    }
    return lo;
}

template <int G, int P, int D, int W, int MINB, bool FULL, bool BF16, bool HINT = false>
__global__ void __launch_bounds__(32 * W, MINB)
spmm_slab_flow(const __grid_constant__ SlabParams p) {
    constexpr int E = SlabPiece<BF16>::kElems;
    constexpr int S = 32 / G;            // slots per step
    constexpr int U = G;                 // steps per 32-slot chunk
    static_assert(G == 8 && P >= 2 && P <= 4, "4 slots per step, 2 to 4 pieces per lane");
    constexpr int kBlk = 4;                                      // steps per block = one padded row unit
    static_assert(S * kBlk == kFlowPad && (D == 4 || D == 8), "ring of one or two blocks");
    constexpr int kStage = 32 * P;                               // float4 per warp stage
    constexpr int32_t kNone = 0x7fffffff;
    extern __shared__ __align__(16) float4 slab_ring[];          // [warps][D][P][S][G]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int e = lane / G, sub = lane % G;
    const int64_t gw = (int64_t)blockIdx.x * W + warp;
    const int64_t nw = (int64_t)gridDim.x * W;
    const uint64_t pol = policy_evict_first();
    // the slots' sampling signature (a whole-call guard)
    if (p.ws_sig && *p.ws_sig != p.sig) {
        if (lane == 0 && p.ws_status) atomicOr(p.ws_status, kWsSignature);
        for (int64_t r = p.n_rows * gw / nw; r < p.n_rows * (gw + 1) / nw; ++r) slab_fill_row(p, r, __int_as_float(0x7fc00000));
        return;
    }
    // this warp's rows: an equal share of the rows' padded slots + kFlowRowCost per row
    const int64_t total = ld_stream(p.s_rowptr + p.n_rows, pol) + kFlowRowCost * p.n_rows;
    const int64_t rb = flow_search(p.s_rowptr, p.n_rows, total / nw * gw + total % nw * gw / nw, lane);
    const int64_t re = gw + 1 == nw ? p.n_rows
                                    : flow_search(p.s_rowptr, p.n_rows, total / nw * (gw + 1) + total % nw * (gw + 1) / nw, lane);
    if (rb >= re) return;

    // the warp's stream: slots [P0, P0 + nsl) of the workspace; overflowing rows (slot end past
    // cap, a suffix of the rows) are poisoned and not streamed
    const int64_t P0 = ld_stream(p.s_rowptr + rb, pol);
    int64_t P1 = ld_stream(p.s_rowptr + re, pol);
    const bool huge = P1 - P0 >= (int64_t)0x7fffffff;                 // > 2^31 slots: not streamed
    if (P1 > p.cap) P1 = p.cap & ~(int64_t)(kFlowPad - 1);
    if (huge) P1 = P0;
    const int32_t nsl = P1 > P0 ? (int32_t)(P1 - P0) : 0;          // a multiple of kFlowPad

    // ---- row metadata (rare-path state, kept in shared memory so the step loop's registers are
    // the per-row kernel's): 32 rows per batch, lane i <-> row rb + bo + i; the next batch's raw
    // slot ends (low 32 bits of s_rowptr[r+1]: the stream spans < 2^31 slots, so differences to
    // P0 are exact in 32-bit arithmetic) and k_i (s_k) arrive by cp.async one batch ahead.
    FlowMeta* fm = reinterpret_cast<FlowMeta*>(slab_ring + (size_t)W * D * kStage) + warp;
    if (lane == 0) {
        fm->rb = rb;
        fm->P0 = P0;
        fm->nrows = (int32_t)(re - rb);
        fm->bo = 0;
        fm->bstart = 0;
        // a row ending past the workspace capacity overflowed (relative to P0; -1: every row)
        fm->caprel = (int32_t)max(min(p.cap - P0, (int64_t)0x7fffffff), (int64_t)-1);
        fm->fetch_t = 0;
    }
    __syncwarp();
    auto fetch = [&](int32_t o, int buf) {           // raw metadata of rows rb + o .. + 31
        const int64_t r = fm->rb + o + lane;
        if (o + lane < fm->nrows) {
            cp_async4(&fm->nse[buf][lane], reinterpret_cast<const int32_t*>(p.s_rowptr + r + 1));
            cp_async4(&fm->nk[buf][lane], p.s_k + r);
        }
    };
    int cur = 0;                                      // lane of the current row in its batch
    int32_t cur_end = kNone, next_flush = kNone;
    auto setup = [&](int buf) {                       // the batch at fm->bo from raw buffer buf
        const int32_t bo = fm->bo, nrows = fm->nrows;
        const bool in = bo + lane < nrows;
        const int32_t nse = in ? fm->nse[buf][lane] : 0, nk = in ? fm->nk[buf][lane] : 0;
        const int32_t rel = (int32_t)((uint32_t)nse - (uint32_t)(uint64_t)fm->P0);
        const bool over = in && rel > fm->caprel;
        const int32_t endstep = in && !over ? (int32_t)(rel / S) : 0x3fffffff;
        int32_t st = __shfl_up_sync(kAll, endstep, 1);
        if (lane == 0) st = fm->bstart;
        bool mism = false;
        float dv = (float)nk;
        if (in && (p.reuse_s > 0 || p.mean_by_degree)) {       // the caller's rowptr (not prefetched)
            const int64_t r = fm->rb + bo + lane;
            const int64_t d = ld_stream(p.rowptr + r + 1, policy_evict_first()) - ld_stream(p.rowptr + r, policy_evict_first());
            if (p.mean_by_degree) dv = (float)d;
            if (p.reuse_s > 0 && !over) {
                const int64_t kr = d < (int64_t)p.reuse_s ? d : (int64_t)p.reuse_s;
                mism = nk != kr || (int64_t)(endstep - st) * S != ((kr + kFlowPad - 1) & ~(int64_t)(kFlowPad - 1));
            }
        }
        if ((over || mism) && p.ws_status) atomicOr(p.ws_status, (over ? kWsOverflow : 0) | (mism ? kWsSignature : 0));
        fm->endstep[lane] = endstep;
        fm->divf[lane] = dv;
        const unsigned live = __ballot_sync(kAll, in && !over && endstep > st);
        const unsigned pmask = __ballot_sync(kAll, mism);
        // rows no step belongs to: empty (0, or NaN if the reuse check failed) and overflowing (NaN)
        unsigned special = __ballot_sync(kAll, in && (over || endstep == st));
        const unsigned bad = __ballot_sync(kAll, over || mism);
        if (lane == 0) {
            fm->live = live;
            fm->pmask = pmask;
        }
        while (special) {
            const int i = __ffs(special) - 1;
            special &= special - 1;
            slab_fill_row(p, fm->rb + bo + i, ((bad >> i) & 1u) ? __int_as_float(0x7fc00000) : 0.0f);
        }
        __syncwarp();
    };
    // the next live row (after step t: the batch switch waits for its cp.async metadata)
    auto next_row = [&](int32_t t) {
        unsigned live = fm->live;
        while (live == 0) {
            const int32_t bo = fm->bo + 32;
            if (bo >= fm->nrows) { cur_end = next_flush = kNone; return; }
            // the raw batch was committed with the refill group after step fetch_t; the step
            // loop's wait_group<D-1> has completed it once D + 1 steps have passed since
            if (t < fm->fetch_t + D + 1) cp_async_wait<0>();
            __syncwarp();
            const int32_t bstart = fm->endstep[31];
            __syncwarp();
            if (lane == 0) {
                fm->bstart = bstart;
                fm->bo = bo;
                fm->fetch_t = t;
            }
            __syncwarp();
            setup((bo >> 5) & 1);
            fetch(bo + 32, ((bo >> 5) + 1) & 1);
            live = fm->live;
        }
        cur = __ffs(live) - 1;
        __syncwarp();                                            // every lane has read fm->live
        if (lane == 0) fm->live = live & (live - 1);
        cur_end = fm->endstep[cur];
        next_flush = (cur == 0 ? fm->bstart : fm->endstep[cur - 1]) + U;
        __syncwarp();
    };
    fetch(0, 0);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    setup(0);
    fetch(32, 1);                                     // lands with the prologue's copies
    next_row(kNone - D - 1);

    const uint32_t my_s = smem_u32(slab_ring + (size_t)warp * D * kStage + e * G + sub);
    const char* bl = reinterpret_cast<const char*>(p.B) + sub * 16;
    const uint32_t row_bytes = (uint32_t)(p.ldb * (BF16 ? 2 : 4));
    // padding slots and slots past the stream's end (col -1): zero-filled pieces, no memory read
    auto copy = [&](uint32_t stage, int32_t col) {
        const bool ok = col >= 0;
        const char* src = bl + (uint64_t)(uint32_t)(ok ? col : 0) * row_bytes;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const bool on = FULL ? ok : (ok && sub + G * q < p.nv);
            if constexpr (HINT) cp_async16_zfill_hint(stage + q * 32 * 16, src + q * G * 16, on ? 16u : 0u,
                                                      policy_evict_last());
            else cp_async16_zfill(stage + q * 32 * 16, src + q * G * 16, on ? 16u : 0u);
        }
    };
    auto load_pair = [&](int32_t j, int32_t& c, float& a) {       // stream slot j (coalesced)
        c = -1;
        a = 0.0f;
        if (j < nsl) {
            c = ld_stream(p.s_colind + P0 + j, pol);
            a = p.s_val ? ld_stream(p.s_val + P0 + j, pol) : 1.0f;
        }
    };
    // (col, val) chunks: c0 = the chunk being consumed, c1 = the next; with an 8-step ring the
    // refills read the next chunk from the first step on, so a third (c2) is in flight
    int32_t c0, c1, c2 = -1;
    float a0, a1, a2 = 0.0f;
    load_pair(lane, c0, a0);
    load_pair(32 + lane, c1, a1);
    if (D == 8) load_pair(64 + lane, c2, a2);
#pragma unroll
    for (int t = 0; t < D; ++t) {
        copy(my_s + (uint32_t)t * (kStage * 16), __shfl_sync(kAll, c0, S * t + e));
        cp_async_commit();
    }
    float part[P][E], tot[P][E];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < E; ++c) { part[q][c] = 0.0f; tot[q][c] = 0.0f; }
    // a stream event after step t: the row's 32-slot chunk partial, and at the row's end a5
    auto event = [&](int32_t t) {
#pragma unroll
        for (int q = 0; q < P; ++q)
#pragma unroll
            for (int c = 0; c < E; ++c) { tot[q][c] += part[q][c]; part[q][c] = 0.0f; }
        if (t + 1 == cur_end) {
            const int64_t r = fm->rb + fm->bo + cur;
#pragma unroll
            for (int o = G; o < 32; o <<= 1)
#pragma unroll
                for (int q = 0; q < P; ++q)
#pragma unroll
                    for (int c = 0; c < E; ++c) {
                        const float other = __shfl_xor_sync(kAll, tot[q][c], o);
                        tot[q][c] = (lane & o) ? other + tot[q][c] : tot[q][c] + other;
                    }
            const float dv = fm->divf[cur];
            if ((fm->pmask >> cur) & 1u) {
                slab_fill_row(p, r, __int_as_float(0x7fc00000));
            } else if (e == 0) {
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    const int piece = sub + G * q;
                    if (FULL || piece < p.nv) slab_store_piece_f<E>(p, r, piece * E, tot[q], dv, pol);
                }
            }
#pragma unroll
            for (int q = 0; q < P; ++q)
#pragma unroll
                for (int c = 0; c < E; ++c) tot[q][c] = 0.0f;
            next_row(t);
        } else {
            next_flush += U;
        }
    };
    // The step loop runs BLOCKS of D = 4 steps with static ring stages -- the per-row kernel's
    // inner loop, which the compiler interleaves across the block.  Rows are padded to multiples
    // of 16 slots (4 steps), so every row starts and ends, and every 32-slot partial flushes, on
    // a block boundary: the block body has no event branch (one inside cost 8 accumulator moves
    // and a reconvergence per step), and the row epilogue exists once in the code (inlined per
    // step it overflowed the instruction cache: D = 2 / 4 / 8 ran 9.5 / 10.9 / 21.5 ms on Reddit
    // F=602, profiles/r02_flow_probe.jsonl).
    const int32_t TS = nsl / S;                                  // a multiple of kBlk
#pragma unroll 1
    for (int32_t t = 0; t < TS; t += kBlk) {
        const int u0 = t & (U - 1);
        const uint32_t base = my_s + (uint32_t)(t & (D - 1)) * (kStage * 16);
#pragma unroll
        for (int d = 0; d < kBlk; ++d) {
            const int u = u0 + d;
            const uint32_t stage = base + (uint32_t)d * (kStage * 16);
            cp_async_wait<D - 1>();                              // step t + d has landed
            const float av = __shfl_sync(kAll, a0, S * u + e);
#pragma unroll
            for (int q = 0; q < P; ++q) {
                float x[E];
                SlabPiece<BF16>::widen(lds128(stage + q * 32 * 16), x);
#pragma unroll
                for (int c = 0; c < E; ++c) part[q][c] = fmaf(av, x[c], part[q][c]);
            }
            const int tn = u + D;                                // the stage takes step t + d + D
            const int32_t cn = D == 8 ? __shfl_sync(kAll, c1, (S * u + e) & (32 - 1))
                                      : __shfl_sync(kAll, tn < U ? c0 : c1, (S * tn + e) & (32 - 1));
            copy(stage, cn);
            cp_async_commit();
        }
        if (u0 + kBlk == U) {                                    // the (col, val) chunk is consumed
            c0 = c1;
            a0 = a1;
            if (D == 8) {
                c1 = c2;
                a1 = a2;
                load_pair(S * (t + kBlk + 2 * U) + lane, c2, a2);
            } else {
                load_pair(S * (t + kBlk + U) + lane, c1, a1);
            }
        }
        if (t + kBlk == min(cur_end, next_flush)) event(t + kBlk - 1); // one call site: one epilogue
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------- TMA gather4 slab kernel
// One elected lane per warp feeds a D-stage shared-memory ring with TMA tile::gather4 copies
// (SASS UTMALDG.2D.GATHER4): ONE instruction moves the 256-B slab rows of 4 slots (1 KB, a whole
// step) from L2 into the stage, completion counted by the stage's mbarrier (expect_tx).  The
// LSU no longer writes shared memory (the LDGSTS half of the shared-memory ring's wavefronts);
// the consumer is that kernel's: 8 lanes x 2 LDS.128 per slot, group e = slot 4u + e.  Slots
// past k_i gather row n_cols (out of bounds: the TMA zero-fills without a memory access) and
// columns past F are zero-filled the same way, so the passes are branch-free.  Same order as
// spmm_slab<8, 2, ...> (bitwise).
template <int D, int W, int MINB, bool BF16>
__global__ void __launch_bounds__(32 * W, MINB)
spmm_slab_tma(const __grid_constant__ CUtensorMap tmap, const SlabParams p, int32_t c0_coord, int32_t n_cols) {
    constexpr int G = 8, P = 2, S = 4, U = 8;
    constexpr int E = SlabPiece<BF16>::kElems;
    constexpr uint32_t kStageBytes = 1024;
    static_assert(U % D == 0, "ring depth must divide the steps of a chunk");
    extern __shared__ __align__(1024) unsigned char tma_smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int e = lane / G, sub = lane % G;
    const int64_t r = (int64_t)blockIdx.x * W + warp;
    unsigned char* ring = tma_smem + (size_t)warp * D * kStageBytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(tma_smem + (size_t)W * D * kStageBytes) + warp * D;
    if (r >= p.n_rows) return;
    int64_t beg;
    int32_t k;
    if (!slab_row_slots(p, r, beg, k)) return;
    if (lane == 0) {
        for (int d = 0; d < D; ++d) mbar_init(&bar[d], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint32_t ring_s = smem_u32(ring);
    const uint32_t my_s = ring_s + e * 256 + sub * 16;
    auto load_pair = [&](int64_t j, int32_t& c, float& a) {      // slot j of the row (coalesced)
        const uint64_t pol = policy_evict_first();
        c = ld_stream(p.s_colind + beg + j, pol);
        a = p.s_val ? ld_stream(p.s_val + beg + j, pol) : 1.0f;
    };
    // step t's 4 rows (slots 4t .. 4t+3 of the current / next chunk); warp-collective
    auto issue = [&](int d, int32_t src_c, int32_t j_first) {
        int32_t rows[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int32_t c = __shfl_sync(kAll, src_c, (j_first + i) & 31);
            rows[i] = j_first + i < k ? c : n_cols;                 // OOB row: zero fill
        }
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar[d], kStageBytes);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(ring_s + d * kStageBytes), "l"(&tmap), "r"(c0_coord), "r"(rows[0]), "r"(rows[1]),
                   "r"(rows[2]), "r"(rows[3]), "r"(smem_u32(&bar[d])) : "memory");
        }
    };
    (void)beg;
    int32_t c0 = 0, c1 = 0;
    float a0 = 0.0f, a1 = 0.0f;
    if (lane < k) load_pair(lane, c0, a0);
    if (32 + lane < k) load_pair(32 + lane, c1, a1);
    // issue(d, cols, first slot index relative to the row): the slot's column lives in lane
    // (slot & 31) of c0 (this chunk) or c1 (next chunk)
#pragma unroll
    for (int t = 0; t < D; ++t) issue(t, c0, S * t);
    float part[P][E], tot[P][E];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < E; ++c) { part[q][c] = 0.0f; tot[q][c] = 0.0f; }
    uint32_t phase = 0;                  // bit d: parity of stage d's next completion
    for (int32_t j0 = 0; j0 < k; j0 += 32) {
#pragma unroll 1
        for (int u0 = 0; u0 < U; u0 += D) {
#pragma unroll
            for (int d = 0; d < D; ++d) {                        // step u = u0 + d, stage d
                const int u = u0 + d;
                mbar_wait(&bar[d], (phase >> d) & 1u);
                phase ^= 1u << d;
                const float av = __shfl_sync(kAll, a0, S * u + e);
#pragma unroll
                for (int q = 0; q < P; ++q) {
                    float x[E];
                    SlabPiece<BF16>::widen(lds128(my_s + d * kStageBytes + q * 128), x);
#pragma unroll
                    for (int c = 0; c < E; ++c) part[q][c] = fmaf(av, x[c], part[q][c]);
                }
                __syncwarp();                                    // stage d fully read
                const int tn = u + D;                            // refill: step u + D
                issue(d, tn < U ? c0 : c1, j0 + S * tn);
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
    // drain: the D copies issued past the row's end (all zero-filled) must land before exit
#pragma unroll
    for (int d = 0; d < D; ++d) mbar_wait(&bar[d], (phase >> d) & 1u);
    const uint64_t pol_a = policy_evict_first();
    int64_t div = k;
    if (p.reduce == kMean && p.mean_by_degree)
        div = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
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
            if (piece < p.nv) slab_store_piece<E>(p, r, piece * E, tot[q], div, pol_a);
        }
    }
}

template <int D, int W, int MINB, bool BF16>
cudaError_t launch_tma_slab_w(const CUtensorMap& tm, const SlabParams& p, int32_t c0, int32_t n_cols,
                              cudaStream_t st) {
    const int64_t blocks = (p.n_rows + W - 1) / W;
    const size_t smem = (size_t)W * D * 1024 + (size_t)W * D * 8;
    auto k = spmm_slab_tma<D, W, MINB, BF16>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * W, smem, st>>>(tm, p, c0, n_cols);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- row-pipelined slab kernel
// spmm_slab's gather-FMA with the per-row start-up taken off the critical path: one warp owns
// R <= 32 consecutive rows (lane i holds row i's slot range) and streams their slots as ONE
// sequence, each row padded to a multiple of S = 32/G slots (padding slots are zero-filled
// copies: no memory access, and they add exactly +0), so every step's S slots belong to one row
// and the cp.async ring stays D steps ahead ACROSS row boundaries -- the rowptr -> slots -> B
// latency chain and the ring's fill/drain are paid once per R rows instead of once per row
// (at ~43 steps per Reddit-shaped row they cost about a third of the per-row time; an ideal
// stream of the same gathers reaches the L2 streaming rate, profiles/l2_peak.json gather_smem).
// When the stream passes a row's last step the group partials are combined by the xor tree and
// stored, exactly as spmm_slab does: same per-element order (group e sums slots j = e mod S in
// slot order with 32-slot chunk partials counted from the row's first slot), bitwise.
template <int G, int P, int D, int MINW, bool FULL, int W, int R, bool BF16>
__global__ void __launch_bounds__(32 * W, MINW / W)
spmm_slab_stream(const SlabParams p) {
    constexpr int E = SlabPiece<BF16>::kElems;
    constexpr int S = 32 / G;            // slots per step
    constexpr int U = 32 / S;            // steps per 32-slot chunk (= G)
    static_assert((G == 2 || G == 4 || G == 8 || G == 16) && G * P <= 16, "lanes x pieces per slot");
    static_assert(D >= 2 && U % D == 0 && R >= 1 && R <= 32, "ring depth / rows per warp");
    constexpr int kStage = 32 * P;
    extern __shared__ __align__(16) float4 slab_ring[];          // [warps][D][P][S][G]
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int e = lane / G, sub = lane % G;
    const int64_t r0 = ((int64_t)blockIdx.x * W + warp) * R;
    if (r0 >= p.n_rows) return;
    const int nr = (int)min((int64_t)R, p.n_rows - r0);
    // row metadata in lane i < nr: slots [beg, beg + k), padded to kp = ceil(k / S) * S stream slots
    const uint64_t pol = policy_evict_first();
    int64_t beg = 0;
    int32_t k = 0;
    bool bad = false;
    if (lane < nr) {
        beg = ld_stream(p.s_rowptr + r0 + lane, pol) - p.slot_base;
        int64_t end = ld_stream(p.s_rowptr + r0 + lane + 1, pol) - p.slot_base;
        if (p.direct_s > 0 && end - beg > p.direct_s) end = beg + p.direct_s;
        bool sig_bad = p.ws_sig != nullptr && *p.ws_sig != p.sig;
        if (p.reuse_s > 0 && !sig_bad && end <= p.cap) {
            const int64_t d = ld_stream(p.rowptr + r0 + lane + 1, pol) - ld_stream(p.rowptr + r0 + lane, pol);
            sig_bad = end - beg != (d < p.reuse_s ? d : (int64_t)p.reuse_s);
        }
        bad = end > p.cap || sig_bad;
        if (bad && p.ws_status) atomicOr(p.ws_status, (end > p.cap ? kWsOverflow : 0) | (sig_bad ? kWsSignature : 0));
        k = (!bad && end > beg) ? (int32_t)(end - beg) : 0;
    }
    // rows the guards tripped on: NaN; empty rows: zeros (no division) -- whole-warp stores
    unsigned special = __ballot_sync(kAll, lane < nr && (bad || k == 0));
    while (special) {
        const int i = __ffs(special) - 1;
        special &= special - 1;
        if (__shfl_sync(kAll, (int)bad, i)) {
            slab_poison_row(p, r0 + i);
        } else {
            for (int c = lane; c < p.w; c += 32) {
                if (p.c_mc) st_multicast(p.c_mc + (p.row_base + r0 + i) * p.ldc + p.col0 + c, 0.0f);
                else if (p.n_peers == 0) p.C[(r0 + i) * p.ldc + c] = 0.0f;
                else
                    for (int q = 0; q < p.n_peers; ++q) p.c_peers[q][(p.row_base + r0 + i) * p.ldc + p.col0 + c] = 0.0f;
            }
        }
    }
    const int32_t kp = (k + S - 1) / S * S;
    int32_t incl = kp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(kAll, incl, o);
        if (lane >= o) incl += v;
    }
    const int32_t TP = __shfl_sync(kAll, incl, 31);              // stream length (slots)
    if (TP == 0) return;
    const unsigned nonempty = __ballot_sync(kAll, k > 0);

    const uint32_t my_s = smem_u32(slab_ring + (size_t)warp * D * kStage + e * G + sub);
    const char* bl = reinterpret_cast<const char*>(p.B) + sub * 16;
    const uint32_t row_bytes = (uint32_t)(p.ldb * (BF16 ? 2 : 4));
    // (col, val) of stream slot t, one slot per lane: col = -1 marks a padding slot
    auto load_slot = [&](int32_t t, int32_t& c, float& a) {
        int lo = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const int32_t v = __shfl_sync(kAll, incl, lo + step - 1);
            if (v <= t) lo += step;
        }
        const int i = lo > 31 ? 31 : lo;
        const int64_t b = __shfl_sync(kAll, beg, i);
        const int32_t ki = __shfl_sync(kAll, k, i);
        const int32_t j = t - (__shfl_sync(kAll, incl, i) - __shfl_sync(kAll, kp, i));
        c = -1;
        a = 0.0f;
        if (t < TP && j < ki) {
            c = ld_stream(p.s_colind + b + j, pol);
            a = p.s_val ? ld_stream(p.s_val + b + j, pol) : 1.0f;
        }
    };
    auto copy = [&](int stage, int32_t col) {
        const bool valid = col >= 0;
        const char* src = bl + (uint64_t)(uint32_t)(valid ? col : 0) * row_bytes;
#pragma unroll
        for (int q = 0; q < P; ++q) {
            const bool on = FULL ? valid : (valid && sub + G * q < p.nv);
            cp_async16_zfill(my_s + (stage * kStage + q * 32) * 16, src + q * G * 16, on ? 16u : 0u);
        }
    };
    int32_t c0, c1;
    float a0, a1;
    load_slot(lane, c0, a0);
    load_slot(32 + lane, c1, a1);
#pragma unroll
    for (int t = 0; t < D; ++t) {
        copy(t, __shfl_sync(kAll, c0, S * t + e));
        cp_async_commit();
    }
    float part[P][E], tot[P][E];
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
        for (int c = 0; c < E; ++c) { part[q][c] = 0.0f; tot[q][c] = 0.0f; }
    int cur = __ffs(nonempty) - 1;                               // row being accumulated
    int32_t cur_end = __shfl_sync(kAll, incl, cur) / S;          // its last stream step + 1
    int32_t js = 0;                                              // step index within the row
    const int32_t TS = TP / S;
    // one step per iteration (not unrolled: the row epilogue below exists once in the code)
#pragma unroll 1
    for (int32_t ts = 0; ts < TS; ++ts) {
        const int u = ts & (U - 1);                              // step within the stream chunk
        const int d = ts & (D - 1);                              // ring stage
        cp_async_wait<D - 1>();                                  // step ts has landed
        const float av = __shfl_sync(kAll, a0, S * u + e);
#pragma unroll
        for (int q = 0; q < P; ++q) {
            float x[E];
            SlabPiece<BF16>::widen(lds128(my_s + (d * kStage + q * 32) * 16), x);
#pragma unroll
            for (int c = 0; c < E; ++c) part[q][c] = fmaf(av, x[c], part[q][c]);
        }
        const int tn = u + D;                                    // refill: stream step ts + D
        const int32_t cn = __shfl_sync(kAll, tn < U ? c0 : c1, (S * tn + e) & 31);
        copy(d, ts + D < TS ? cn : -1);
        cp_async_commit();
        if (u == U - 1) {                                        // the stream chunk is consumed
            c0 = c1;
            a0 = a1;
            load_slot(S * (ts + 1 + U) + lane, c1, a1);
        }
        ++js;
        const bool row_done = ts + 1 == cur_end;
        if ((js & (U - 1)) == 0 || row_done) {                   // the row's 32-slot chunk partial
#pragma unroll
            for (int q = 0; q < P; ++q)
#pragma unroll
                for (int c = 0; c < E; ++c) { tot[q][c] += part[q][c]; part[q][c] = 0.0f; }
        }
        if (row_done) {                                          // a5: row r0 + cur is complete
            const int32_t kc = __shfl_sync(kAll, k, cur);
            int64_t div = kc;
            if (p.reduce == kMean && p.mean_by_degree)
                div = ld_stream(p.rowptr + r0 + cur + 1, pol) - ld_stream(p.rowptr + r0 + cur, pol);
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
                    if (FULL || piece < p.nv) slab_store_piece<E>(p, r0 + cur, piece * E, tot[q], div, pol);
                }
            }
#pragma unroll
            for (int q = 0; q < P; ++q)
#pragma unroll
                for (int c = 0; c < E; ++c) tot[q][c] = 0.0f;
            const unsigned rest = nonempty & ~((2u << cur) - 1u);
            cur = rest ? __ffs(rest) - 1 : 31;
            cur_end = __shfl_sync(kAll, incl, cur) / S;
            js = 0;
        }
    }
    cp_async_wait<0>();
}

template <int G, int P, int D, int MINW, int W, int R>
cudaError_t launch_slab_stream_w(const SlabParams& p, cudaStream_t st) {
    const int64_t warps = (p.n_rows + R - 1) / R;
    const int64_t blocks = (warps + W - 1) / W;
    const size_t smem = (size_t)W * D * 32 * P * 16;
    auto k = p.nv == G * P ? spmm_slab_stream<G, P, D, MINW, true, W, R, false>
                           : spmm_slab_stream<G, P, D, MINW, false, W, R, false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

// rows per warp = tune.variant >> 8 (2, 4 default, 8, 16), warps per CTA 4
template <int G, int P, int D, int MINW>
cudaError_t launch_slab_stream_k(const SlabParams& p, const Tune& t, cudaStream_t st) {
    const int R = (t.variant >> 8) & 0xff;
    if (R == 2) return launch_slab_stream_w<G, P, D, MINW, 4, 2>(p, st);
    if (R == 8) return launch_slab_stream_w<G, P, D, MINW, 4, 8>(p, st);
    if (R == 16) return launch_slab_stream_w<G, P, D, MINW, 4, 16>(p, st);
    return launch_slab_stream_w<G, P, D, MINW, 4, 4>(p, st);
}

template <int G, int P, int D, int MINB, int W, bool BF16 = false, bool LA2 = false>
cudaError_t launch_slab_w(const SlabParams& p, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + W - 1) / W;
    const size_t smem = (size_t)W * D * 32 * P * 16;
    auto k = p.nv == G * P ? spmm_slab<G, P, D, MINB, true, W, BF16, LA2> : spmm_slab<G, P, D, MINB, false, W, BF16, LA2>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k<<<(unsigned)blocks, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

template <int G, int D, int MINB, int P = 16 / G>
cudaError_t launch_slab_k(const SlabParams& p, int cta_warps, cudaStream_t st, bool la2 = false) {
    if constexpr (G != 16)
        if (la2) return cta_warps == 2 ? launch_slab_w<G, P, D, MINB, 2, false, true>(p, st)
                                       : launch_slab_w<G, P, D, MINB, 4, false, true>(p, st);
    if (cta_warps == 1) return launch_slab_w<G, P, D, MINB, 1>(p, st);
    if (cta_warps == 2) return launch_slab_w<G, P, D, MINB, 2>(p, st);
    if (cta_warps == 8) return launch_slab_w<G, P, D, MINB, 8>(p, st);
    return launch_slab_w<G, P, D, MINB, 4>(p, st);
}

// MINW: min resident warps per SM the register cap is set for
template <int G, int P, int D, int W, int MINW, bool BF16>
cudaError_t launch_ldg_w(const SlabParams& p, int cache, cudaStream_t st) {
    const int64_t blocks = (p.n_rows + W - 1) / W;
    const bool full = p.nv == G * P;
    auto k = full ? (cache ? spmm_slab_ldg<G, P, D, W, MINW, BF16, true, 1> : spmm_slab_ldg<G, P, D, W, MINW, BF16, true, 0>)
                  : (cache ? spmm_slab_ldg<G, P, D, W, MINW, BF16, false, 1>
                           : spmm_slab_ldg<G, P, D, W, MINW, BF16, false, 0>);
    k<<<(unsigned)blocks, 32 * W, 0, st>>>(p);
    return cudaGetLastError();
}

template <int G, int P, int D, int MINW, bool BF16>
cudaError_t launch_ldg_k(const SlabParams& p, const Tune& t, cudaStream_t st) {
    const int cache = t.variant & 1;
    if (t.cta_warps == 2) return launch_ldg_w<G, P, D, 2, MINW, BF16>(p, cache, st);
    return launch_ldg_w<G, P, D, 4, MINW, BF16>(p, cache, st);
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
    if (p.direct_s > 0 && end - beg > p.direct_s) end = beg + p.direct_s;
    bool sig_bad = p.ws_sig != nullptr && *p.ws_sig != p.sig;
    const int64_t deg = ld_stream(p.rowptr + r + 1, pol_a) - ld_stream(p.rowptr + r, pol_a);
    const int32_t pad = p.pad > 1 ? p.pad : 1;
    if (p.reuse_s > 0 && !sig_bad && end <= p.cap) {
        const int64_t kr = deg < p.reuse_s ? deg : (int64_t)p.reuse_s;
        sig_bad = end - beg != (kr + pad - 1) / pad * pad;
    }
    if (slab_row_guard(p, end, sig_bad)) return;      // dB is accumulated into: flagged, not poisoned
    // slots [beg, end): k_i sampled ones, then (flow layout) padding slots with column -1
    const int32_t k = end > beg ? (int32_t)(end - beg) : 0;
    if (k == 0) return;
    const int64_t ks = deg < (int64_t)p.s ? deg : (int64_t)p.s;
    float div = (float)ks;
    if (p.reduce == kMean && p.mean_by_degree) div = (float)deg;
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
            if (slot < n_here && cn >= 0) {
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

// ---- flow launchers.  Register caps (blocks of 4 warps per SM): 8 (64 registers) for 2 fp32
// pieces per lane, 6 (80) for 3; bf16 (8 accumulators per piece) 6 and 5.  Each pass runs a
// persistent grid of SMs x (that kernel's occupancy) CTAs: every warp is resident at once.
template <int P, bool BF16> struct FlowCap;
template <> struct FlowCap<2, false> { static constexpr int kMinB = 8; };
template <> struct FlowCap<3, false> { static constexpr int kMinB = 6; };
template <> struct FlowCap<2, true> { static constexpr int kMinB = 6; };
template <> struct FlowCap<3, true> { static constexpr int kMinB = 5; };
template <> struct FlowCap<4, false> { static constexpr int kMinB = 5; };

template <int P, int D, int W, bool BF16, bool FULL, bool HINT = false>
cudaError_t launch_flow_k(const SlabParams& p, cudaStream_t st) {
    // one block less for the variants whose extra predicates / accumulators would otherwise spill
    // (an 8-step ring is shared-memory bound at 6 / 4 blocks: its register cap follows)
    constexpr int kMinB = D == 8 ? (P == 2 ? 6 : 4)
                                 : FlowCap<P, BF16>::kMinB -
                                       ((BF16 || (P == 2 && (!FULL || HINT)) || (P == 4 && FULL && !HINT)) ? 1 : 0);
    auto k = spmm_slab_flow<8, P, D, W, kMinB * 4 / W, FULL, BF16, HINT>;
    constexpr size_t smem = (size_t)W * D * 32 * P * 16 + (size_t)W * sizeof(FlowMeta);
    // grid = SMs x resident CTAs, computed once per device (occupancy queries are not free)
    static std::atomic<int> grid_cache[8];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    int grid = dev < 8 ? grid_cache[dev].load(std::memory_order_relaxed) : 0;
    if (grid <= 0) {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
        int sms = 0, nb = 0;
        cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32 * W, smem);
        if (e != cudaSuccess) return e;
        grid = sms * (nb > 0 ? nb : 1);
        if (dev < 8) grid_cache[dev].store(grid, std::memory_order_relaxed);
    }
    k<<<(unsigned)grid, 32 * W, smem, st>>>(p);
    return cudaGetLastError();
}

template <int P, int D, int W, bool BF16, bool HINT = false>
cudaError_t launch_flow_w(const SlabParams& p, cudaStream_t st) {
    return p.nv == 8 * P ? launch_flow_k<P, D, W, BF16, true, HINT>(p, st)
                         : launch_flow_k<P, D, W, BF16, false, HINT>(p, st);
}

}  // namespace

// ring depth tune.stages (4 default = one 4-step block; 8), warps per CTA W = tune.cta_warps (8
// default; 4); bf16 B: 4-step ring, 4-warp CTAs
cudaError_t launch_slab_flow(const SlabParams& p, const Tune& t, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    if (p.nv > 32 || p.nv < 1 || (p.b_bf16 && p.nv > 24)) return cudaErrorInvalidValue;
    const bool p3 = p.nv > 16;
    // a slice of 25-32 pieces (the last one, with a short remainder merged): 4 pieces per lane,
    // 4-warp CTAs, 4-step ring
    if (p.nv > 24) return (t.variant & 1) ? launch_flow_w<4, 4, 4, false, true>(p, st)
                                          : launch_flow_w<4, 4, 4, false>(p, st);
    if (p.b_bf16) {
        if (t.stages == 8) return cudaErrorInvalidValue;
        return p3 ? launch_flow_w<3, 4, 4, true>(p, st) : launch_flow_w<2, 4, 4, true>(p, st);
    }
    if (t.stages == 8) return p3 ? launch_flow_w<3, 8, 4, false>(p, st) : launch_flow_w<2, 8, 4, false>(p, st);
    if (t.variant & 1) {                 // A/B: evict_last L2 policy on the slab gathers
        if (p.nv > 24) return launch_flow_w<4, 4, 4, false, true>(p, st);
        return p3 ? launch_flow_w<3, 4, 8, false, true>(p, st) : launch_flow_w<2, 4, 8, false, true>(p, st);
    }
    // 8-warp CTAs by default (Reddit F=602 6.97 vs 7.16 ms, F=128 1.61 vs 1.65, Proteins 1.093 vs
    // 1.121 with 4; profiles/r02_flow_probe.jsonl)
    if (t.cta_warps == 4) return p3 ? launch_flow_w<3, 4, 4, false>(p, st) : launch_flow_w<2, 4, 4, false>(p, st);
    return p3 ? launch_flow_w<3, 4, 8, false>(p, st) : launch_flow_w<2, 4, 8, false>(p, st);
}

// Slab kernel selection.  Default: the shared-memory ring, G = tune.width (8 default, or 16)
// lanes x 16-B pieces per slot (profiles/r02.md: it beats the register-direct and the TMA
// gather4 kernels on every measured config -- they are latency- resp. TMA-rate-bound).
// ES_KERNEL_SLAB_LDG: the register-direct kernel, 8 lanes x one 32-B piece per slot (4 slots per
// step) for a full 256-B slice, 4 lanes (8 slots per step) for a slice of <= 4 pieces, 2 lanes for
// <= 2 -- needs B and its row pitch 32-B aligned (p.b32); ring depth tune.stages (4 default; 2,
// 8).  The register caps below are the largest that do not spill (spilling cp.async kernels
// trapped on B200, _build.py refuses them).
cudaError_t launch_slab_pass(const SlabParams& p, const Tune& t, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    const bool ldg = p.b32 && t.kernel == ES_KERNEL_SLAB_LDG;
    if (ldg) {
        const int np = p.nv;                 // 32-B pieces in this slice (<= 8)
        // register caps (MINW resident warps per SM) that do not spill: the D-deep ring holds
        // D x 8 registers per piece
        if (p.b_bf16) {
            if (np <= 2) return launch_ldg_k<2, 1, 2, 24, true>(p, t, st);
            if (np <= 4) return launch_ldg_k<4, 1, 4, 16, true>(p, t, st);
            return launch_ldg_k<8, 1, 4, 16, true>(p, t, st);
        }
        if (np <= 2) return launch_ldg_k<2, 1, 2, 24, false>(p, t, st);
        if (np <= 4) return launch_ldg_k<4, 1, 4, 16, false>(p, t, st);
        if (t.stages == 8) return launch_ldg_k<8, 1, 8, 12, false>(p, t, st);
        if (t.stages == 2) return launch_ldg_k<8, 1, 2, 24, false>(p, t, st);
        return launch_ldg_k<8, 1, 4, 16, false>(p, t, st);
    }
    if (t.kernel == ES_KERNEL_SLAB_STREAM && !p.b_bf16) {
        if (p.nv <= 4) return launch_slab_stream_k<2, 2, 2, 32>(p, t, st);
        if (p.nv <= 8) return launch_slab_stream_k<4, 2, 4, 32>(p, t, st);
        return launch_slab_stream_k<8, 2, 4, 28>(p, t, st);
    }
    const int cw = t.cta_warps;
    if (p.b_bf16) {                      // bf16 B (NEXT-4): 128-element slices, 8 elements per piece
        if (p.nv <= 4) return launch_slab_w<2, 2, 2, 3, 4, true>(p, st);
        if (p.nv <= 8) return launch_slab_w<4, 2, 4, 3, 4, true>(p, st);
        return t.width == 16 ? launch_slab_w<16, 1, 4, 4, 4, true>(p, st)
                             : launch_slab_w<8, 2, 4, 3, 4, true>(p, st);
    }
    if (t.width == 16) {
        switch (t.stages) {
            case 2: return launch_slab_k<16, 2, 5>(p, cw, st);
            case 8: return launch_slab_k<16, 8, 4>(p, cw, st);
            default: return launch_slab_k<16, 4, 5>(p, cw, st);
        }
    }
    // narrow last slice: 4 lanes x 2 pieces (8 slots per step) for <= 8 pieces, 2 x 2 (16 slots
    // per step) for <= 4 -- half / a quarter of the steps of a full slice
    const bool la2 = (t.variant & 1) != 0;  // A/B: two-chunk (col, val) lookahead
    if (p.nv <= 4) return launch_slab_k<2, 2, 4, 2>(p, cw, st, la2);
    if (p.nv <= 8) return launch_slab_k<4, 4, 4, 2>(p, cw, st, la2);
    switch (t.stages) {
        case 2: return launch_slab_k<8, 2, 4>(p, cw, st);
        case 8: return launch_slab_k<8, 8, 4>(p, cw, st);
        default:
            if (t.variant & 2) return launch_slab_k<8, 4, 3>(p, cw, st, la2);   // 80-register cap
            return launch_slab_k<8, 4, 4>(p, cw, st, la2);
    }
}

// The TMA gather4 kernel over one slice: column coordinate c0 of the tensor map over all of B
// (es_abi.cu encodes it once per call).  ring depth tune.stages (4 default; 2, 8), warps per CTA
// tune.cta_warps (4 default; 2, 8).
cudaError_t launch_slab_pass_tma(const CUtensorMap& tm, const SlabParams& p, int32_t c0, int32_t n_cols,
                                 const Tune& t, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    if (p.b_bf16) return launch_tma_slab_w<4, 4, 4, true>(tm, p, c0, n_cols, st);
    if (t.stages == 2) return t.cta_warps == 8 ? launch_tma_slab_w<2, 8, 4, false>(tm, p, c0, n_cols, st)
                                               : launch_tma_slab_w<2, 4, 8, false>(tm, p, c0, n_cols, st);
    if (t.stages == 8) return t.cta_warps == 8 ? launch_tma_slab_w<8, 8, 3, false>(tm, p, c0, n_cols, st)
                                               : launch_tma_slab_w<8, 4, 6, false>(tm, p, c0, n_cols, st);
    if (t.cta_warps == 8) return launch_tma_slab_w<4, 8, 4, false>(tm, p, c0, n_cols, st);
    if (t.cta_warps == 2) return launch_tma_slab_w<4, 2, 16, false>(tm, p, c0, n_cols, st);
    return launch_tma_slab_w<4, 4, 8, false>(tm, p, c0, n_cols, st);
}

cudaError_t launch_slab_backward(const SlabParams& p, const float* dC, float* dB, cudaStream_t st) {
    if (p.n_rows <= 0) return cudaSuccess;
    constexpr int W = 4;
    spmm_slab_bwd<W><<<(unsigned)((p.n_rows + W - 1) / W), 32 * W, 0, st>>>(p, dC, dB);
    return cudaGetLastError();
}

bool encode_b_tensor_map(CUtensorMap* tm, const void* B, int64_t F, int64_t ldb, int64_t n_cols, bool bf16) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    // resolved once (thread-safe static initialisation); immutable afterwards
    static const Encode encode = []() -> Encode {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<Encode>(fn);
    }();
    const int64_t esz = bf16 ? 2 : 4;
    if (!encode || reinterpret_cast<uintptr_t>(B) % 16 != 0 || (ldb * esz) % 16 != 0 || n_cols < 1 ||
        n_cols >= (int64_t)1 << 31 || F < 1)
        return false;
    const cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)n_cols};   // columns >= F: zero fill
    const cuuint64_t strides[1] = {(cuuint64_t)(ldb * esz)};
    const cuuint32_t box[2] = {(cuuint32_t)(256 / esz), 1};          // one 256-B slab row
    const cuuint32_t estr[2] = {1, 1};
    return encode(tm, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(B), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t slab_scan_temp_bytes(int64_t n) {
    size_t temp = 0;
    if (n > 0) cub::DeviceScan::InclusiveSum(nullptr, temp, (int64_t*)nullptr, (int64_t*)nullptr, n);
    return temp;
}

cudaError_t launch_slab_count(const int64_t* rowptr, int64_t n, int32_t s, int64_t* s_rowptr, void* temp,
                              size_t temp_bytes, cudaStream_t st, int* launches, WsHeader* hdr, int32_t pad,
                              int32_t* s_k) {
    cudaError_t err = launch_sample_count_only(rowptr, n, s, s_rowptr, st, hdr, pad, s_k);
    ++*launches;
    if (err != cudaSuccess || n == 0) return err;
    err = cub::DeviceScan::InclusiveSum(temp, temp_bytes, s_rowptr + 1, s_rowptr + 1, n, st);
    *launches += 2;                      // CUB's scan: DeviceScanInitKernel + DeviceScanKernel (ncu)
    return err;
}

}  // namespace es
