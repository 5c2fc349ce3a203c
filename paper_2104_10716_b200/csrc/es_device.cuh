// es_device.cuh -- device helpers of the sm_100a ES-SpMM path (sampling arithmetic,
// cache-hinted memory ops).  Shares nothing with oracle/ (independent implementation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace es {

constexpr uint32_t kPrime = 577u;                      // P'
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;    // reading R6
constexpr int kBucket = 1, kFastRand = 2;
constexpr int kSum = 0, kMean = 1;

// splitmix64 finalizer (reading R6).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

// Per-row sampling state: Alg. 1 l.5-6 (S = min(row_nnz, s)) plus the R6 rotation.
struct RowSampler {
    int64_t beg;      // first nonzero of the row (index into the local colind/val)
    int64_t d;        // row_nnz
    int32_t k;        // min(d, s)
    int32_t strategy;
    uint64_t off;     // FastRand rotation, 0 for seed == 0
    uint32_t prime;   // P' (577, L1058; NEXT-4 override)
    bool narrow;      // all positions computable in 32-bit unsigned arithmetic

    __device__ __forceinline__ void init(int64_t b, int64_t e, int32_t s, int32_t strat,
                                         uint64_t seed, int64_t global_row, uint32_t pp) {
        beg = b;
        d = e - b;
        k = d < (int64_t)s ? (int32_t)d : s;
        strategy = strat;
        prime = pp;
        off = (strat == kFastRand && seed != 0 && d > 0)
                  ? mix64(seed + kGolden * (uint64_t)(global_row + 1)) % (uint64_t)d : 0;
        // off < d, j < k <= s: off + j*P' < 2^32 guarantees exact 32-bit arithmetic.
        narrow = (uint64_t)d + (uint64_t)(k > 0 ? k - 1 : 0) * pp < (1ull << 32);
    }

    // Position within the row of slot j < k.  Bucket: j (L1043).  FastRand: Eq. 2
    // (L1066) rotated by off (R6): (off + j*P') mod d.
    __device__ __forceinline__ int64_t pos(int32_t j) const {
        if (strategy == kBucket) return j;
        if (narrow) return (int64_t)(((uint32_t)off + (uint32_t)j * prime) % (uint32_t)d);
        return (int64_t)((off + (uint64_t)j * prime) % (uint64_t)d);
    }
};

// ---- L2 cache policies: A-side streams once (evict_first), B rows are re-gathered
// across rows (evict_last), C is written once (evict_first).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int64_t ld_stream(const int64_t* p, uint64_t pol) {
    int64_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}

// Vector of VEC fp32 values.
template <int VEC> struct Vec;
template <> struct Vec<4> { float v[4]; };
template <> struct Vec<2> { float v[2]; };
template <> struct Vec<1> { float v[1]; };

template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_gather(const float* p, uint64_t pol);

template <> __device__ __forceinline__ Vec<4> ld_gather<4>(const float* p, uint64_t pol) {
    Vec<4> r;
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "l"(p), "l"(pol));
    return r;
}
template <> __device__ __forceinline__ Vec<2> ld_gather<2>(const float* p, uint64_t pol) {
    Vec<2> r;
    asm("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
        : "=f"(r.v[0]), "=f"(r.v[1]) : "l"(p), "l"(pol));
    return r;
}
template <> __device__ __forceinline__ Vec<1> ld_gather<1>(const float* p, uint64_t pol) {
    Vec<1> r;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.v[0]) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ void st_stream(float* p, float a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(a), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream4(float* p, const float* a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]), "f"(a[3]), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream2(float* p, const float* a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;"
                 :: "l"(p), "f"(a[0]), "f"(a[1]), "l"(pol) : "memory");
}

// Stores to an NVLS multicast address (multimem.st): one store, delivered by the NVSwitch to
// the bound buffer of every rank (the fused C all-gather, NEXT-1).
__device__ __forceinline__ void st_multicast4(float* p, const float* a) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(a[0]), "f"(a[1]), "f"(a[2]), "f"(a[3]) : "memory");
}
__device__ __forceinline__ void st_multicast(float* p, float a) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" :: "l"(p), "f"(a) : "memory");
}

// Vector reductions into global memory (SASS REDG.E.ADD.F32x4): relaxed, gpu scope.  Note the
// hardware add flushes fp32 denormals to zero (FTZ), unlike the FMA path.
__device__ __forceinline__ void red_add4(float* p, float a, float b, float c, float d) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red_add2(float* p, float a, float b) {
    asm volatile("red.relaxed.gpu.global.add.v2.f32 [%0], {%1,%2};" :: "l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red_add1(float* p, float a) {
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" :: "l"(p), "f"(a) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- per-thread async copies (cp.async, SASS LDGSTS): global -> shared, 16 B, L2 only
template <bool kHint = true>
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint64_t pol) {
    if constexpr (kHint)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
                     :: "r"(smem_u32(dst)), "l"(src), "l"(pol) : "memory");
    else
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
// 4-B global -> shared copy (cp.async.ca; the flow kernel's row metadata)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// ---- mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.b32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-B aligned ends), completion
// reported to `bar` as transaction bytes; L2 eviction policy hint.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                 " [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

}  // namespace es
