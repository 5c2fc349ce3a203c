// L2 ceilings on this B200 (roofline denominators for L2-resident gathers; tuning evidence, not
// part of the library).  Prints one JSON line per probe.
//   stream      : every thread streams float4 (ld.global.cg, L2 only) over a footprint of X bytes,
//                 R times: the L2 streaming read rate -- bench.py's roofline peak for the slab
//                 passes and L2-resident fused configs (profiles/l2_peak.json).
//   gather_ldg  : random 256-B rows of an X-byte slab, 8 lanes x 2 float4 per row, U rows in
//                 flight per lane group (register-direct gathers).
//   gather_smem : the same rows through a per-warp cp.async ring (LDGSTS) read back with LDS --
//                 the shared-memory-staged pattern of es::spmm_slab at ideal row lengths.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2peak scripts/l2peak.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\":\"%s at %d\"}\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
  return (uint32_t)x;
}

__global__ void stream_read(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
      float4 a = __ldcg(p + i), b = __ldcg(p + i + stride), c = __ldcg(p + i + 2 * stride),
             d = __ldcg(p + i + 3 * stride);
      acc += a.x + b.y + c.z + d.w;
    }
    for (; i < n4; i += stride) { float4 a = __ldcg(p + i); acc += a.x; }
  }
  if (acc == 1234.5f) *sink = acc;
}

// each warp: rows g = warp*steps*4 + 4t + e (group e = lane/8), lane sub = lane%8 owns float4 sub, sub+8
template <int U>
__global__ void gather_ldg(const float4* __restrict__ slab, uint32_t nrows, long steps, float* sink) {
  const int lane = threadIdx.x & 31, e = lane >> 3, sub = lane & 7;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  for (long t = 0; t < steps; t += U) {
    float4 v[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t row = hash32((uint64_t)(warp * steps + t + u) * 4 + e) % nrows;
      v[u][0] = __ldcg(slab + (size_t)row * 16 + sub);
      v[u][1] = __ldcg(slab + (size_t)row * 16 + sub + 8);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u][0].x + v[u][1].w;
  }
  if (acc == 1234.5f) *sink = acc;
}

template <int D>
__global__ void gather_smem(const float4* __restrict__ slab, uint32_t nrows, long steps, float* sink) {
  extern __shared__ float4 ring[];                       // [warps][D][4 rows][16]
  const int lane = threadIdx.x & 31, e = lane >> 3, sub = lane & 7, w = threadIdx.x >> 5;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4* my = ring + (size_t)w * D * 64 + e * 16 + sub;
  auto issue = [&](int d, long t) {
    const uint32_t row = hash32((uint64_t)(warp * steps + t) * 4 + e) % nrows;
    const float4* src = slab + (size_t)row * 16 + sub;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(my + d * 64);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0), "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0 + 128), "l"(src + 8) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc = 0.f;
#pragma unroll
  for (int d = 0; d < D; ++d) issue(d, d);
  for (long t = 0; t < steps; t += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      asm volatile("cp.async.wait_group %0;" :: "n"(D - 1) : "memory");
      const float4 a = my[d * 64], b = my[d * 64 + 8];
      acc += a.x + b.w;
      issue(d, t + d + D);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 1234.5f) *sink = acc;
}

// gather_smem + the slab kernel's per-step work: row indices from a coalesced index array in a
// 32-slot chunk window (one chunk ahead), the column broadcast by shuffle, a value broadcast, 8 FMAs
// per lane per step -- no row boundaries (an endless row).  MODE 0: all of it; 1: no FMA/value;
// 2: hashed indices (no index loads) but with FMAs
template <int D, int MODE>
__global__ void gather_smem_fma(const float4* __restrict__ slab, const int* __restrict__ idx, long steps,
                                float* sink) {
  extern __shared__ float4 ring[];
  const int lane = threadIdx.x & 31, e = lane >> 3, sub = lane & 7, w = threadIdx.x >> 5;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int* my_idx = idx + warp * steps * 4;
  float4* my = ring + (size_t)w * D * 64 + e * 16 + sub;
  auto copy = [&](int d, int row) {
    const float4* src = slab + (size_t)row * 16 + sub;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(my + d * 64);
    if (MODE == 3) {                                   // the zero-fill (src-size) form the kernel uses
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(s0), "l"(src), "r"(16) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(s0 + 128), "l"(src + 8), "r"(16) : "memory");
    } else {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0), "l"(src) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0 + 128), "l"(src + 8) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto row_of = [&](long slot, int c_lane) {
    if (MODE == 2) return (int)(hash32((uint64_t)(warp * steps * 4 + slot)) % 245760u);
    return c_lane;
  };
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto ldi = [&](const int* q) {             // MODE 4: the kernel's ld_stream (L1::no_allocate + evict_first)
    if (MODE != 4) return __ldcs(q);
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(q), "l"(pol));
    return v;
  };
  int c0 = MODE == 2 ? 0 : ldi(my_idx + lane), c1 = MODE == 2 ? 0 : ldi(my_idx + 32 + lane);
  float a0 = 1.0f;
  float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int d = 0; d < D; ++d) copy(d, row_of(4 * d + e, __shfl_sync(~0u, c0, 4 * d + e)));
  const long nslots = steps * 4;
  for (long j0 = 0; j0 < nslots; j0 += 32) {
#pragma unroll 1
    for (int u0 = 0; u0 < 8; u0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int u = u0 + d;
        asm volatile("cp.async.wait_group %0;" :: "n"(D - 1) : "memory");
        const float4 a = my[d * 64], b = my[d * 64 + 8];
        if (MODE == 1) {
          part[0] += a.x + b.w;
        } else {
          const float av = __shfl_sync(~0u, a0, 4 * u + e);
          part[0] = fmaf(av, a.x, part[0]); part[1] = fmaf(av, a.y, part[1]);
          part[2] = fmaf(av, a.z, part[2]); part[3] = fmaf(av, a.w, part[3]);
          part[4] = fmaf(av, b.x, part[4]); part[5] = fmaf(av, b.y, part[5]);
          part[6] = fmaf(av, b.z, part[6]); part[7] = fmaf(av, b.w, part[7]);
        }
        const int tn = u + D;
        const int cn = __shfl_sync(~0u, tn < 8 ? c0 : c1, (4 * tn + e) & 31);
        copy(d, row_of(j0 + 4 * tn + e, cn));
      }
    }
    c0 = c1;
    if (MODE != 2) c1 = (j0 + 64 + 32 <= nslots) ? ldi(my_idx + j0 + 64 + lane) : 0;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += part[i];
  if (acc == 1234.5f) *sink = acc;
}

// MODE 5: the index chunks arrive by TMA (cp.async.bulk.tensor.1d over the index array, 32
// indices = 128 B per chunk, issued two chunks ahead by one lane, mbarrier completion) and are
// read back from shared memory -- the index loads leave the LSU / L1 miss path the gathers use.
template <int D>
__global__ void gather_smem_tmaidx(const __grid_constant__ CUtensorMap tm, const float4* __restrict__ slab,
                                   long steps, float* sink) {
  extern __shared__ float4 ring[];
  constexpr int W = 4;
  const int lane = threadIdx.x & 31, e = lane >> 3, sub = lane & 7, w = threadIdx.x >> 5;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4* my = ring + (size_t)w * D * 64 + e * 16 + sub;
  __shared__ __align__(128) int idxbuf[W][3][32];
  __shared__ __align__(8) uint64_t bars[W][3];
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[w][0]);
  const uint32_t ib0 = (uint32_t)__cvta_generic_to_shared(&idxbuf[w][0][0]);
  if (lane == 0) {
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0 + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const long base = warp * steps * 4;
  auto fetch = [&](long chunk) {                       // chunk -> buffer chunk % 3
    if (lane == 0) {
      const int b = (int)(chunk % 3);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" :: "r"(bar0 + 8 * b) : "memory");
      asm volatile("cp.async.bulk.tensor.1d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   :: "r"(ib0 + 128 * b), "l"(&tm), "r"((int)(base + 32 * chunk)), "r"(bar0 + 8 * b) : "memory");
    }
  };
  uint32_t phase[3] = {0, 0, 0};
  auto wait = [&](long chunk) {
    const int b = (int)(chunk % 3);
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.b32 %0,1,0,p;}"
                   : "=r"(done) : "r"(bar0 + 8 * b), "r"(phase[b]) : "memory");
    phase[b] ^= 1;
  };
  auto copy = [&](int d, int row) {
    const float4* src = slab + (size_t)row * 16 + sub;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(my + d * 64);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0), "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s0 + 128), "l"(src + 8) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  fetch(0); fetch(1); fetch(2);
  wait(0);
  float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int d = 0; d < D; ++d) copy(d, idxbuf[w][0][4 * d + e]);
  const long nchunks = steps * 4 / 32;
  for (long ch = 0; ch < nchunks; ++ch) {
    const int b = (int)(ch % 3), bn = (int)((ch + 1) % 3);
    if (ch + 1 < nchunks) wait(ch + 1);                // the next chunk's indices (two chunks of lead)
#pragma unroll 1
    for (int u0 = 0; u0 < 8; u0 += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int u = u0 + d;
        asm volatile("cp.async.wait_group %0;" :: "n"(D - 1) : "memory");
        const float4 a = my[d * 64], bb = my[d * 64 + 8];
        part[0] = fmaf(1.0f, a.x, part[0]); part[1] = fmaf(1.0f, a.y, part[1]);
        part[2] = fmaf(1.0f, a.z, part[2]); part[3] = fmaf(1.0f, a.w, part[3]);
        part[4] = fmaf(1.0f, bb.x, part[4]); part[5] = fmaf(1.0f, bb.y, part[5]);
        part[6] = fmaf(1.0f, bb.z, part[6]); part[7] = fmaf(1.0f, bb.w, part[7]);
        const int tn = u + D;
        const int cn = tn < 8 ? idxbuf[w][b][4 * tn + e] : idxbuf[w][bn][(4 * tn + e) & 31];
        copy(d, cn);
      }
    }
    __syncwarp();
    if (ch + 3 < nchunks) fetch(ch + 3);               // buffer b is free again
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += part[i];
  if (acc == 1234.5f) *sink = acc;
}

int main() {
  int nsm = 148, dev = 0, sm_clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&sm_clk, cudaDevAttrClockRate, dev));
  const size_t maxbytes = (size_t)1 << 30;
  float4* buf;
  float* sink;
  CK(cudaMalloc(&buf, maxbytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 0, maxbytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_best = [&](auto launch, int reps) {
    float best = 1e30f;
    launch();                                             // warm
    for (int i = 0; i < reps; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const size_t foot[] = {32u << 20, 48u << 20, 60u << 20, 64u << 20, 80u << 20, 96u << 20, 112u << 20,
                         128u << 20, (size_t)1 << 30};
  for (size_t X : foot) {
    const size_t n4 = X / 16;
    const int reps = (int)(((size_t)8 << 30) / X) > 0 ? (int)(((size_t)8 << 30) / X) : 1;
    const int grid = nsm * 4;
    const float ms = time_best([&] { stream_read<<<grid, 512>>>(buf, n4, reps, sink); }, 5);
    printf("{\"probe\":\"stream\",\"footprint_MB\":%.0f,\"GBps\":%.1f,\"sm_clock_attr_khz\":%d}\n",
           X / 1048576.0, (double)X * reps / ms / 1e6, sm_clk);
  }
  for (size_t X : {(size_t)60 << 20, (size_t)96 << 20}) {
    const uint32_t nrows = (uint32_t)(X / 256);
    const long steps = 4096;
    for (int wps : {16, 32, 48}) {                        // resident warps per SM
      const int threads = 256;
      const int grid = nsm * wps / 8;
      const double bytes = (double)grid * 8 * steps * 4 * 256;
      float ms = time_best([&] { gather_ldg<4><<<grid, threads>>>(buf, nrows, steps, sink); }, 3);
      printf("{\"probe\":\"gather_ldg\",\"row_B\":256,\"footprint_MB\":%.0f,\"warps_per_sm\":%d,\"rows_in_flight_per_warp\":16,\"GBps\":%.1f}\n",
             X / 1048576.0, wps, bytes / ms / 1e6);
      const size_t smem = (size_t)8 * 4 * 64 * 16;
      ms = time_best([&] { gather_smem<4><<<grid, threads, smem>>>(buf, nrows, steps, sink); }, 3);
      printf("{\"probe\":\"gather_smem\",\"row_B\":256,\"footprint_MB\":%.0f,\"warps_per_sm\":%d,\"ring_depth\":4,\"GBps\":%.1f}\n",
             X / 1048576.0, wps, bytes / ms / 1e6);
    }
  }
  {  // the slab kernel's inner loop as a probe: 60 MB slab, endless rows, index array in HBM
    const uint32_t nrows = (uint32_t)((60u << 20) / 256);
    const long steps = 4096;
    const int threads = 128;                             // 4-warp CTAs as es::spmm_slab
    for (int wps : {24, 32}) {
      const int grid = nsm * wps / 4;
      const long nidx = (long)grid * 4 * steps * 4;
      int* idx;
      CK(cudaMalloc(&idx, (nidx + 64) * sizeof(int)));
      std::vector<int> h(nidx + 64);
      uint64_t x = 0x9E3779B97F4A7C15ull;
      for (long i = 0; i < nidx + 64; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x % nrows); }
      CK(cudaMemcpy(idx, h.data(), (nidx + 64) * sizeof(int), cudaMemcpyHostToDevice));
      const double bytes = (double)grid * 4 * steps * 4 * 256;
      const size_t smem = (size_t)4 * 4 * 64 * 16;
      float ms = time_best([&] { gather_smem_fma<4, 0><<<grid, threads, smem>>>(buf, idx, steps, sink); }, 3);
      printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"index loads + shuffles + FMA\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      ms = time_best([&] { gather_smem_fma<4, 1><<<grid, threads, smem>>>(buf, idx, steps, sink); }, 3);
      printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"index loads + shuffles, no FMA\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      ms = time_best([&] { gather_smem_fma<4, 2><<<grid, threads, smem>>>(buf, idx, steps, sink); }, 3);
      printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"hashed rows + FMA\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      ms = time_best([&] { gather_smem_fma<4, 4><<<grid, threads, smem>>>(buf, idx, steps, sink); }, 3);
      printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"index loads L1::no_allocate + L2 evict_first hint + FMA\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      {
        using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        CUtensorMap tm;
        const cuuint64_t dims[1] = {(cuuint64_t)(nidx + 64)};
        const cuuint64_t strides[1] = {4};
        const cuuint32_t box[1] = {32};
        const cuuint32_t es[1] = {1};
        ((Encode)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_INT32, 1, idx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        ms = time_best([&] { gather_smem_tmaidx<4><<<grid, threads, smem>>>(tm, buf, steps, sink); }, 3);
        printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"index chunks by TMA (1-D tensor map) into smem\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      }
      ms = time_best([&] { gather_smem_fma<4, 3><<<grid, threads, smem>>>(buf, idx, steps, sink); }, 3);
      printf("{\"probe\":\"slab_inner_loop\",\"mode\":\"index loads + FMA, zero-fill cp.async form\",\"warps_per_sm\":%d,\"GBps\":%.1f}\n", wps, bytes / ms / 1e6);
      cudaFree(idx);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
