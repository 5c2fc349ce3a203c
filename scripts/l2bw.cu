// L2 / DRAM read-bandwidth probe (tuning evidence only, not part of the library).
// What bounds a B-row gather once B (or a feature slice of it) is L2-resident?
//   stream: every thread reads float4 in a grid-stride loop over a footprint of X bytes, R times
//   gather: one warp per gather of a W-byte row picked by a random index, footprint X bytes
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2bw scripts/l2bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void stream_read(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  size_t stride = (size_t)gridDim.x * blockDim.x;
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

// Each warp performs gathers g = warp, warp + nwarps, ...; row = idx[g]; lanes cover W bytes.
template <int U>
__global__ void gather_read(const float4* __restrict__ B, int ld4, int w4, const int* __restrict__ idx,
                            long ngather, float* sink) {
  int lane = threadIdx.x & 31;
  long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long g = warp * U; g < ngather; g += nw * U) {
    int rows[U];
#pragma unroll
    for (int u = 0; u < U; ++u) rows[u] = (g + u < ngather) ? __ldg(idx + g + u) : 0;
    for (int c = lane; c < w4; c += 32) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(B + (size_t)rows[u] * ld4 + c);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
    }
  }
  if (acc == 1234.5f) *sink = acc;
}

int main(int argc, char** argv) {
  int nsm = 148;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  size_t maxbytes = (size_t)4 << 30;
  float4* buf; float* sink;
  CK(cudaMalloc(&buf, maxbytes)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 0, maxbytes));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t foot[] = {8u << 20, 16u << 20, 32u << 20, 48u << 20, 64u << 20, 80u << 20, 96u << 20,
                   112u << 20, 128u << 20, 192u << 20, (size_t)1 << 30, (size_t)4 << 30};
  // stream
  for (size_t X : foot) {
    size_t n4 = X / 16;
    int reps = (int)(((size_t)16 << 30) / X); if (reps < 1) reps = 1;
    for (int bpsm : {4}) {
      int grid = nsm * bpsm;
      stream_read<<<grid, 512>>>(buf, n4, 1, sink);
      CK(cudaEventRecord(e0));
      stream_read<<<grid, 512>>>(buf, n4, reps, sink);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\":\"stream\",\"footprint_MB\":%.0f,\"GBps\":%.1f}\n", X / 1048576.0,
             (double)X * reps / ms / 1e6);
    }
  }
  // gather
  long ng = 40000000;
  int* idx; CK(cudaMalloc(&idx, ng * 4));
  std::vector<int> h(ng);
  for (int W : {128, 256, 512, 1024, 2432}) {
    for (size_t X : foot) {
      long nrows = (long)(X / W);
      if (nrows < 64) continue;
      if ((long)W * nrows > (long)maxbytes) continue;
      uint64_t s = 0x9E3779B97F4A7C15ull ^ W ^ X;
      for (long g = 0; g < ng; ++g) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[g] = (int)(s % nrows); }
      CK(cudaMemcpy(idx, h.data(), ng * 4, cudaMemcpyHostToDevice));
      long ngx = ng;
      if ((double)ngx * W > 60e9) ngx = (long)(60e9 / W);
      int grid = nsm * 4;
      gather_read<4><<<grid, 512>>>(buf, W / 16, W / 16, idx, ngx / 8, sink);
      CK(cudaEventRecord(e0));
      gather_read<4><<<grid, 512>>>(buf, W / 16, W / 16, idx, ngx, sink);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\":\"gather\",\"row_B\":%d,\"footprint_MB\":%.0f,\"GBps\":%.1f}\n", W,
             X / 1048576.0, (double)ngx * W / ms / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
