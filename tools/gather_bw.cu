// gather_bw.cu -- HBM throughput of row gathers (the finish kernels' access
// pattern): every warp reads `rows` rows of `row_bytes` bytes at indices drawn
// from a 16 GiB buffer, 16 bytes per lane with plain LDG.128 (kept in flight
// by unrolling), and the achieved GB/s is printed per pattern:
//   seq      consecutive rows (streaming copy)
//   sorted   rows sorted within each unit (the decode workload: ~1000 of 128k
//            rows per (request, KV-head) unit, clustered)
//   random   uniform random rows
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gather_bw.cu -o tools/gather_bw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void gather(const uint4* __restrict__ base, const int* __restrict__ idx, int nidx,
                       int row_u4, unsigned long long* sink) {
  // a warp takes rows; lanes cover row_u4 16-byte chunks of each row (row_u4 <= 32 per pass)
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int rpw = 32 / row_u4;                    // rows per warp instruction
  const int sub = lane / row_u4, ch = lane % row_u4;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int i0 = gw * rpw * 8; i0 < nidx; i0 += nw * rpw * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * rpw + sub;
      v[u] = i < nidx ? __ldcg(base + (size_t)idx[i] * row_u4 + ch) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 16ull << 30;
  uint4* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  std::mt19937_64 rng(1);
  const int units = 2048, per_unit = 1066, unit_rows = 131072;
  for (int row_bytes : {256, 512}) {
    const int row_u4 = row_bytes / 16;
    const long long nrows = (long long)(bytes / row_bytes);
    for (int pat = 0; pat < 3; ++pat) {
      std::vector<int> h;
      h.reserve((size_t)units * per_unit);
      for (int u = 0; u < units; ++u) {
        std::vector<int> r;
        const long long ubase = (long long)u * (nrows / units);
        const long long span = std::min<long long>(unit_rows, nrows / units);
        for (int j = 0; j < per_unit; ++j) {
          long long x;
          if (pat == 0) x = (long long)u * per_unit + j;
          else if (pat == 1) x = ubase + (long long)(rng() % span);
          else x = (long long)(rng() % nrows);
          r.push_back((int)x);
        }
        if (pat == 1) std::sort(r.begin(), r.end());
        h.insert(h.end(), r.begin(), r.end());
      }
      int* d;
      cudaMalloc(&d, h.size() * 4);
      cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      const int n = (int)h.size();
      // row_bytes = 512 with row_u4 = 32: one row per warp instruction
      for (int rep = 0; rep < 2; ++rep) gather<<<148 * 8, 256>>>(buf, d, n, row_u4 > 32 ? 32 : row_u4, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      const int it = 10;
      cudaEventRecord(a);
      for (int rep = 0; rep < it; ++rep) gather<<<148 * 8, 256>>>(buf, d, n, row_u4, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gb = (double)n * row_bytes / 1e9;
      printf("row %3d B  %-6s  rows %d  %.1f us  %.0f GB/s\n", row_bytes, pat == 0 ? "seq" : pat == 1 ? "sorted" : "random",
             n, ms * 1e3 / it, gb / (ms * 1e-3 / it));
      cudaFree(d);
    }
  }
  return 0;
}
