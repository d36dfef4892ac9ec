// scan_bench.cu -- standalone timing of the table-scan kernel variants at the
// C4 table size (2048 sessions x 131200 slots, random phys tables).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//   -Ipaper_2506_15704_b200/csrc tools/scan_bench.cu paper_2506_15704_b200/csrc/k_scan.cu -o tools/scan_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"

using namespace lfps;

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffff) * 1e-6;
  }
}

int main(int argc, char** argv) {
  const int NS = argc > 1 ? atoi(argv[1]) : 2048;
  const int m = argc > 2 ? atoi(argv[2]) : 131200;
  Ctx c = {};
  c.B = NS / 32; c.Hkv = 8; c.G = 4; c.Hq = 32; c.NS = NS; c.S = 4; c.d = 128;
  c.m_cap = m + 64; c.ring_cap = c.m_cap + 2; c.a = 0.2;
  c.words = (c.m_cap + 11776 + 31) / 32;
  size_t nt = (size_t)NS * c.m_cap, nr = (size_t)NS * c.ring_cap;
  cudaMalloc(&c.ver, nt * 8); cudaMalloc(&c.sla, nr * 8);
  cudaMalloc(&c.scale, NS * 8); cudaMalloc(&c.sla_base, NS * 4);
  cudaMalloc(&c.bypass, NS * 4); cudaMalloc(&c.n_ctx, c.B * 4);
  cudaMalloc(&c.bits, (size_t)NS * 4 * c.words * 4); cudaMalloc(&c.thr, (size_t)NS * 8 * 8);
  cudaMalloc(&c.err, (NS + 1) * 4);
  cudaMalloc(&c.scratch, 16 * 16 * 12 * 8);
  cudaMemset(c.scratch, 0, 16 * 16 * 12 * 8);
  fill<<<2048, 256>>>(c.ver, nt, 1); fill<<<2048, 256>>>(c.sla, nr, 2);
  std::vector<double> sc(NS, 1.0); cudaMemcpy(c.scale, sc.data(), NS * 8, cudaMemcpyHostToDevice);
  std::vector<int> base(NS); for (int i = 0; i < NS; ++i) base[i] = (i * 7919) % c.ring_cap;
  cudaMemcpy(c.sla_base, base.data(), NS * 4, cudaMemcpyHostToDevice);
  cudaMemset(c.bypass, 0, NS * 4); cudaMemset(c.err, 0, (NS + 1) * 4);
  std::vector<int> n(c.B, m + 4); cudaMemcpy(c.n_ctx, n.data(), c.B * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)NS * 2 * 8 * m;
  int slices[] = {0, 12288, 4096};
  for (int mode = 0; mode < 1; ++mode) {
    for (int si = 0; si < 3; ++si) {
      cudaError_t e = launch_scan_experiment(c, m, mode, slices[si], 0);
      if (e != cudaSuccess) { printf("mode %d slice %d: %s\n", mode, slices[si], cudaGetErrorString(e)); cudaGetLastError(); continue; }
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      const int reps = 5;
      for (int r = 0; r < reps; ++r) launch_scan_experiment(c, m, mode, slices[si], 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0; cudaEventElapsedTime(&ms, a, b); ms /= reps;
      e = cudaGetLastError();
      printf("mode %d slice %5d: %.3f ms  %.0f GB/s  %s\n", mode, slices[si], ms, bytes / ms / 1e6,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  // phase trace of cluster 0 (mode 3)
  launch_scan_experiment(c, m, 3, 0, 0);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> tr(16 * 16 * 12);
  cudaMemcpy(tr.data(), c.scratch, tr.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = tr[0];
  for (int r = 0; r < 16; ++r) t0 = (tr[r * 16 * 12] && tr[r * 16 * 12] < t0) ? tr[r * 16 * 12] : t0;
  printf("trace (us): rank item: start stats sent lead_done - - bits_prev - | lead_gathered\n");
  for (int it = 0; it < 6; ++it)
    for (int r = 0; r < 16; r += 5) {
      const unsigned long long* t = &tr[((size_t)r * 16 + it) * 12];
      printf("r%2d i%d:", r, it);
      for (int k = 0; k < 10; ++k) printf(" %7.2f", t[k] ? (t[k] - t0) / 1e3 : -1.0);
      printf("\n");
    }
  return 0;
}
