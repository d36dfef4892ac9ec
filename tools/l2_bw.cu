// l2_bw.cu -- L2-resident read bandwidth vs HBM read bandwidth (scratch tool).
#include <cstdio>
__global__ void rd(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 1234.5) out[0] = acc;
}
int main() {
  size_t big = (size_t)4 << 30;  // 4 GiB
  double2* p; cudaMalloc(&p, big); cudaMemset(p, 0, big);
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)96 << 20, big};
  for (size_t sz : sizes) {
    size_t n = sz / 16;
    int reps = sz >= big ? 2 : (int)(((size_t)8 << 30) / sz);
    rd<<<148 * 8, 256>>>(p, n, 1, o);
    cudaEventRecord(a); rd<<<148 * 8, 256>>>(p, n, reps, o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("working set %6zu MiB: %.0f GB/s\n", sz >> 20, (double)sz * reps / ms / 1e6);
  }
  return 0;
}
