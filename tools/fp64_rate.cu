// fp64_rate.cu -- measure DADD/DMUL/DFMA throughput per SM (scratch tool).
#include <cstdio>
__global__ void k(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kl(double* out, int iters, double a) {  // latency: one dependent chain per thread
  double x0 = threadIdx.x;
  for (int i = 0; i < iters; ++i) x0 = __dadd_rn(x0, a);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 1024 * 8 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 20000;
  k<<<148 * 4, 512>>>(o, 100, 1.0, 2.0);
  cudaEventRecord(a); k<<<148 * 4, 512>>>(o, iters, 1.0, 2.0); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 148.0 * 4 * 512 * iters * 8;
  printf("DADD throughput: %.1f Gop/s = %.1f lane-ops/clk/SM at 1.965 GHz\n", ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaEventRecord(a); kl<<<1, 32>>>(o, iters, 1.0); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("DADD dependent latency: %.1f cycles\n", ms * 1e-3 * 1.965e9 / iters);
  return 0;
}
