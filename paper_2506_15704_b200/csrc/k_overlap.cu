// k_overlap.cu -- recall eta = |C2 ∩ I_exact| / |I_exact| per session
// (overlap_ratio, attention.py:116-124; the run_trace metric, bench.py:210).
#include "common.cuh"

namespace lfps {

namespace {

__global__ void lfps_overlap_kernel(const int* sel, const int* sel_cnt, const int* ex,
                               const int* ex_cnt, int list_stride, int cnt_stride, double* eta) {
  __shared__ int red[8];
  const int s = blockIdx.x;
  const int ns = sel_cnt[(size_t)s * cnt_stride];
  const int ne = ex_cnt[(size_t)s * cnt_stride];
  const int* a = sel + (size_t)s * list_stride;
  const int* e = ex + (size_t)s * list_stride;
  int hit = 0;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const int v = a[i];
    int lo = 0, hi = ne;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (e[mid] < v) lo = mid + 1; else hi = mid;
    }
    hit += (lo < ne && e[lo] == v);
  }
  for (int o = 16; o >= 1; o >>= 1) hit += __shfl_xor_sync(LFPS_FULL, hit, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = hit;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    eta[s] = ne > 0 ? (double)t / (double)ne : NAN;
  }
}

}  // namespace

cudaError_t launch_overlap(const Ctx& c, const int* sel, const int* sel_cnt, const int* ex,
                           const int* ex_cnt, int list_stride, int cnt_stride, double* eta,
                           cudaStream_t st) {
  lfps_overlap_kernel<<<c.NS, 256, 0, st>>>(sel, sel_cnt, ex, ex_cnt, list_stride, cnt_stride, eta);
  return cudaGetLastError();
}

}  // namespace lfps
