// kv_pool.cu -- paged KV store behind lfps_state.k_cache / v_cache
// (include/lfps_b200.h, lfps_kv_pool_*).
//
// One virtual reservation per cache of B * Hkv spans of n_max rows; each
// span is backed by physical pages (the device's minimum allocation
// granularity) mapped in order as its context grows and unmapped when the
// request is released.  The decode kernels keep addressing the contiguous
// [B, Hkv, n_max, d] layout -- the page table is the GPU's own MMU -- so
// the hot path is unchanged.  The driver's virtual-memory API is resolved
// at run time through cudaGetDriverEntryPoint (no link-time libcuda
// dependency: the library still loads on a machine without a driver).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "../../include/lfps_b200.h"

int lfps_abi_fail(int code, const char* msg);
int lfps_check_dims(const lfps_dims* d);

namespace {

constexpr int64_t kSlackRows = 64;      // one row tile past the last row

struct Driver {
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*free_va)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                     unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                  unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  bool ok = false;
};

std::mutex g_drv_mu;
Driver g_drv;

template <typename F>
bool entry(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver* driver() {
  std::lock_guard<std::mutex> g(g_drv_mu);
  if (!g_drv.ok) {
    Driver d;
    if (entry("cuMemAddressReserve", &d.reserve) && entry("cuMemAddressFree", &d.free_va) &&
        entry("cuMemCreate", &d.create) && entry("cuMemRelease", &d.release) &&
        entry("cuMemMap", &d.map) && entry("cuMemUnmap", &d.unmap) &&
        entry("cuMemSetAccess", &d.access) &&
        entry("cuMemGetAllocationGranularity", &d.gran)) {
      d.ok = true;
      g_drv = d;
    }
  }
  return g_drv.ok ? &g_drv : nullptr;
}

CUmemAllocationProp prop_for(int dev) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = dev;
  return p;
}

int page_bytes_for(const Driver* d, int dev, size_t* out) {
  const CUmemAllocationProp p = prop_for(dev);
  if (d->gran(out, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || *out == 0)
    return lfps_abi_fail(LFPS_E_CUDA, "cuMemGetAllocationGranularity failed");
  return LFPS_OK;
}

int no_driver() {
  return lfps_abi_fail(LFPS_E_UNSUPPORTED, "CUDA driver virtual-memory API unavailable (no GPU?)");
}

}  // namespace

struct lfps_kv_pool {
  int dev = 0;
  int B = 0, Hkv = 0, d = 0;
  int64_t n_max = 0;
  size_t page = 0, span = 0, total = 0;
  CUdeviceptr base[2] = {0, 0};                           // K, V
  std::vector<std::vector<CUmemGenericAllocationHandle>> pages[2];   // per (b, h)
  int64_t mapped = 0;
  std::mutex mu;
  cudaStream_t zero = nullptr;     // zeroes fresh pages (created on first growth)
};

namespace {

// the pool's device current for the scope of a call (callers may sit on
// another device); restores the caller's device
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int unmap_span(const Driver* drv, lfps_kv_pool* p, size_t u) {
  int rc = LFPS_OK;
  for (int t = 0; t < 2; ++t) {
    std::vector<CUmemGenericAllocationHandle>& v = p->pages[t][u];
    for (size_t i = 0; i < v.size(); ++i) {
      const CUdeviceptr at = p->base[t] + u * p->span + i * p->page;
      if (drv->unmap(at, p->page) != CUDA_SUCCESS || drv->release(v[i]) != CUDA_SUCCESS)
        rc = lfps_abi_fail(LFPS_E_CUDA, "cuMemUnmap / cuMemRelease failed");
      p->mapped -= (int64_t)p->page;
    }
    v.clear();
  }
  return rc;
}

}  // namespace

extern "C" {

int64_t lfps_kv_pool_page_bytes(void) {
  const Driver* drv = driver();
  if (!drv) return no_driver();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return lfps_abi_fail(LFPS_E_CUDA, "cudaGetDevice failed");
  size_t g = 0;
  const int rc = page_bytes_for(drv, dev, &g);
  return rc ? rc : (int64_t)g;
}

int lfps_kv_pool_create(const lfps_dims* dims, lfps_kv_pool** pool, void** k_cache,
                        void** v_cache) {
  int rc = lfps_check_dims(dims);
  if (rc) return rc;
  if (!pool || !k_cache || !v_cache) return lfps_abi_fail(LFPS_E_INVALID, "NULL output pointer");
  const Driver* drv = driver();
  if (!drv) return no_driver();
  lfps_kv_pool* p = new lfps_kv_pool;
  if (cudaGetDevice(&p->dev) != cudaSuccess) {
    delete p;
    return lfps_abi_fail(LFPS_E_CUDA, "cudaGetDevice failed");
  }
  if ((rc = page_bytes_for(drv, p->dev, &p->page))) {
    delete p;
    return rc;
  }
  p->B = dims->batch; p->Hkv = dims->kv_heads; p->d = dims->d; p->n_max = dims->n_max;
  p->span = (size_t)dims->n_max * dims->d * 2;
  if (p->span % p->page != 0) {
    delete p;
    return lfps_abi_fail(LFPS_E_INVALID,
                         "n_max * d * 2 must be a multiple of lfps_kv_pool_page_bytes()");
  }
  const size_t units = (size_t)p->B * p->Hkv;
  p->total = units * p->span;
  for (int t = 0; t < 2; ++t) {
    if (drv->reserve(&p->base[t], p->total, p->page, 0, 0) != CUDA_SUCCESS) {
      if (t) drv->free_va(p->base[0], p->total);
      delete p;
      return lfps_abi_fail(LFPS_E_CUDA, "cuMemAddressReserve failed");
    }
    p->pages[t].resize(units);
  }
  *pool = p;
  *k_cache = reinterpret_cast<void*>(p->base[0]);
  *v_cache = reinterpret_cast<void*>(p->base[1]);
  return LFPS_OK;
}

int lfps_kv_pool_reserve(lfps_kv_pool* p, int32_t b, int32_t h, int64_t rows) {
  if (!p) return lfps_abi_fail(LFPS_E_INVALID, "pool is NULL");
  if (b < 0 || b >= p->B || h < 0 || h >= p->Hkv || rows < 0 || rows > p->n_max)
    return lfps_abi_fail(LFPS_E_INVALID, "reserve: (b, h, rows) out of range");
  const Driver* drv = driver();
  if (!drv) return no_driver();
  std::lock_guard<std::mutex> g(p->mu);
  DeviceScope scope(p->dev);
  const size_t u = (size_t)b * p->Hkv + h;
  const int64_t want_rows = rows + kSlackRows < p->n_max ? rows + kSlackRows : p->n_max;
  const size_t want = ((size_t)want_rows * p->d * 2 + p->page - 1) / p->page;
  const CUmemAllocationProp prop = prop_for(p->dev);
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = p->dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  bool grew = false;
  for (int t = 0; t < 2; ++t) {
    std::vector<CUmemGenericAllocationHandle>& v = p->pages[t][u];
    while (v.size() < want) {
      CUmemGenericAllocationHandle hdl;
      if (drv->create(&hdl, p->page, &prop, 0) != CUDA_SUCCESS)
        return lfps_abi_fail(LFPS_E_CUDA, "cuMemCreate failed (device memory exhausted?)");
      const CUdeviceptr at = p->base[t] + u * p->span + v.size() * p->page;
      if (drv->map(at, p->page, 0, hdl, 0) != CUDA_SUCCESS) {
        drv->release(hdl);
        return lfps_abi_fail(LFPS_E_CUDA, "cuMemMap failed");
      }
      if (drv->access(at, p->page, &acc, 1) != CUDA_SUCCESS) {
        drv->unmap(at, p->page);
        drv->release(hdl);
        return lfps_abi_fail(LFPS_E_CUDA, "cuMemSetAccess failed");
      }
      v.push_back(hdl);
      p->mapped += (int64_t)p->page;
      // fresh pages hold whatever the memory held: zero them, as the
      // contiguous cache is, so that padding rows a kernel touches past the
      // context (weight 0) are finite -- on the pool's own stream, so the
      // wait below does not drain the device
      if (!p->zero && cudaStreamCreateWithFlags(&p->zero, cudaStreamNonBlocking) != cudaSuccess)
        return lfps_abi_fail(LFPS_E_CUDA, "cudaStreamCreate failed");
      if (cudaMemsetAsync(reinterpret_cast<void*>(at), 0, p->page, p->zero) != cudaSuccess)
        return lfps_abi_fail(LFPS_E_CUDA, "cudaMemsetAsync failed");
      grew = true;
    }
  }
  if (grew && cudaStreamSynchronize(p->zero) != cudaSuccess)
    return lfps_abi_fail(LFPS_E_CUDA, "cudaStreamSynchronize failed");
  return LFPS_OK;
}

int lfps_kv_pool_release(lfps_kv_pool* p, int32_t b) {
  if (!p) return lfps_abi_fail(LFPS_E_INVALID, "pool is NULL");
  if (b < 0 || b >= p->B) return lfps_abi_fail(LFPS_E_INVALID, "release: request out of range");
  const Driver* drv = driver();
  if (!drv) return no_driver();
  DeviceScope scope(p->dev);
  // the caller's queued work on the pool's device may still read these rows
  if (cudaDeviceSynchronize() != cudaSuccess)
    return lfps_abi_fail(LFPS_E_CUDA, "cudaDeviceSynchronize failed");
  std::lock_guard<std::mutex> g(p->mu);
  int rc = LFPS_OK;
  for (int h = 0; h < p->Hkv; ++h) {
    const int r = unmap_span(drv, p, (size_t)b * p->Hkv + h);
    if (r) rc = r;
  }
  return rc;
}

int64_t lfps_kv_pool_mapped_bytes(const lfps_kv_pool* p) {
  if (!p) return lfps_abi_fail(LFPS_E_INVALID, "pool is NULL");
  return p->mapped;
}

int lfps_kv_pool_destroy(lfps_kv_pool* p) {
  if (!p) return LFPS_OK;
  const Driver* drv = driver();
  if (!drv) return no_driver();
  DeviceScope scope(p->dev);
  if (cudaDeviceSynchronize() != cudaSuccess)
    return lfps_abi_fail(LFPS_E_CUDA, "cudaDeviceSynchronize failed");
  if (p->zero) cudaStreamDestroy(p->zero);
  int rc = LFPS_OK;
  {
    std::lock_guard<std::mutex> g(p->mu);
    for (size_t u = 0; u < (size_t)p->B * p->Hkv; ++u) {
      const int r = unmap_span(drv, p, u);
      if (r) rc = r;
    }
    for (int t = 0; t < 2; ++t)
      if (drv->free_va(p->base[t], p->total) != CUDA_SUCCESS)
        rc = lfps_abi_fail(LFPS_E_CUDA, "cuMemAddressFree failed");
  }
  delete p;
  return rc;
}

}  // extern "C"
