// crossover_nvls.cu -- the collective-fused update through NVSwitch multicast (NVLS).
//
// Same job as the P2P kernel (crossover_p2p.cu: reduce-scatter + K2 + all-gather in one kernel),
// but the reduction and the broadcast happen in the switch:
//   acc      = multimem.ld_reduce.add(mc_bucket + shard)   -- the switch reads this shard from
//              every rank's bucket and returns the fp32 sum (one 16-byte load per 4 elements)
//   p        = SGD(p, acc / W)                            -- same sgd_elem as K2
//   multimem.st(mc_param + shard, p)                       -- the switch writes it into every
//              rank's flat parameters
// so each rank reads S/W and writes S/W through its NVLink ports and moves no peer copy itself.
// The switch's summation order is unspecified: results match the rank-order transports within
// fp32 rounding, not bit for bit (tests state the tolerance).
//
// The memory is multicast-bound physical memory (cuMemCreate + cuMulticastBindMem); the driver
// entry points are resolved at run time (cudaGetDriverEntryPointByVersion), so the library loads
// without a driver.  The multicast object travels between processes as a POSIX file descriptor
// (the Python side passes it over a UNIX socket).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "crossover.h"
#include "crossover_internal.h"
#include "crossover_sgd.cuh"

namespace cs {
namespace {

typedef CUresult (*PFN_mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                                  size_t, size_t, unsigned long long);
typedef CUresult (*PFN_mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
typedef CUresult (*PFN_mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
typedef CUresult (*PFN_memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                                  unsigned long long);
typedef CUresult (*PFN_memRelease)(CUmemGenericAllocationHandle);
typedef CUresult (*PFN_memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                  unsigned long long);
typedef CUresult (*PFN_memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
typedef CUresult (*PFN_addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_addrFree)(CUdeviceptr, size_t);
typedef CUresult (*PFN_memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_memUnmap)(CUdeviceptr, size_t);
typedef CUresult (*PFN_memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_devAttr)(int*, CUdevice_attribute, CUdevice);

struct Api {
  PFN_mcCreate mc_create = nullptr;
  PFN_mcAddDevice mc_add = nullptr;
  PFN_mcBindMem mc_bind = nullptr;
  PFN_mcUnbind mc_unbind = nullptr;
  PFN_mcGranularity mc_gran = nullptr;
  PFN_memCreate mem_create = nullptr;
  PFN_memRelease mem_release = nullptr;
  PFN_memExport mem_export = nullptr;
  PFN_memImport mem_import = nullptr;
  PFN_addrReserve addr_reserve = nullptr;
  PFN_addrFree addr_free = nullptr;
  PFN_memMap mem_map = nullptr;
  PFN_memUnmap mem_unmap = nullptr;
  PFN_memSetAccess mem_access = nullptr;
  PFN_devAttr dev_attr = nullptr;
  int status = (int)cudaErrorNotSupported;
};
Api g_api;
std::once_flag g_api_once;

template <class T>
bool resolve(T& f, const char* name) {
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, (void**)&f, 12090, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    f = nullptr;
  return f != nullptr;
}

void load_api() {
  Api& a = g_api;
  bool ok = resolve(a.mc_create, "cuMulticastCreate") & resolve(a.mc_add, "cuMulticastAddDevice") &
            resolve(a.mc_bind, "cuMulticastBindMem") & resolve(a.mc_unbind, "cuMulticastUnbind") &
            resolve(a.mc_gran, "cuMulticastGetGranularity") & resolve(a.mem_create, "cuMemCreate") &
            resolve(a.mem_release, "cuMemRelease") & resolve(a.mem_export, "cuMemExportToShareableHandle") &
            resolve(a.mem_import, "cuMemImportFromShareableHandle") &
            resolve(a.addr_reserve, "cuMemAddressReserve") & resolve(a.addr_free, "cuMemAddressFree") &
            resolve(a.mem_map, "cuMemMap") & resolve(a.mem_unmap, "cuMemUnmap") &
            resolve(a.mem_access, "cuMemSetAccess") & resolve(a.dev_attr, "cuDeviceGetAttribute");
  a.status = ok ? 0 : (int)cudaErrorNotSupported;
  cudaGetLastError();
}

int api_ready(const char* who) {
  std::call_once(g_api_once, load_api);
  if (g_api.status) return set_error(g_api.status, "%s: driver multicast entry points unavailable", who);
  return 0;
}

int cu_status(CUresult r, const char* where) {
  if (r == CUDA_SUCCESS) return 0;
  return set_error((int)r, "%s failed (CUresult %d)", where, (int)r);
}

CUmemAccessDesc rw_access(int device) {
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = device;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return ad;
}

// ---------------------------------------------------------------------------------------------
// the fused kernel: U float4 per thread, all ld_reduce's in flight before the first update
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ float4 mc_ld_reduce(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

constexpr int kNvlsUnroll = 4;
constexpr int kNvlsChunk = kThreads * 4 * kNvlsUnroll;

template <bool kMom>
__global__ void __launch_bounds__(kThreads)
nvls_reduce_sgd_bcast_kernel(const __grid_constant__ cs_nvls_desc d, const __grid_constant__ cs_sgd_hyper h) {
  const Rule r = make_rule(h, kMom);
  const int64_t nvec = d.numel >> 2;                     // host checked: numel % 4 == 0
  const int64_t chunks = (d.numel + kNvlsChunk - 1) / kNvlsChunk;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    const int64_t v0 = c * (kNvlsChunk / 4);
    float4 acc[kNvlsUnroll], pv[kNvlsUnroll], mv[kNvlsUnroll];
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u) {
      const int64_t v = v0 + u * kThreads + threadIdx.x;
      acc[u] = pv[u] = mv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (v < nvec) {
        acc[u] = mc_ld_reduce(d.mc_bucket + 4 * v);
        pv[u] = *(const float4*)(d.param + 4 * v);
        if (kMom) mv[u] = *(const float4*)(d.momentum_buf + 4 * v);
      }
    }
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u) {
      const int64_t v = v0 + u * kThreads + threadIdx.x;
      if (v < nvec) {
        float4 o;
        o.x = sgd_elem(r, acc[u].x, pv[u].x, &mv[u].x);
        o.y = sgd_elem(r, acc[u].y, pv[u].y, &mv[u].y);
        o.z = sgd_elem(r, acc[u].z, pv[u].z, &mv[u].z);
        o.w = sgd_elem(r, acc[u].w, pv[u].w, &mv[u].w);
        if (kMom) *(float4*)(d.momentum_buf + 4 * v) = mv[u];
        mc_st(d.mc_param + 4 * v, o);                    // every rank's copy, through the switch
      }
    }
  }
  __threadfence_system();
}

}  // namespace
}  // namespace cs

using namespace cs;

extern "C" {

int cs_nvls_supported(int device) {
  if (api_ready("cs_nvls_supported")) return 0;
  int v = 0;
  if (g_api.dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, device) != CUDA_SUCCESS) return 0;
  return v ? 1 : 0;
}

int cs_nvls_granularity(int nranks, size_t bytes, size_t* gran) {
  int rc = api_ready("cs_nvls_granularity");
  if (rc) return rc;
  if (nranks < 1 || gran == nullptr) return set_error(CS_ERR_ARG, "cs_nvls_granularity: invalid arguments");
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)nranks;
  mp.size = bytes ? bytes : 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return cu_status(g_api.mc_gran(gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
}

int cs_nvls_create(int nranks, size_t bytes, uint64_t* mc, int* fd) {
  int rc = api_ready("cs_nvls_create");
  if (rc) return rc;
  if (nranks < 1 || bytes == 0 || mc == nullptr || fd == nullptr)
    return set_error(CS_ERR_ARG, "cs_nvls_create: invalid arguments");
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)nranks;
  mp.size = bytes;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h;
  rc = cu_status(g_api.mc_create(&h, &mp), "cuMulticastCreate");
  if (rc) return rc;
  int f = -1;
  rc = cu_status(g_api.mem_export(&f, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                 "cuMemExportToShareableHandle");
  if (rc) {
    g_api.mem_release(h);
    return rc;
  }
  *mc = (uint64_t)h;
  *fd = f;
  return 0;
}

int cs_nvls_import(int fd, uint64_t* mc) {
  int rc = api_ready("cs_nvls_import");
  if (rc) return rc;
  if (fd < 0 || mc == nullptr) return set_error(CS_ERR_ARG, "cs_nvls_import: invalid arguments");
  CUmemGenericAllocationHandle h;
  rc = cu_status(g_api.mem_import(&h, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 "cuMemImportFromShareableHandle");
  if (rc) return rc;
  *mc = (uint64_t)h;
  return 0;
}

int cs_nvls_add_device(uint64_t mc, int device) {
  int rc = api_ready("cs_nvls_add_device");
  if (rc) return rc;
  return cu_status(g_api.mc_add((CUmemGenericAllocationHandle)mc, device), "cuMulticastAddDevice");
}

int cs_nvls_alloc_bind(uint64_t mc, int device, size_t bytes, size_t gran, uint64_t* phys,
                       void** uc_ptr, void** mc_ptr) {
  int rc = api_ready("cs_nvls_alloc_bind");
  if (rc) return rc;
  if (bytes == 0 || gran == 0 || bytes % gran || phys == nullptr || uc_ptr == nullptr || mc_ptr == nullptr)
    return set_error(CS_ERR_ARG, "cs_nvls_alloc_bind: invalid arguments");
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle h;
  if ((rc = cu_status(g_api.mem_create(&h, bytes, &ap, 0), "cuMemCreate"))) return rc;
  if ((rc = cu_status(g_api.mc_bind((CUmemGenericAllocationHandle)mc, 0, h, 0, bytes, 0),
                      "cuMulticastBindMem"))) {
    g_api.mem_release(h);
    return rc;
  }
  const CUmemAccessDesc ad = rw_access(device);
  CUdeviceptr uc = 0, mcv = 0;
  if ((rc = cu_status(g_api.addr_reserve(&uc, bytes, gran, 0, 0), "cuMemAddressReserve")) ||
      (rc = cu_status(g_api.mem_map(uc, bytes, 0, h, 0), "cuMemMap (unicast)")) ||
      (rc = cu_status(g_api.mem_access(uc, bytes, &ad, 1), "cuMemSetAccess (unicast)")) ||
      (rc = cu_status(g_api.addr_reserve(&mcv, bytes, gran, 0, 0), "cuMemAddressReserve")) ||
      (rc = cu_status(g_api.mem_map(mcv, bytes, 0, (CUmemGenericAllocationHandle)mc, 0), "cuMemMap (multicast)")) ||
      (rc = cu_status(g_api.mem_access(mcv, bytes, &ad, 1), "cuMemSetAccess (multicast)")))
    return rc;
  cudaMemset((void*)uc, 0, bytes);
  *phys = (uint64_t)h;
  *uc_ptr = (void*)uc;
  *mc_ptr = (void*)mcv;
  return cuda_status(cudaDeviceSynchronize(), "cs_nvls_alloc_bind zero-fill");
}

int cs_nvls_free(uint64_t mc, int device, uint64_t phys, void* uc_ptr, void* mc_ptr, size_t bytes) {
  int rc = api_ready("cs_nvls_free");
  if (rc) return rc;
  if (mc_ptr) {
    g_api.mem_unmap((CUdeviceptr)mc_ptr, bytes);
    g_api.addr_free((CUdeviceptr)mc_ptr, bytes);
  }
  if (uc_ptr) {
    g_api.mem_unmap((CUdeviceptr)uc_ptr, bytes);
    g_api.addr_free((CUdeviceptr)uc_ptr, bytes);
  }
  if (mc && phys) g_api.mc_unbind((CUmemGenericAllocationHandle)mc, device, 0, bytes);
  if (phys) g_api.mem_release((CUmemGenericAllocationHandle)phys);
  return 0;
}

int cs_nvls_release(uint64_t mc) {
  int rc = api_ready("cs_nvls_release");
  if (rc) return rc;
  return mc ? cu_status(g_api.mem_release((CUmemGenericAllocationHandle)mc), "cuMemRelease (multicast)") : 0;
}

int cs_nvls_reduce_sgd_bcast(const cs_nvls_desc* d, const cs_sgd_hyper* h, void* stream) {
  if (d == nullptr || h == nullptr) return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: NULL argument");
  if (d->numel < 0 || d->numel % 4 || (d->numel > 0 && (!d->mc_bucket || !d->mc_param || !d->param)))
    return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: bad shard (numel must be a multiple of 4)");
  if (h->divisor != d->nranks || d->nranks < 1)
    return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: divisor %d != nranks %d", h->divisor, d->nranks);
  if (!(h->lr > 0.0f)) return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: learning rate must be > 0");
  if (h->momentum != 0.0f && d->momentum_buf == nullptr)
    return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: momentum buffer is NULL");
  if (((uintptr_t)d->mc_bucket | (uintptr_t)d->mc_param | (uintptr_t)d->param |
       (uintptr_t)d->momentum_buf) & 15u)
    return set_error(CS_ERR_ARG, "cs_nvls_reduce_sgd_bcast: shards must be 16-byte aligned");
  if (d->numel == 0) return 0;
  int64_t grid = (d->numel + kNvlsChunk - 1) / kNvlsChunk;
  int cap = d->max_ctas;
  if (cap <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = 2 * sms;
  }
  if (grid > cap) grid = cap;
  cudaStream_t s = (cudaStream_t)stream;
  if (h->momentum != 0.0f) nvls_reduce_sgd_bcast_kernel<true><<<(unsigned)grid, kThreads, 0, s>>>(*d, *h);
  else nvls_reduce_sgd_bcast_kernel<false><<<(unsigned)grid, kThreads, 0, s>>>(*d, *h);
  return cuda_status(cudaGetLastError(), "cs_nvls_reduce_sgd_bcast launch");
}

}  // extern "C"
