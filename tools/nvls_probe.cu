// nvls_probe.cu -- does NVSwitch multicast (NVLS) work on this box?  One process, two GPUs:
// a multicast object over both devices, one physical buffer bound per device, a kernel on GPU 0
// that multimem.ld_reduce's the sum of both buffers through the switch and multimem.st's a value
// into both.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o nvls_probe tools/nvls_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; \
  p_cuGetErrorString(r_, &s_); printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?"); return 1; } } while (0)

#define FN(name) static PFN_##name p_##name = nullptr;
typedef CUresult (*PFN_cuGetErrorString)(CUresult, const char**);
typedef CUresult (*PFN_cuMulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_cuMulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_cuMulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
typedef CUresult (*PFN_cuMulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
typedef CUresult (*PFN_cuMemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PFN_cuMemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_cuMemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_cuMemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_cuDeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
FN(cuGetErrorString) FN(cuMulticastCreate) FN(cuMulticastAddDevice) FN(cuMulticastBindMem)
FN(cuMulticastGetGranularity) FN(cuMemCreate) FN(cuMemAddressReserve) FN(cuMemMap) FN(cuMemSetAccess)
FN(cuDeviceGetAttribute)

template <class T> static void load(T& f, const char* name) {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion(name, (void**)&f, 12090, cudaEnableDefault, &q);
  if (!f) { printf("no entry point %s\n", name); exit(2); }
}

__global__ void probe(float* mc, float* out) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
  out[0] = v.x; out[1] = v.w;
  float4 w = make_float4(7.f, 7.f, 7.f, 7.f);
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(mc + 4), "f"(w.x), "f"(w.y), "f"(w.z), "f"(w.w) : "memory");
}

int main() {
  cudaFree(0);
  load(p_cuGetErrorString, "cuGetErrorString"); load(p_cuMulticastCreate, "cuMulticastCreate");
  load(p_cuMulticastAddDevice, "cuMulticastAddDevice"); load(p_cuMulticastBindMem, "cuMulticastBindMem");
  load(p_cuMulticastGetGranularity, "cuMulticastGetGranularity"); load(p_cuMemCreate, "cuMemCreate");
  load(p_cuMemAddressReserve, "cuMemAddressReserve"); load(p_cuMemMap, "cuMemMap");
  load(p_cuMemSetAccess, "cuMemSetAccess"); load(p_cuDeviceGetAttribute, "cuDeviceGetAttribute");
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  for (int d = 0; d < 2; ++d) {
    int mcs = 0;
    CK(p_cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
    printf("device %d multicast supported: %d\n", d, mcs);
  }
  CUmulticastObjectProp mp = {};
  mp.numDevices = 2;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = 2 << 20;
  CK(p_cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t size = ((2 << 20) + gran - 1) / gran * gran;
  mp.size = size;
  printf("granularity %zu size %zu\n", gran, size);
  CUmemGenericAllocationHandle mc;
  CK(p_cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < 2; ++d) CK(p_cuMulticastAddDevice(mc, d));
  CUdeviceptr uc[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle h;
    CK(p_cuMemCreate(&h, size, &ap, 0));
    CK(p_cuMulticastBindMem(mc, 0, h, 0, size, 0));
    CK(p_cuMemAddressReserve(&uc[d], size, gran, 0, 0));
    CK(p_cuMemMap(uc[d], size, 0, h, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(p_cuMemSetAccess(uc[d], size, &ad, 1));
    float host[8];
    for (int i = 0; i < 8; ++i) host[i] = (float)(d + 1);
    cudaMemcpy((void*)uc[d], host, sizeof(host), cudaMemcpyHostToDevice);
  }
  cudaSetDevice(0);
  CUdeviceptr mcva;
  CK(p_cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CK(p_cuMemMap(mcva, size, 0, mc, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(p_cuMemSetAccess(mcva, size, &ad, 1));
  float* out;
  cudaMalloc(&out, 16);
  probe<<<1, 1>>>((float*)mcva, out);
  cudaError_t e = cudaDeviceSynchronize();
  float o[2] = {0, 0};
  cudaMemcpy(o, out, 8, cudaMemcpyDeviceToHost);
  printf("kernel: %s; ld_reduce sum = %g %g (expect 3 3)\n", cudaGetErrorString(e), o[0], o[1]);
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    float h[8];
    cudaMemcpy(h, (void*)uc[d], sizeof(h), cudaMemcpyDeviceToHost);
    printf("device %d buffer after multimem.st: %g %g %g %g | %g %g %g %g (expect 1/2s then 7s)\n", d,
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
