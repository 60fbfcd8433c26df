// nvls_ceiling.cu -- the NVSwitch multicast (NVLS) ceiling on this box: how fast can W GPUs
// multimem.ld_reduce / multimem.st their shards of one multicast-bound buffer, with nothing else
// in the kernel?  The measured peak for the nvls transport's roofline (bench.py, DESIGN §3/§6).
//
// One process drives W GPUs (default: all visible, >= 2).  One multicast object of `mb` MB per
// buffer (bucket, params), one physical allocation per GPU bound to it.  Every GPU runs the same
// kernel at once over its own shard (S/W), timed with events on each device (max over devices):
//   ld_reduce   v = multimem.ld_reduce(bucket shard); store v locally           (the reduce half)
//   st          multimem.st(params shard, local values)                          (the broadcast half)
//   fused       v = multimem.ld_reduce(bucket shard); multimem.st(params shard, v) (both, no update)
// per CTA count in {32, 64, 148, 296}.  Per GPU and link direction the fused pattern moves
// (W + 1) * S / W bytes (the switch reads every member's copy of each shard and delivers every
// rank's stores to every member); the all-reduce bus-bytes convention is 2 (W - 1) / W * S.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o nvls_ceiling tools/nvls_ceiling.cu
// Run:   ./nvls_ceiling [mb=512] [reps=20]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <algorithm>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { printf("FAIL %s -> %d\n", #x, (int)r_); exit(1); } } while (0)
#define CR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(r_)); exit(1); } } while (0)

#define FN(name) static PFN_##name p_##name = nullptr;
typedef CUresult (*PFN_cuMulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_cuMulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_cuMulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t, unsigned long long);
typedef CUresult (*PFN_cuMulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
typedef CUresult (*PFN_cuMemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PFN_cuMemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_cuMemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_cuMemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
FN(cuMulticastCreate) FN(cuMulticastAddDevice) FN(cuMulticastBindMem) FN(cuMulticastGetGranularity)
FN(cuMemCreate) FN(cuMemAddressReserve) FN(cuMemMap) FN(cuMemSetAccess)

template <class T> static void load(T& f, const char* name) {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion(name, (void**)&f, 12090, cudaEnableDefault, &q);
  if (!f) { printf("no entry point %s\n", name); exit(2); }
}

constexpr int kThreads = 256, kUnroll = 4;

__device__ __forceinline__ float4 ld_reduce(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// mode 0 ld_reduce -> local store, 1 local load -> multimem.st, 2 ld_reduce -> multimem.st
__global__ void __launch_bounds__(kThreads) shard_kernel(int mode, const float* mc_bucket, float* mc_param,
                                                         float* local, long long nvec) {
  const long long chunk = (long long)kThreads * kUnroll;
  for (long long c = blockIdx.x; c * chunk < nvec; c += gridDim.x) {
    float4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      long long i = c * chunk + u * kThreads + threadIdx.x;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i < nvec) v[u] = mode == 1 ? ((const float4*)local)[i] : ld_reduce(mc_bucket + 4 * i);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      long long i = c * chunk + u * kThreads + threadIdx.x;
      if (i < nvec) {
        if (mode == 0) ((float4*)local)[i] = v[u];
        else mc_st(mc_param + 4 * i, v[u]);
      }
    }
  }
}

struct McBuf {
  CUmemGenericAllocationHandle mc;
  std::vector<CUdeviceptr> uc, mcva;
};

static McBuf make_buf(int W, size_t size, size_t gran) {
  McBuf b;
  CUmulticastObjectProp mp = {};
  mp.numDevices = W;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = size;
  CK(p_cuMulticastCreate(&b.mc, &mp));
  for (int d = 0; d < W; ++d) CK(p_cuMulticastAddDevice(b.mc, d));
  b.uc.resize(W);
  b.mcva.resize(W);
  for (int d = 0; d < W; ++d) {
    CR(cudaSetDevice(d));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CUmemGenericAllocationHandle h;
    CK(p_cuMemCreate(&h, size, &ap, 0));
    CK(p_cuMulticastBindMem(b.mc, 0, h, 0, size, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(p_cuMemAddressReserve(&b.uc[d], size, gran, 0, 0));
    CK(p_cuMemMap(b.uc[d], size, 0, h, 0));
    CK(p_cuMemSetAccess(b.uc[d], size, &ad, 1));
    CR(cudaMemset((void*)b.uc[d], 0, size));
    CK(p_cuMemAddressReserve(&b.mcva[d], size, gran, 0, 0));
    CK(p_cuMemMap(b.mcva[d], size, 0, b.mc, 0));
    CK(p_cuMemSetAccess(b.mcva[d], size, &ad, 1));
  }
  return b;
}

int main(int argc, char** argv) {
  size_t mb = argc > 1 ? atoi(argv[1]) : 512;
  int reps = argc > 2 ? atoi(argv[2]) : 20;
  CR(cudaFree(0));
  load(p_cuMulticastCreate, "cuMulticastCreate"); load(p_cuMulticastAddDevice, "cuMulticastAddDevice");
  load(p_cuMulticastBindMem, "cuMulticastBindMem"); load(p_cuMulticastGetGranularity, "cuMulticastGetGranularity");
  load(p_cuMemCreate, "cuMemCreate"); load(p_cuMemAddressReserve, "cuMemAddressReserve");
  load(p_cuMemMap, "cuMemMap"); load(p_cuMemSetAccess, "cuMemSetAccess");
  int W = 0;
  CR(cudaGetDeviceCount(&W));
  if (W < 2) { printf("{\"skipped\": \"need >= 2 GPUs\"}\n"); return 0; }
  CUmulticastObjectProp mp = {};
  mp.numDevices = W;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = mb << 20;
  size_t gran = 0;
  CK(p_cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t size = ((mb << 20) + gran * W - 1) / (gran * W) * (gran * W);
  McBuf bucket = make_buf(W, size, gran), param = make_buf(W, size, gran);
  size_t shard = size / W;                                  // bytes per rank (allocation stride)
  size_t used = std::min(shard, ((mb << 20) / W) & ~(size_t)15);   // bytes per rank processed
  std::vector<float*> local(W);
  std::vector<cudaStream_t> st(W);
  std::vector<cudaEvent_t> e0(W), e1(W);
  for (int d = 0; d < W; ++d) {
    CR(cudaSetDevice(d));
    CR(cudaMalloc(&local[d], shard));
    CR(cudaMemset(local[d], 0, shard));
    CR(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CR(cudaEventCreate(&e0[d]));
    CR(cudaEventCreate(&e1[d]));
  }
  const char* names[3] = {"ld_reduce", "st", "fused"};
  printf("{\"world\": %d, \"bucket_MB\": %.1f, \"allocation_MB\": %.1f, \"rows\": [\n", W,
         used * W / 1048576.0, size / 1048576.0);
  bool first = true;
  for (int mode = 0; mode < 3; ++mode) {
    for (int ctas : {32, 64, 148, 296}) {
      float worst = 0.f;
      for (int rep = -2; rep < reps; ++rep) {
        for (int d = 0; d < W; ++d) { CR(cudaSetDevice(d)); CR(cudaDeviceSynchronize()); }
        for (int d = 0; d < W; ++d) {
          CR(cudaSetDevice(d));
          CR(cudaEventRecord(e0[d], st[d]));
          shard_kernel<<<ctas, kThreads, 0, st[d]>>>(mode, (const float*)(bucket.mcva[d] + d * shard),
                                                     (float*)(param.mcva[d] + d * shard), local[d],
                                                     (long long)(used / 16));
          CR(cudaEventRecord(e1[d], st[d]));
        }
        float mx = 0.f;
        for (int d = 0; d < W; ++d) {
          CR(cudaSetDevice(d));
          CR(cudaEventSynchronize(e1[d]));
          float ms = 0.f;
          CR(cudaEventElapsedTime(&ms, e0[d], e1[d]));
          mx = std::max(mx, ms);
        }
        if (rep >= 0) worst += mx;
      }
      float ms = worst / reps;
      double S = (double)used * W;
      double link = mode == 0 ? S : mode == 1 ? S : S * (W + 1) / W;   // per GPU, busiest direction
      double bus = 2.0 * (W - 1) / W * S;
      printf("%s {\"kernel\": \"%s\", \"ctas\": %d, \"ms\": %.4f, \"shard_GBps\": %.1f, "
             "\"link_GBps\": %.1f, \"busbw_equiv_GBps\": %.1f}",
             first ? "" : ",\n", names[mode], ctas, ms, used / (ms * 1e6), link / (ms * 1e6),
             mode == 2 ? bus / (ms * 1e6) : 0.0);
      first = false;
    }
  }
  printf("\n]}\n");
  return 0;
}
