// crossover_kernels.cu -- register-path sm_100a kernels of the crossover step.
//
//   K1  pack_kernel        gradient fusion into one contiguous bucket
//                          (reference: workload.fuse_gradients, workload.py:94-101)
//   K2  unpack_sgd_kernel  fixed-order reduction over sources, / W, SGD(-momentum)
//                          (reference: equivalence.average_gradients + sgd_step,
//                           equivalence.py:150-168)
//   K3  stats_kernel       warp-reduced gradient sum-of-squares / non-finite count
//
// All three are HBM-streaming kernels: no data reuse, so no shared-memory
// staging and no tensor cores.  Work is cut into fixed CHUNK-element chunks
// (one CTA each, CHUNK = 256 threads x 4 floats x U) so a 64-element BatchNorm
// bias and a 2.4M-element conv weight get the same per-CTA shape; the tensor
// owning a chunk is found by a binary search over the chunk prefix held in
// __grid_constant__ kernel parameters (uniform per CTA -> constant-cache
// broadcast, no device-side table, no per-step H2D copy).  Each thread keeps
// U independent 128-bit loads per stream in flight before its first store.
// The launch shape (U, CTAs per SM) is a template choice selected at run time
// (reg_shape(), cs_tune "reg_shape"); results never depend on it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"
#include "crossover_sgd.cuh"

namespace cs {

int g_tune_reg_shape = 1;
int g_tune_sync_ctas = 0;   // 0: one CTA per chunk; >0: persistent grid capped at this many CTAs

// grid of K1 / K2: one CTA per chunk, or a persistent grid of at most `cap` CTAs (per-launch cap,
// else the process-wide cs_tune("sync_ctas")).  A sync that overlaps another app's compute on a
// high-priority stream should be persistent: a one-CTA-per-chunk grid keeps thousands of
// high-priority CTAs pending, and the block scheduler dispatches none of the other stream's CTAs
// until the last of them has been placed.
static int sync_grid(int chunks, int cap) {
  if (cap <= 0) cap = g_tune_sync_ctas;
  return cap > 0 && chunks > cap ? cap : chunks;
}

// ---------------------------------------------------------------------------
// 128-bit memory helpers (inline PTX so the cache policy is explicit)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream(const float* p) {
  // read-once data (gradients, reduced buckets): non-coherent path, no L1 allocation
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_rw(const float* p) {
  // read-then-written data (parameters, momentum buffers)
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ int find_segment(const int* chunk_begin, int n, int c) {
  // largest i with chunk_begin[i] <= c (zero-chunk tensors are skipped naturally)
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (chunk_begin[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// K1: pack
// ---------------------------------------------------------------------------
template <int CAP, int U>
__device__ __forceinline__ void pack_chunk(const PackArgs<CAP>& a, int c);

// grid = #chunks (one chunk per CTA) or capped (cs_tune "sync_ctas"): persistent over chunks.
// The min-blocks hint keeps ptxas from capping the kernel at 32 registers (which spilled 8 bytes).
template <int CAP, int U>
__global__ void __launch_bounds__(kThreads, 4)
pack_kernel(const __grid_constant__ PackArgs<CAP> a) {
  for (int c = blockIdx.x; c < a.total_chunks; c += gridDim.x) pack_chunk<CAP, U>(a, c);
}

template <int CAP, int U>
__device__ __forceinline__ void pack_chunk(const PackArgs<CAP>& a, int c) {
  constexpr int CH = kThreads * 4 * U;
  const int i = find_segment(a.chunk_begin, a.n, c);
  const int64_t e0 = (int64_t)(c - a.chunk_begin[i]) * CH;
  const float* __restrict__ src = a.src[i] + e0;
  float* __restrict__ dst = a.dst[i] + e0;
  const int64_t rem = a.numel[i] - e0;
  const int n = rem < CH ? (int)rem : CH;
  const int tid = threadIdx.x;

  if ((((uintptr_t)src) | ((uintptr_t)dst)) & 15u) {
    // misaligned tensor/bucket offset: scalar, still coalesced
    for (int k = tid; k < n; k += kThreads) dst[k] = src[k];
    return;
  }
  const int nvec = n >> 2;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int idx = u * kThreads + tid;
    if (idx < nvec) v[u] = ld_stream(src + 4 * idx);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int idx = u * kThreads + tid;
    if (idx < nvec) st_v4(dst + 4 * idx, v[u]);
  }
  for (int k = 4 * nvec + tid; k < n; k += kThreads) dst[k] = src[k];
}

// ---------------------------------------------------------------------------
// K2: fixed-order reduce over sources, average, SGD update
// ---------------------------------------------------------------------------
template <int CAP, bool kMom, int U>
__device__ __forceinline__ void unpack_sgd_chunk(const UpdateArgs<CAP>& a, const Rule& r, int c);

template <int CAP, bool kMom, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
unpack_sgd_kernel(const __grid_constant__ UpdateArgs<CAP> a) {
  const Rule r = make_rule(a.h, kMom);
  for (int c = blockIdx.x; c < a.total_chunks; c += gridDim.x) unpack_sgd_chunk<CAP, kMom, U>(a, r, c);
}

template <int CAP, bool kMom, int U>
__device__ __forceinline__ void unpack_sgd_chunk(const UpdateArgs<CAP>& a, const Rule& r, int c) {
  constexpr int CH = kThreads * 4 * U;
  const int i = find_segment(a.chunk_begin, a.n, c);
  const int64_t e0 = (int64_t)(c - a.chunk_begin[i]) * CH;
  const int64_t rem = a.numel[i] - e0;
  const int n = rem < CH ? (int)rem : CH;
  const int tid = threadIdx.x;

  float* __restrict__ p = a.param[i] + e0;
  float* __restrict__ m = kMom ? a.mom[i] + e0 : nullptr;
  float* __restrict__ snap =
      a.snapshot ? (float*)((char*)a.snapshot + a.snap_off[i]) + e0 : nullptr;
  const uint64_t goff = a.grad_off[i] + (uint64_t)e0 * 4u;
  const int nsrc = a.nsrc;

  uintptr_t align = (uintptr_t)p | (uintptr_t)goff | (kMom ? (uintptr_t)m : 0) |
                    (snap ? (uintptr_t)snap : 0);
  for (int s = 0; s < nsrc; ++s) align |= (uintptr_t)a.base[s];

  if (align & 15u) {
    for (int k = tid; k < n; k += kThreads) {
      float acc = 0.0f;
      for (int s = 0; s < nsrc; ++s)
        acc = __fadd_rn(acc, ((const float*)(a.base[s] + goff))[k]);
      float b = kMom ? m[k] : 0.0f;
      float np = sgd_elem(r, acc, p[k], &b);
      p[k] = np;
      if (kMom) m[k] = b;
      if (snap) snap[k] = np;
    }
    return;
  }

  const int nvec = n >> 2;
  float4 acc[U], pv[U], mv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int idx = u * kThreads + tid;
    acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    mv[u] = acc[u];
    if (idx < nvec) {
      pv[u] = ld_rw(p + 4 * idx);
      if (kMom) mv[u] = ld_rw(m + 4 * idx);
    }
  }
  for (int s = 0; s < nsrc; ++s) {
    const float* g = (const float*)(a.base[s] + goff);
    float4 gv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = u * kThreads + tid;
      gv[u] = idx < nvec ? ld_stream(g + 4 * idx) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc[u].x = __fadd_rn(acc[u].x, gv[u].x);
      acc[u].y = __fadd_rn(acc[u].y, gv[u].y);
      acc[u].z = __fadd_rn(acc[u].z, gv[u].z);
      acc[u].w = __fadd_rn(acc[u].w, gv[u].w);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int idx = u * kThreads + tid;
    if (idx < nvec) {
      float4 o;
      o.x = sgd_elem(r, acc[u].x, pv[u].x, &mv[u].x);
      o.y = sgd_elem(r, acc[u].y, pv[u].y, &mv[u].y);
      o.z = sgd_elem(r, acc[u].z, pv[u].z, &mv[u].z);
      o.w = sgd_elem(r, acc[u].w, pv[u].w, &mv[u].w);
      st_v4(p + 4 * idx, o);
      if (kMom) st_v4(m + 4 * idx, mv[u]);
      if (snap) st_v4(snap + 4 * idx, o);
    }
  }
  for (int k = 4 * nvec + tid; k < n; k += kThreads) {
    float accs = 0.0f;
    for (int s = 0; s < nsrc; ++s)
      accs = __fadd_rn(accs, ((const float*)(a.base[s] + goff))[k]);
    float b = kMom ? m[k] : 0.0f;
    float np = sgd_elem(r, accs, p[k], &b);
    p[k] = np;
    if (kMom) m[k] = b;
    if (snap) snap[k] = np;
  }
}

// ---------------------------------------------------------------------------
// K3: gradient health (sum of squares in fp64, non-finite count)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stats_accum(float x, double& ss, unsigned long long& bad) {
  if (isfinite(x)) ss += (double)x * (double)x; else bad += 1ull;
}

__global__ void __launch_bounds__(kThreads)
stats_kernel(const float* __restrict__ data, int64_t numel, double* __restrict__ out,
             double* __restrict__ partial, unsigned int* __restrict__ ticket) {
  double ss = 0.0;
  unsigned long long bad = 0ull;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t t0 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int head = (int)(((16u - ((uintptr_t)data & 15u)) & 15u) >> 2);
  const int64_t h = head < numel ? head : numel;
  if (((uintptr_t)data & 3u) == 0) {
    for (int64_t k = t0; k < h; k += stride) stats_accum(data[k], ss, bad);
    const int64_t nvec = (numel - h) >> 2;
    const float* d4 = data + h;
    for (int64_t v = t0; v < nvec; v += stride) {
      float4 x = ld_stream(d4 + 4 * v);
      stats_accum(x.x, ss, bad); stats_accum(x.y, ss, bad);
      stats_accum(x.z, ss, bad); stats_accum(x.w, ss, bad);
    }
    for (int64_t k = h + 4 * nvec + t0; k < numel; k += stride) stats_accum(data[k], ss, bad);
  } else {
    for (int64_t k = t0; k < numel; k += stride) stats_accum(data[k], ss, bad);
  }
  // warp-level reduction (fixed shuffle tree -> deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_down_sync(0xffffffffu, ss, o);
    bad += __shfl_down_sync(0xffffffffu, bad, o);
  }
  __shared__ double s_ss[kThreads / 32];
  __shared__ unsigned long long s_bad[kThreads / 32];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_ss[warp] = ss; s_bad[warp] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bs = 0.0; unsigned long long bb = 0ull;
    for (int w = 0; w < kThreads / 32; ++w) { bs += s_ss[w]; bb += s_bad[w]; }
    partial[2 * blockIdx.x] = bs;
    partial[2 * blockIdx.x + 1] = (double)bb;
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    double ts = 0.0, tb = 0.0;
    for (unsigned int b = 0; b < gridDim.x; ++b) {
      ts += ((volatile double*)partial)[2 * b];
      tb += ((volatile double*)partial)[2 * b + 1];
    }
    out[0] += ts;
    out[1] += tb;
    *ticket = 0u;  // leave the workspace ready for the next launch
  }
}

// ---------------------------------------------------------------------------
// host-side launchers (called from crossover_abi.cu)
//   reg shapes: 0 = (U4, 2 CTA/SM)  1 = (U4, 3)  2 = (U2, 4)  3 = (U8, 1)  4 = (U2, 3)
// ---------------------------------------------------------------------------
static int shape_unroll(int shape) {
  static const int u[] = {4, 4, 2, 8, 2};
  return u[shape];
}

int reg_pack_chunk() { return kThreads * 4 * (g_tune_reg_shape == 3 ? 8 : 4); }
int reg_update_chunk() { return kThreads * 4 * shape_unroll(g_tune_reg_shape); }

template <int CAP>
cudaError_t launch_pack(const PackArgs<CAP>& a, int cap, cudaStream_t s) {
  if (a.total_chunks == 0) return cudaSuccess;
  const int g = sync_grid(a.total_chunks, cap);
  if (g_tune_reg_shape == 3) pack_kernel<CAP, 8><<<g, kThreads, 0, s>>>(a);
  else pack_kernel<CAP, 4><<<g, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

template <int CAP, bool kMom>
static void launch_update_shape(const UpdateArgs<CAP>& a, int cap, cudaStream_t s) {
  const int g = sync_grid(a.total_chunks, cap);
  switch (g_tune_reg_shape) {
    case 1: unpack_sgd_kernel<CAP, kMom, 4, 3><<<g, kThreads, 0, s>>>(a); break;
    case 2: unpack_sgd_kernel<CAP, kMom, 2, 4><<<g, kThreads, 0, s>>>(a); break;
    case 3: unpack_sgd_kernel<CAP, kMom, 8, 1><<<g, kThreads, 0, s>>>(a); break;
    case 4: unpack_sgd_kernel<CAP, kMom, 2, 3><<<g, kThreads, 0, s>>>(a); break;
    default: unpack_sgd_kernel<CAP, kMom, 4, 2><<<g, kThreads, 0, s>>>(a); break;
  }
}

template <int CAP>
cudaError_t launch_unpack_sgd(const UpdateArgs<CAP>& a, bool mom, int cap, cudaStream_t s) {
  if (a.total_chunks == 0) return cudaSuccess;
  if (mom) launch_update_shape<CAP, true>(a, cap, s);
  else launch_update_shape<CAP, false>(a, cap, s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// fixed-duration compute stand-in: one thread spins on the global nanosecond timer
// ---------------------------------------------------------------------------
__global__ void spin_ns_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t s) {
  spin_ns_kernel<<<1, 1, 0, s>>>(ns);
  return cudaGetLastError();
}

int stats_grid(int64_t numel) {
  int64_t per_cta = (int64_t)kThreads * 4 * 8;
  int64_t g = (numel + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  if (g > kStatsMaxGrid) g = kStatsMaxGrid;
  return (int)g;
}

cudaError_t launch_stats(const float* data, int64_t numel, double* out, void* ws,
                         cudaStream_t s) {
  const int g = stats_grid(numel);
  unsigned int* ticket = (unsigned int*)ws;
  double* partial = (double*)((char*)ws + 256);
  stats_kernel<<<g, kThreads, 0, s>>>(data, numel, out, partial, ticket);
  return cudaGetLastError();
}

template cudaError_t launch_pack<kCapSmall>(const PackArgs<kCapSmall>&, int, cudaStream_t);
template cudaError_t launch_pack<kCapMid>(const PackArgs<kCapMid>&, int, cudaStream_t);
template cudaError_t launch_pack<kCapLarge>(const PackArgs<kCapLarge>&, int, cudaStream_t);
template cudaError_t launch_unpack_sgd<kCapSmall>(const UpdateArgs<kCapSmall>&, bool, int, cudaStream_t);
template cudaError_t launch_unpack_sgd<kCapMid>(const UpdateArgs<kCapMid>&, bool, int, cudaStream_t);
template cudaError_t launch_unpack_sgd<kCapLarge>(const UpdateArgs<kCapLarge>&, bool, int, cudaStream_t);

}  // namespace cs
