// crossover_p2p.cu -- collective-fused update over NVLink peer memory.
//
// One kernel replaces reduce-scatter + K2 + all-gather.  Every rank owns one shard of the
// app's flat parameter buffer.  For its shard it
//   1. reads the shard of EVERY rank's bucket over NVLink (peer pointers opened with CUDA IPC)
//      and sums them in rank order 0..W-1 -- the reference's left-to-right
//      average_gradients order (equivalence.py:156-159), so the result is bit-identical to
//      the fp32 oracle for any W (NCCL's ring order is not);
//   2. divides by W and applies the SGD(-momentum) rule (same sgd_elem as K2);
//   3. writes the new parameters into EVERY rank's flat buffer (local + W-1 remote stores),
//      i.e. the all-gather is fused into the epilogue.
// The host brackets the kernel with two stream-ordered NCCL barriers (all K1 packs done
// before the first peer read; all peer writes done before any rank's next forward).
// Memory: cs_device_alloc'd (cudaMalloc, IPC-capable) buffers only.
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"
#include "crossover_sgd.cuh"

namespace cs {

// persistent grid cap; 0 = 2 CTAs per SM (measured best in isolation at W = 2 and 4,
// profiles/r01_c1/); a smaller cap trades sync speed for fewer SMs under a concurrent GEMM
int g_tune_p2p_ctas = 0;

namespace {
__device__ __forceinline__ float4 ld_peer(const float* p) {
  // peer (NVLink) or local read-once data; L2-bypassed for peer apertures by the hardware
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
}  // namespace

// U float4 per thread per source: W * U = 8 peer loads in flight per thread for W = 2, 4, 8
template <int U>
__host__ __device__ constexpr int p2p_chunk_elems() { return kThreads * 4 * U; }

template <bool kMom, int U, int MAXW>
__device__ __forceinline__ void p2p_chunk(const cs_p2p_desc& d, const Rule& r, int64_t e0);

// Persistent when the grid is capped (cs_tune "p2p_ctas"): a comm kernel that overlaps another
// app's compute should hold as few SMs as keep NVLink busy; each CTA walks chunks with stride.
template <bool kMom, int U, int MAXW>
__global__ void __launch_bounds__(kThreads)
p2p_reduce_sgd_bcast_kernel(const __grid_constant__ cs_p2p_desc d, const __grid_constant__ cs_sgd_hyper h) {
  constexpr int CH = p2p_chunk_elems<U>();
  const Rule r = make_rule(h, kMom);
  const int64_t chunks = (d.numel + CH - 1) / CH;
  for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x) p2p_chunk<kMom, U, MAXW>(d, r, c * CH);
  __threadfence_system();   // remote stores performed before the kernel retires
}

template <bool kMom, int kP2PUnroll, int MAXW>
__device__ __forceinline__ void p2p_chunk(const cs_p2p_desc& d, const Rule& r, int64_t e0) {
  constexpr int kP2PChunk = p2p_chunk_elems<kP2PUnroll>();
  const int64_t rem = d.numel - e0;
  const int n = rem < kP2PChunk ? (int)rem : kP2PChunk;
  const int tid = threadIdx.x;
  const int W = d.nranks;
  float* p = d.param + e0;
  float* m = kMom ? d.momentum_buf + e0 : nullptr;
  const int nvec = n >> 2;

  float4 acc[kP2PUnroll], pv[kP2PUnroll], mv[kP2PUnroll];
#pragma unroll
  for (int u = 0; u < kP2PUnroll; ++u) {
    const int idx = u * kThreads + tid;
    acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    mv[u] = acc[u];
    pv[u] = acc[u];
    if (idx < nvec) {
      pv[u] = *(const float4*)(p + 4 * idx);
      if (kMom) mv[u] = *(const float4*)(m + 4 * idx);
    }
  }
  // all W x U peer loads in flight before the first add
  float4 g[MAXW][kP2PUnroll];
#pragma unroll
  for (int s = 0; s < MAXW; ++s) {
    if (s < W) {
      const float* src = (const float*)d.src[s] + e0;
#pragma unroll
      for (int u = 0; u < kP2PUnroll; ++u) {
        const int idx = u * kThreads + tid;
        g[s][u] = idx < nvec ? ld_peer(src + 4 * idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < MAXW; ++s) {
    if (s < W) {
#pragma unroll
      for (int u = 0; u < kP2PUnroll; ++u) {
        acc[u].x = __fadd_rn(acc[u].x, g[s][u].x);
        acc[u].y = __fadd_rn(acc[u].y, g[s][u].y);
        acc[u].z = __fadd_rn(acc[u].z, g[s][u].z);
        acc[u].w = __fadd_rn(acc[u].w, g[s][u].w);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kP2PUnroll; ++u) {
    const int idx = u * kThreads + tid;
    if (idx < nvec) {
      float4 o;
      o.x = sgd_elem(r, acc[u].x, pv[u].x, &mv[u].x);
      o.y = sgd_elem(r, acc[u].y, pv[u].y, &mv[u].y);
      o.z = sgd_elem(r, acc[u].z, pv[u].z, &mv[u].z);
      o.w = sgd_elem(r, acc[u].w, pv[u].w, &mv[u].w);
      if (kMom) st4(m + 4 * idx, mv[u]);
      for (int s = 0; s < W; ++s) st4((float*)d.dst[s] + e0 + 4 * idx, o);   // fused all-gather
    }
  }
  for (int k = 4 * nvec + tid; k < n; k += kThreads) {
    float a = 0.0f;
    for (int s = 0; s < W; ++s) a = __fadd_rn(a, ((const float*)d.src[s])[e0 + k]);
    float b = kMom ? m[k] : 0.0f;
    const float np = sgd_elem(r, a, p[k], &b);
    if (kMom) m[k] = b;
    for (int s = 0; s < W; ++s) ((float*)d.dst[s])[e0 + k] = np;
  }
}

template <int U, int MAXW>
static void launch_p2p_u(const cs_p2p_desc& d, const cs_sgd_hyper& h, cudaStream_t s) {
  int64_t grid = (d.numel + p2p_chunk_elems<U>() - 1) / p2p_chunk_elems<U>();
  int cap = d.max_ctas > 0 ? d.max_ctas : g_tune_p2p_ctas;
  if (cap <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = 2 * sms;
  }
  if (grid > cap) grid = cap;
  if (h.momentum != 0.0f) p2p_reduce_sgd_bcast_kernel<true, U, MAXW><<<(unsigned)grid, kThreads, 0, s>>>(d, h);
  else p2p_reduce_sgd_bcast_kernel<false, U, MAXW><<<(unsigned)grid, kThreads, 0, s>>>(d, h);
}

// ---------------------------------------------------------------------------------------------
// Bulk-copy (TMA) variant for a capped grid.  At the crossover cap (a few dozen CTAs) the register
// kernel is latency-bound: each thread keeps only W x U 16-byte peer loads in flight.  Here one
// thread per CTA streams whole tiles -- every source rank's 8 KB slice, the parameter slice and the
// momentum slice -- into a ring of shared-memory stages with cp.async.bulk (the TMA engine, no
// registers), completion counted by one mbarrier per stage; all threads reduce a landed stage in
// rank order, apply the update and store the new slice to every rank while the next stages are in
// flight.  The arithmetic is p2p_chunk's (same order, same sgd_elem), so the result is bitwise
// identical.  Used for every launch whose grid cap is set (the crossover case), unless
// cs_tune("p2p_bulk", 0); the uncapped whole-GPU launch keeps the register kernel.
// ---------------------------------------------------------------------------------------------
int g_tune_p2p_bulk = 1;
constexpr int kDescVecs = (int)(sizeof(cs_p2p_desc) / 16);
static_assert(sizeof(cs_p2p_desc) % 16 == 0, "cs_p2p_desc must be a whole number of 16-byte vectors");

// floats per buffer per stage: 16 KB at W <= 2 (fewer, longer tiles: the per-tile wait / barrier /
// issue overhead is paid half as often), 8 KB above; stages so a CTA keeps 128-192 KB in flight
template <int MAXW>
__host__ __device__ constexpr int bulk_tile() { return MAXW <= 2 ? 4096 : 2048; }
template <int MAXW>
__host__ __device__ constexpr int bulk_stages() { return MAXW <= 2 ? 3 : (MAXW <= 4 ? 3 : 2); }
template <bool kMom, int MAXW>
__host__ __device__ constexpr int bulk_buffers() { return MAXW + (kMom ? 2 : 1); }
template <bool kMom, int MAXW>
constexpr size_t bulk_smem_bytes() {
  return (size_t)bulk_stages<MAXW>() * bulk_buffers<kMom, MAXW>() * bulk_tile<MAXW>() * 4;
}
static_assert(bulk_smem_bytes<true, 2>() <= 227 * 1024 && bulk_smem_bytes<true, 4>() <= 227 * 1024 &&
              bulk_smem_bytes<true, CS_MAX_SOURCES>() <= 227 * 1024, "bulk P2P ring exceeds shared memory");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity)
      : "memory");
}

// kTable = false: the tiles of one contiguous shard (d); kTable = true: the p2p_gather chunk table
// (one cs_p2p_desc per chunk, numel <= one tile, not necessarily a multiple of 4: the copy is
// rounded up to 16 bytes -- inside the caching allocator's 512-byte blocks and the padded layout --
// and the last n & 3 elements take a scalar path).  Thread 0 writes each stage's tile descriptor
// into shared memory before arming its mbarrier, so the consumers read it after the wait.
template <bool kMom, int MAXW, bool kTable>
__global__ void __launch_bounds__(kThreads, 1)
p2p_bulk_kernel(const __grid_constant__ cs_p2p_desc d, const cs_p2p_desc* __restrict__ table, int64_t ntable,
                const __grid_constant__ cs_sgd_hyper h) {
  constexpr int S = bulk_stages<MAXW>();
  constexpr int kBulkTile = bulk_tile<MAXW>();
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full[S];
  __shared__ __align__(16) cs_p2p_desc info[S];
  __shared__ __align__(16) cs_p2p_desc pf[kTable ? S : 1];   // table entries prefetched S tiles ahead
  const Rule r = make_rule(h, kMom);
  const int W = d.nranks;
  const int nb = W + (kMom ? 2 : 1);             // buffers of a stage: W sources, p (, m)
  const int64_t units = kTable ? ntable : (d.numel + kBulkTile - 1) / kBulkTile;
  const int64_t mine = units > blockIdx.x ? (units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto prefetch = [&](int64_t k, int s) {        // thread 0: table entry of tile k -> pf[s], one group
    if (k < mine) {
      const char* g = reinterpret_cast<const char*>(table + blockIdx.x + k * gridDim.x);
      for (int v = 0; v < kDescVecs; ++v)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(reinterpret_cast<char*>(&pf[s]) + 16 * v)),
                     "l"(g + 16 * v)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t k, int s) {           // thread 0: tile k of this CTA into stage s
    const int64_t u = blockIdx.x + k * gridDim.x;
    cs_p2p_desc& t = info[s];
    if (kTable) {
      // entry k landed: groups are committed one per tile in order (S in the prologue, then one
      // per issue), so at most S - 1 younger ones may still be pending
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
      t = pf[s];
      prefetch(k + S, s);
    } else {
      const int64_t e0 = u * kBulkTile;
      const int64_t rem = d.numel - e0;
      for (int b = 0; b < W; ++b) {
        t.src[b] = d.src[b] + 4 * (uint64_t)e0;
        t.dst[b] = d.dst[b] + 4 * (uint64_t)e0;
      }
      t.param = d.param + e0;
      t.momentum_buf = kMom ? d.momentum_buf + e0 : nullptr;
      t.numel = rem < kBulkTile ? rem : kBulkTile;
    }
    const uint32_t bytes = (uint32_t)((t.numel * 4 + 15) & ~(int64_t)15);
    const uint32_t bar = smem_u32(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * nb) : "memory");
    float* st = ring + (size_t)s * nb * kBulkTile;
    for (int b = 0; b < nb; ++b) {
      const float* src = b < W ? (const float*)t.src[b] : (b == W ? t.param : t.momentum_buf);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(st + (size_t)b * kBulkTile)), "l"(src), "r"(bytes), "r"(bar)
                   : "memory");
    }
  };
  if (threadIdx.x == 0) {
    if (kTable)
      for (int k = 0; k < S; ++k) prefetch(k, k);
    for (int k = 0; k < S && k < mine; ++k) issue(k, k);
  }
  constexpr int V = kBulkTile / 4;                 // float4 per buffer
  for (int64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % S);
    mbar_wait(smem_u32(&full[s]), (uint32_t)((k / S) & 1));
    const cs_p2p_desc& t = info[s];
    const int n = (int)t.numel;
    const int nvec = n >> 2;
    const float* sf = ring + (size_t)s * nb * kBulkTile;
    const float4* st = reinterpret_cast<const float4*>(sf);
    for (int v = threadIdx.x; v < nvec; v += kThreads) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int src = 0; src < MAXW; ++src) {
        if (src < W) {
          const float4 g = st[src * V + v];
          acc.x = __fadd_rn(acc.x, g.x);
          acc.y = __fadd_rn(acc.y, g.y);
          acc.z = __fadd_rn(acc.z, g.z);
          acc.w = __fadd_rn(acc.w, g.w);
        }
      }
      const float4 pv = st[W * V + v];
      float4 mv = kMom ? st[(W + 1) * V + v] : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 o;
      o.x = sgd_elem(r, acc.x, pv.x, &mv.x);
      o.y = sgd_elem(r, acc.y, pv.y, &mv.y);
      o.z = sgd_elem(r, acc.z, pv.z, &mv.z);
      o.w = sgd_elem(r, acc.w, pv.w, &mv.w);
      if (kMom) st4(t.momentum_buf + 4 * v, mv);
      for (int dst = 0; dst < W; ++dst) st4((float*)t.dst[dst] + 4 * v, o);   // fused all-gather
    }
    if (kTable) {
      for (int e = 4 * nvec + threadIdx.x; e < n; e += kThreads) {   // tensor tail (n & 3 elements)
        float a = 0.0f;
        for (int src = 0; src < W; ++src) a = __fadd_rn(a, sf[src * kBulkTile + e]);
        float b = kMom ? sf[(W + 1) * kBulkTile + e] : 0.0f;
        const float np = sgd_elem(r, a, sf[W * kBulkTile + e], &b);
        if (kMom) t.momentum_buf[e] = b;
        for (int dst = 0; dst < W; ++dst) ((float*)t.dst[dst])[e] = np;
      }
    }
    __syncthreads();                               // every thread is done with stage s
    if (threadIdx.x == 0 && k + S < mine) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
      issue(k + S, s);
    }
  }
  if (kTable && threadIdx.x == 0) asm volatile("cp.async.wait_all;" ::: "memory");
  __threadfence_system();
}

template <int MAXW, bool kTable>
static cudaError_t launch_bulk(const cs_p2p_desc& d, const cs_p2p_desc* table, int64_t ntable, int max_ctas,
                               const cs_sgd_hyper& h, cudaStream_t s) {
  const int64_t units = kTable ? ntable : (d.numel + bulk_tile<MAXW>() - 1) / bulk_tile<MAXW>();
  const int grid = (int)(units < max_ctas ? units : max_ctas);
  if (grid <= 0) return cudaSuccess;
  const bool mom = h.momentum != 0.0f;
  const size_t smem = mom ? bulk_smem_bytes<true, MAXW>() : bulk_smem_bytes<false, MAXW>();
  auto* k = mom ? p2p_bulk_kernel<true, MAXW, kTable> : p2p_bulk_kernel<false, MAXW, kTable>;
  // the dynamic shared-memory opt-in, once per instantiation and device (a racing second call
  // only repeats the same idempotent setting)
  static bool opted[2][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !opted[mom][dev]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) opted[mom][dev] = true;
  }
  k<<<(unsigned)grid, kThreads, smem, s>>>(d, table, ntable, h);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K1-free variant: the chunks of this rank's shard read every rank's gradient tensors in place.
// One self-contained descriptor per chunk (pointers already at the chunk, numel <= one chunk);
// the next chunk's descriptor is fetched into shared memory with cp.async while the current one
// is processed, so the table lookup adds no latency to the peer loads.  The per-element code is
// p2p_chunk's, so the arithmetic is bit-identical to the bucket kernel.
// ---------------------------------------------------------------------------------------------

__device__ __forceinline__ void desc_prefetch(cs_p2p_desc* dst, const cs_p2p_desc* src) {
  if (threadIdx.x < kDescVecs) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(reinterpret_cast<char*>(dst) + 16 * threadIdx.x);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s),
                 "l"(reinterpret_cast<const char*>(src) + 16 * threadIdx.x)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <bool kMom, int U, int MAXW>
__global__ void __launch_bounds__(kThreads)
p2p_gather_kernel(const cs_p2p_desc* __restrict__ chunks, int64_t nchunks, const __grid_constant__ cs_sgd_hyper h) {
  __shared__ __align__(16) cs_p2p_desc sd[2];
  const Rule r = make_rule(h, kMom);
  int64_t c = blockIdx.x;
  if (c < nchunks) desc_prefetch(&sd[0], chunks + c);
  for (int buf = 0; c < nchunks; c += gridDim.x, buf ^= 1) {
    const int64_t next = c + gridDim.x;
    if (next < nchunks) desc_prefetch(&sd[buf ^ 1], chunks + next);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");   // this chunk's descriptor landed
    __syncthreads();
    p2p_chunk<kMom, U, MAXW>(sd[buf], r, 0);
    __syncthreads();          // sd[buf] is the prefetch target of the next iteration but one
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __threadfence_system();
}

template <int U, int MAXW>
static void launch_gather_u(const cs_p2p_desc* chunks, int64_t nchunks, int max_ctas, const cs_sgd_hyper& h,
                            cudaStream_t s) {
  int cap = max_ctas > 0 ? max_ctas : g_tune_p2p_ctas;
  if (cap <= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = 2 * sms;
  }
  const unsigned grid = (unsigned)(nchunks < cap ? nchunks : cap);
  if (h.momentum != 0.0f) p2p_gather_kernel<true, U, MAXW><<<grid, kThreads, 0, s>>>(chunks, nchunks, h);
  else p2p_gather_kernel<false, U, MAXW><<<grid, kThreads, 0, s>>>(chunks, nchunks, h);
}

int64_t p2p_gather_chunk_elems(int nranks) {
  if (nranks <= 2) return p2p_chunk_elems<4>();
  if (nranks <= 4) return p2p_chunk_elems<2>();
  return p2p_chunk_elems<1>();
}

cudaError_t launch_p2p_gather(const cs_p2p_desc* chunks, int64_t nchunks, int nranks, int max_ctas,
                              const cs_sgd_hyper& h, cudaStream_t s) {
  if (nchunks == 0) return cudaSuccess;
  if (g_tune_p2p_bulk && max_ctas > 0) {           // capped: the TMA-fed ring (the tile fields come
    cs_p2p_desc d = {};                            // from the table; d carries only W)
    d.nranks = nranks;
    if (nranks <= 2) return launch_bulk<2, true>(d, chunks, nchunks, max_ctas, h, s);
    if (nranks <= 4) return launch_bulk<4, true>(d, chunks, nchunks, max_ctas, h, s);
    return launch_bulk<CS_MAX_SOURCES, true>(d, chunks, nchunks, max_ctas, h, s);
  }
  if (nranks <= 2) launch_gather_u<4, 2>(chunks, nchunks, max_ctas, h, s);
  else if (nranks <= 4) launch_gather_u<2, 4>(chunks, nchunks, max_ctas, h, s);
  else launch_gather_u<1, CS_MAX_SOURCES>(chunks, nchunks, max_ctas, h, s);
  return cudaGetLastError();
}

cudaError_t launch_p2p(const cs_p2p_desc& d, const cs_sgd_hyper& h, cudaStream_t s) {
  if (d.numel == 0) return cudaSuccess;
  if (g_tune_p2p_bulk && d.max_ctas > 0 && d.numel % 4 == 0) {
    if (d.nranks <= 2) return launch_bulk<2, false>(d, nullptr, 0, d.max_ctas, h, s);
    if (d.nranks <= 4) return launch_bulk<4, false>(d, nullptr, 0, d.max_ctas, h, s);
    return launch_bulk<CS_MAX_SOURCES, false>(d, nullptr, 0, d.max_ctas, h, s);
  }
  if (d.nranks <= 2) launch_p2p_u<4, 2>(d, h, s);
  else if (d.nranks <= 4) launch_p2p_u<2, 4>(d, h, s);
  else launch_p2p_u<1, CS_MAX_SOURCES>(d, h, s);
  return cudaGetLastError();
}

}  // namespace cs
