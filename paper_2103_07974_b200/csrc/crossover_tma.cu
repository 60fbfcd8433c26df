// crossover_tma.cu -- TMA-pipelined (cp.async.bulk + mbarrier) versions of K1 and K2.
//
// Persistent CTAs (one per SM, grid = #SMs) walk the chunk list with stride
// gridDim.x.  Thread 0 is the TMA producer: it keeps up to STAGES chunks of
// every input stream in flight with 1-D bulk copies global -> shared that
// complete on a per-stage mbarrier (expect_tx).  All 256 threads compute out
// of shared memory (LDS.128, conflict-free), write the results back into the
// same stage buffers, fence the generic->async proxy, and thread 0 streams
// them out with bulk stores shared -> global (bulk_group).  A stage is
// refilled one iteration after its store was issued (wait_group.read 1), so
// STAGES-2 loads are always in flight per SM without any register staging.
//
// Chunks whose addresses are not 16-byte aligned (exact reference layout with
// odd offsets, views at odd offsets) skip the bulk path: the producer arrives
// on the stage barrier without transactions and the consumers process the
// chunk straight from global memory.  Tails (numel % 4) are always handled
// by direct global accesses.  Arithmetic is identical to crossover_kernels.cu
// (same sgd_elem), so results are bit-identical to the register variant.
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"
#include "crossover_sgd.cuh"

namespace cs {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void st_v4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Descriptor tables live in __grid_constant__ kernel parameters (constant bank).
// A persistent CTA touches every descriptor many times, and dependent constant-
// cache misses on one producer thread serialise the whole pipeline, so each CTA
// first copies the n descriptors it needs into shared memory and walks its
// (monotonically increasing) chunk sequence with a cursor instead of a search.
struct Chunk {
  int seg;
  int64_t e0;
  int n;
};

struct Cursor {
  int seg = 0;
  __device__ __forceinline__ Chunk at(const int* cb, const int64_t* numel, int c, int chunk) {
    while (cb[seg + 1] <= c) ++seg;
    Chunk k;
    k.seg = seg;
    k.e0 = (int64_t)(c - cb[seg]) * chunk;
    const int64_t rem = numel[seg] - k.e0;
    k.n = rem < chunk ? (int)rem : chunk;
    return k;
  }
};

__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~(size_t)127; }

// shared-memory table sizes (bytes) for n descriptors
__host__ __device__ inline size_t pack_table_bytes(int n) {
  return align128((size_t)(n + 1) * 4 + (size_t)n * 24);
}
__host__ __device__ inline size_t update_table_bytes(int n) {
  return align128((size_t)(n + 1) * 4 + (size_t)n * 40);
}

}  // namespace

// ---------------------------------------------------------------------------
// K1 (TMA): bucket <- gradients, staged through shared memory
//   all threads: copy descriptor table to smem; thread 0 = producer + storer
// ---------------------------------------------------------------------------
template <int CAP>
__global__ void __launch_bounds__(kThreads)
pack_tma_kernel(const __grid_constant__ PackArgs<CAP> a, int chunk, int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  const int n = a.n;
  int64_t* t_numel = (int64_t*)(smem + kTmaBarrierBytes);
  const float** t_src = (const float**)(t_numel + n);
  float** t_dst = (float**)(t_src + n);
  int* t_cb = (int*)(t_dst + n);
  float* slots = (float*)(smem + kTmaBarrierBytes + pack_table_bytes(n));
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  const int my_n = (a.total_chunks - (int)blockIdx.x + G - 1) / G;

  for (int i = tid; i <= n; i += kThreads) {
    t_cb[i] = a.chunk_begin[i];
    if (i < n) { t_numel[i] = a.numel[i]; t_src[i] = a.src[i]; t_dst[i] = a.dst[i]; }
  }
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto vec_ok = [&](const Chunk& k) {
    return ((((uintptr_t)(t_src[k.seg] + k.e0)) | ((uintptr_t)(t_dst[k.seg] + k.e0))) & 15u) == 0;
  };
  Cursor prod, cons;
  auto issue = [&](int i) {
    const int slot = i % stages;
    const Chunk k = prod.at(t_cb, t_numel, (int)blockIdx.x + i * G, chunk);
    const uint32_t bytes = (uint32_t)(k.n & ~3) * 4u;
    if (vec_ok(k) && bytes) {
      mbar_arrive_expect_tx(&full[slot], bytes);
      bulk_load(slots + (size_t)slot * chunk, t_src[k.seg] + k.e0, bytes, &full[slot]);
    } else {
      mbar_arrive(&full[slot]);
    }
  };
  if (tid == 0)
    for (int i = 0; i < stages && i < my_n; ++i) issue(i);

  for (int i = 0; i < my_n; ++i) {
    const int slot = i % stages;
    const Chunk k = cons.at(t_cb, t_numel, (int)blockIdx.x + i * G, chunk);
    const float* src = t_src[k.seg] + k.e0;
    float* dst = t_dst[k.seg] + k.e0;
    const int n4 = vec_ok(k) ? (k.n & ~3) : 0;
    mbar_wait(&full[slot], (uint32_t)(i / stages) & 1u);
    for (int e = n4 + tid; e < k.n; e += kThreads) dst[e] = src[e];   // tail / misaligned
    __syncthreads();
    if (tid == 0) {
      if (n4) bulk_store(dst, slots + (size_t)slot * chunk, (uint32_t)n4 * 4u);
      bulk_commit();
      if (i >= 1 && i - 1 + stages < my_n) {
        bulk_wait_read_1();  // stage of iteration i-1 has been read out by its store
        issue(i - 1 + stages);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// K2 (TMA, warp-specialised): sources + param (+ momentum) -> param (+ momentum, snapshot)
//   warp 0     producer : waits empty[s], issues the stage's bulk loads on full[s]
//   warps 1..8 consumers: wait full[s], read the stage from shared memory, update,
//                         store straight to global (STG.128), arrive empty[s]
// stage layout: [g_0 | g_1 | ... | g_{S-1} | p | m], each `chunk` floats
// ---------------------------------------------------------------------------
template <int CAP, bool kMom>
__global__ void __launch_bounds__(kTmaWsThreads)
unpack_sgd_tma_kernel(const __grid_constant__ UpdateArgs<CAP> a, int chunk, int stages, int debug) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + kTmaMaxStages;
  const int n = a.n;
  int64_t* t_numel = (int64_t*)(smem + kTmaBarrierBytes);
  uint64_t* t_goff = (uint64_t*)(t_numel + n);
  uint64_t* t_soff = t_goff + n;
  float** t_param = (float**)(t_soff + n);
  float** t_mom = t_param + n;
  int* t_cb = (int*)(t_mom + n);
  float* slots = (float*)(smem + kTmaBarrierBytes + update_table_bytes(n));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int my_n = (a.total_chunks - (int)blockIdx.x + G - 1) / G;
  const int nsrc = a.nsrc;
  const int nin = nsrc + 1 + (kMom ? 1 : 0);
  const size_t stage_floats = (size_t)nin * chunk;
  constexpr int kConsumers = kTmaWsThreads - 32;
  uint64_t base[CS_MAX_SOURCES];
#pragma unroll
  for (int s = 0; s < CS_MAX_SOURCES; ++s) base[s] = a.base[s];
  float* const snapshot = a.snapshot;

  for (int i = threadIdx.x; i <= n; i += kTmaWsThreads) {
    t_cb[i] = a.chunk_begin[i];
    if (i < n) {
      t_numel[i] = a.numel[i]; t_goff[i] = a.grad_off[i]; t_soff[i] = a.snap_off[i];
      t_param[i] = a.param[i]; t_mom[i] = a.mom[i];
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  auto gsrc = [&](int s, const Chunk& k) {
    return (const float*)(base[s] + t_goff[k.seg] + (uint64_t)k.e0 * 4u);
  };
  auto snap_ptr = [&](const Chunk& k) {
    return snapshot ? (float*)((char*)snapshot + t_soff[k.seg]) + k.e0 : nullptr;
  };
  auto vec_ok = [&](const Chunk& k) {
    uintptr_t al = (uintptr_t)(t_param[k.seg] + k.e0);
    if (kMom) al |= (uintptr_t)(t_mom[k.seg] + k.e0);
    if (snapshot) al |= (uintptr_t)snap_ptr(k);
    for (int s = 0; s < nsrc; ++s) al |= (uintptr_t)gsrc(s, k);
    return (al & 15u) == 0 && k.n >= 4;
  };

  Cursor cur;
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < my_n; ++i) {
        const int slot = i % stages;
        if (i >= stages) mbar_wait(&empty[slot], (uint32_t)((i / stages) + 1) & 1u);
        const Chunk k = cur.at(t_cb, t_numel, (int)blockIdx.x + i * G, chunk);
        if (vec_ok(k)) {
          const uint32_t bytes = (uint32_t)(k.n & ~3) * 4u;
          float* st = slots + (size_t)slot * stage_floats;
          mbar_arrive_expect_tx(&full[slot], bytes * (uint32_t)nin);
          for (int s = 0; s < nsrc; ++s) bulk_load(st + (size_t)s * chunk, gsrc(s, k), bytes, &full[slot]);
          bulk_load(st + (size_t)nsrc * chunk, t_param[k.seg] + k.e0, bytes, &full[slot]);
          if (kMom) bulk_load(st + (size_t)(nsrc + 1) * chunk, t_mom[k.seg] + k.e0, bytes, &full[slot]);
        } else {
          mbar_arrive(&full[slot]);
        }
      }
    }
    return;
  }

  const Rule r = make_rule(a.h, kMom);
  const int ctid = threadIdx.x - 32;
  for (int i = 0; i < my_n; ++i) {
    const int slot = i % stages;
    const Chunk k = cur.at(t_cb, t_numel, (int)blockIdx.x + i * G, chunk);
    const int n4 = vec_ok(k) ? (k.n & ~3) : 0;
    const float* st = slots + (size_t)slot * stage_floats;
    const float* sp = st + (size_t)nsrc * chunk;
    const float* sm = sp + chunk;
    float* p = t_param[k.seg] + k.e0;
    float* m = kMom ? t_mom[k.seg] + k.e0 : nullptr;
    float* snap = snap_ptr(k);
    mbar_wait(&full[slot], (uint32_t)(i / stages) & 1u);
    if (debug == 2) { __syncwarp(); if (lane == 0) mbar_arrive(&empty[slot]); continue; }
    for (int e4 = ctid * 4; e4 < n4; e4 += kConsumers * 4) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < nsrc; ++s) {
        const float4 g = *(const float4*)(st + (size_t)s * chunk + e4);
        acc.x = __fadd_rn(acc.x, g.x); acc.y = __fadd_rn(acc.y, g.y);
        acc.z = __fadd_rn(acc.z, g.z); acc.w = __fadd_rn(acc.w, g.w);
      }
      float4 pv = *(const float4*)(sp + e4);
      float4 mv = kMom ? *(const float4*)(sm + e4) : make_float4(0.f, 0.f, 0.f, 0.f);
      pv.x = sgd_elem(r, acc.x, pv.x, &mv.x);
      pv.y = sgd_elem(r, acc.y, pv.y, &mv.y);
      pv.z = sgd_elem(r, acc.z, pv.z, &mv.z);
      pv.w = sgd_elem(r, acc.w, pv.w, &mv.w);
      if (debug == 1) { if (pv.x == 12345.f && mv.x == 3.f) st_v4(p + e4, pv); continue; }
      st_v4(p + e4, pv);
      if (kMom) st_v4(m + e4, mv);
      if (snap) st_v4(snap + e4, pv);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);           // stage may be refilled
    for (int e = n4 + ctid; e < k.n; e += kConsumers) {  // tail / misaligned: global memory
      float acc = 0.0f;
      for (int s = 0; s < nsrc; ++s) acc = __fadd_rn(acc, gsrc(s, k)[e]);
      float b = kMom ? m[e] : 0.0f;
      const float np = sgd_elem(r, acc, p[e], &b);
      p[e] = np;
      if (kMom) m[e] = b;
      if (snap) snap[e] = np;
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

template <typename K>
static cudaError_t opt_in_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// experiment knobs (cs_tune); 0 = built-in heuristics
int g_tune_k1_chunk = 0, g_tune_k2_chunk = 0, g_tune_k2_stages = 0, g_tune_ctas_per_sm = 0;
int g_tune_k2_debug = 0;

int tma_pack_chunk() { return g_tune_k1_chunk ? g_tune_k1_chunk : kTmaPackChunk; }

int tma_update_chunk(int nsrc, bool mom) {
  if (g_tune_k2_chunk) return g_tune_k2_chunk;
  const int nin = nsrc + 1 + (mom ? 1 : 0);
  int chunk = kTmaMaxChunk;
  while (chunk > 512 && (size_t)nin * chunk * 4 * kTmaMinStages >
                           (size_t)(kTmaSmemBudget - kTmaBarrierBytes) - update_table_bytes(kCapLarge))
    chunk >>= 1;
  return chunk;
}

static int tma_grid(int total) {
  const int g = sm_count() * (g_tune_ctas_per_sm > 0 ? g_tune_ctas_per_sm : 1);
  return total < g ? total : g;
}

static int budget() {
  return g_tune_ctas_per_sm > 1 ? kTmaSmemBudget / g_tune_ctas_per_sm : kTmaSmemBudget;
}

template <int CAP>
cudaError_t launch_pack_tma(const PackArgs<CAP>& a, cudaStream_t s) {
  if (a.total_chunks == 0) return cudaSuccess;
  const int chunk = tma_pack_chunk();
  const int table = (int)pack_table_bytes(a.n);
  int stages = (budget() - kTmaBarrierBytes - table) / (chunk * 4);
  if (stages > kTmaMaxStages) stages = kTmaMaxStages;
  if (stages < 2) return cudaErrorInvalidConfiguration;
  const int smem = kTmaBarrierBytes + table + stages * chunk * 4;
  cudaError_t e = opt_in_smem(pack_tma_kernel<CAP>, smem);
  if (e != cudaSuccess) return e;
  const int grid = tma_grid(a.total_chunks);
  pack_tma_kernel<CAP><<<grid, kThreads, smem, s>>>(a, chunk, stages);
  return cudaGetLastError();
}

template <int CAP>
cudaError_t launch_unpack_sgd_tma(const UpdateArgs<CAP>& a, bool mom, cudaStream_t s) {
  if (a.total_chunks == 0) return cudaSuccess;
  const int chunk = tma_update_chunk(a.nsrc, mom);
  const int nin = a.nsrc + 1 + (mom ? 1 : 0);
  const int table = (int)update_table_bytes(a.n);
  int stages = (budget() - kTmaBarrierBytes - table) / (nin * chunk * 4);
  if (stages > kTmaMaxStages) stages = kTmaMaxStages;
  if (g_tune_k2_stages && g_tune_k2_stages < stages) stages = g_tune_k2_stages;
  if (stages < 2) return cudaErrorInvalidConfiguration;
  const int smem = kTmaBarrierBytes + table + stages * nin * chunk * 4;
  const int grid = tma_grid(a.total_chunks);
  cudaError_t e;
  if (mom) {
    e = opt_in_smem(unpack_sgd_tma_kernel<CAP, true>, smem);
    if (e != cudaSuccess) return e;
    unpack_sgd_tma_kernel<CAP, true><<<grid, kTmaWsThreads, smem, s>>>(a, chunk, stages, g_tune_k2_debug);
  } else {
    e = opt_in_smem(unpack_sgd_tma_kernel<CAP, false>, smem);
    if (e != cudaSuccess) return e;
    unpack_sgd_tma_kernel<CAP, false><<<grid, kTmaWsThreads, smem, s>>>(a, chunk, stages, g_tune_k2_debug);
  }
  return cudaGetLastError();
}

template cudaError_t launch_pack_tma<kCapSmall>(const PackArgs<kCapSmall>&, cudaStream_t);
template cudaError_t launch_pack_tma<kCapMid>(const PackArgs<kCapMid>&, cudaStream_t);
template cudaError_t launch_pack_tma<kCapLarge>(const PackArgs<kCapLarge>&, cudaStream_t);
template cudaError_t launch_unpack_sgd_tma<kCapSmall>(const UpdateArgs<kCapSmall>&, bool, cudaStream_t);
template cudaError_t launch_unpack_sgd_tma<kCapMid>(const UpdateArgs<kCapMid>&, bool, cudaStream_t);
template cudaError_t launch_unpack_sgd_tma<kCapLarge>(const UpdateArgs<kCapLarge>&, bool, cudaStream_t);

}  // namespace cs
