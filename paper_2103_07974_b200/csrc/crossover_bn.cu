// crossover_bn.cu -- channels_last (NHWC) BatchNorm2d training kernels for the apps' compute.
//
// The ResNet-50 iteration the crossover step overlaps is ~51 % PyTorch channels_last BatchNorm
// kernels (profiles/r01_launches.md) running several times below the HBM roofline.  These four
// streaming kernels replace them (bf16 activations, fp32 weight / bias / statistics):
//
//   bn_reduce   (fwd)  per-channel (count, mean, M2) over the M = N*H*W rows, Welford per thread,
//                      Chan merge across the CTA and -- in the last CTA of each channel tile --
//                      across CTAs in fixed order (deterministic); writes mean, invstd, updates
//                      running_mean / running_var (unbiased), and the affine scale / shift.
//   bn_apply    (fwd)  y = x * scale + shift                                   (one read, one write)
//   bn_reduce   (bwd)  per-channel sum(dy), sum(dy * (x - mean)); the last CTA writes grad_weight,
//                      grad_bias and the three per-channel coefficients of dx
//   bn_apply    (bwd)  dx = dy * k1 + x * k2 + k3                              (two reads, one write)
//
// Layout: row r, channel c at x[r * C + c]; every thread owns 8 consecutive channels (one 16-byte
// bf16x8 access), C must be a multiple of 8.  Grid: x = row blocks, y = channel tiles.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"

namespace cs {

namespace {

constexpr int kBnThreads = 256;
constexpr int kBnMaxTile = 256;   // channels per CTA tile

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ uint4 ld_nc16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Chan et al. merge of (n, mean, m2) statistics
__device__ __forceinline__ void chan_merge(float& n, float& mean, float& m2, float nb, float meanb,
                                           float m2b) {
  if (nb == 0.f) return;
  const float nt = n + nb;
  const float delta = meanb - mean;
  const float fb = nb / nt;
  mean = mean + delta * fb;
  m2 = m2 + m2b + delta * delta * n * fb;
  n = nt;
}

struct TileShape {
  int tile;   // channels per CTA
  int tx;     // threads across channels (tile / 8)
  int ty;     // row lanes per CTA (256 / tx)
};

__host__ __device__ inline TileShape tile_shape(int C) {
  TileShape s;
  s.tile = C < kBnMaxTile ? C : kBnMaxTile;
  s.tx = s.tile / 8;
  s.ty = kBnThreads / s.tx;
  return s;
}

}  // namespace

// ---------------------------------------------------------------------------
// forward statistics
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBnThreads)
bn_fwd_reduce_kernel(const __nv_bfloat16* __restrict__ x, int64_t M, int C,
                     const float* __restrict__ weight, const float* __restrict__ bias,
                     float* __restrict__ running_mean, float* __restrict__ running_var,
                     float momentum, float eps, float* __restrict__ save_mean,
                     float* __restrict__ save_invstd, float* __restrict__ scale,
                     float* __restrict__ shift, float* __restrict__ partial,
                     unsigned int* __restrict__ tickets) {
  const TileShape s = tile_shape(C);
  const int tx = threadIdx.x % s.tx, ty = threadIdx.x / s.tx;
  const int c0 = blockIdx.y * s.tile + tx * 8;
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;

  float n = 0.f, mean[8], m2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { mean[i] = 0.f; m2[i] = 0.f; }
  for (int64_t r = r0 + ty; r < r1; r += s.ty) {
    float v[8];
    unpack8(ld_nc16(x + r * C + c0), v);
    n += 1.f;
    const float inv = 1.0f / n;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float d = v[i] - mean[i];
      mean[i] += d * inv;
      m2[i] += d * (v[i] - mean[i]);
    }
  }
  // merge the ty row lanes of every channel through shared memory (fixed order)
  __shared__ float s_n[kBnThreads], s_mean[kBnThreads * 8], s_m2[kBnThreads * 8];
  s_n[threadIdx.x] = n;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s_mean[threadIdx.x * 8 + i] = mean[i];
    s_m2[threadIdx.x * 8 + i] = m2[i];
  }
  __syncthreads();
  if (ty == 0) {
    for (int k = 1; k < s.ty; ++k) {
      const int t = k * s.tx + tx;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float nn = n, mm = mean[i], qq = m2[i];
        chan_merge(nn, mm, qq, s_n[t], s_mean[t * 8 + i], s_m2[t * 8 + i]);
        mean[i] = mm;
        m2[i] = qq;
      }
      n += s_n[t];
    }
    float* out = partial + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * (size_t)s.tile * 3;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      out[(tx * 8 + i) * 3 + 0] = n;
      out[(tx * 8 + i) * 3 + 1] = mean[i];
      out[(tx * 8 + i) * 3 + 2] = m2[i];
    }
  }
  // last CTA of this channel tile merges all row blocks in order
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&tickets[blockIdx.y], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // parallel fixed-order merge: L = 256 / tile lanes per channel, then the lanes in order
  {
    const int L = kBnThreads / s.tile;
    const int c = threadIdx.x % s.tile, lane = threadIdx.x / s.tile;
    float nt = 0.f, mt = 0.f, qt = 0.f;
    for (unsigned b = lane; b < gridDim.x; b += L) {
      const float* p = partial + ((size_t)blockIdx.y * gridDim.x + b) * (size_t)s.tile * 3 + (size_t)c * 3;
      chan_merge(nt, mt, qt, __ldcg(p), __ldcg(p + 1), __ldcg(p + 2));
    }
    __syncthreads();                       // s_n / s_mean / s_m2 are free again
    s_n[threadIdx.x] = nt;
    s_mean[threadIdx.x] = mt;
    s_m2[threadIdx.x] = qt;
    __syncthreads();
    if (lane == 0) {
      for (int l = 1; l < L; ++l) {
        const int t = l * s.tile + c;
        chan_merge(nt, mt, qt, s_n[t], s_mean[t], s_m2[t]);
      }
      const int ch = blockIdx.y * s.tile + c;
      const float var = qt / nt;
      const float invstd = rsqrtf(var + eps);
      save_mean[ch] = mt;
      save_invstd[ch] = invstd;
      if (running_mean != nullptr) {
        const float unbiased = nt > 1.f ? qt / (nt - 1.f) : var;
        running_mean[ch] = (1.f - momentum) * running_mean[ch] + momentum * mt;
        running_var[ch] = (1.f - momentum) * running_var[ch] + momentum * unbiased;
      }
      const float w = weight != nullptr ? weight[ch] : 1.f;
      const float b = bias != nullptr ? bias[ch] : 0.f;
      scale[ch] = invstd * w;
      shift[ch] = b - mt * invstd * w;
    }
  }
  if (threadIdx.x == 0) tickets[blockIdx.y] = 0u;
}

// y = x * scale + shift  (also the backward elementwise: dx = dy * k1 + x * k2 + k3)
template <bool kBwd>
__global__ void __launch_bounds__(kBnThreads)
bn_apply_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                int64_t M, int C, const float* __restrict__ k1, const float* __restrict__ k2,
                const float* __restrict__ k3, __nv_bfloat16* __restrict__ out) {
  const int64_t vecs = M * (C / 8);
  const int cv = C / 8;
  for (int64_t v = (int64_t)blockIdx.x * kBnThreads + threadIdx.x; v < vecs;
       v += (int64_t)gridDim.x * kBnThreads) {
    const int c = (int)(v % cv) * 8;
    float fa[8], o[8];
    unpack8(ld_nc16(a + v * 8), fa);
    if (kBwd) {
      float fb[8];
      unpack8(ld_nc16(b + v * 8), fb);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = fmaf(fa[i], k1[c + i], fmaf(fb[i], k2[c + i], k3[c + i]));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = fmaf(fa[i], k1[c + i], k2[c + i]);
    }
    *reinterpret_cast<uint4*>(out + v * 8) = pack8(o);
  }
}

// ---------------------------------------------------------------------------
// backward reduction: sum(dy), sum(dy * (x - mean)) per channel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBnThreads)
bn_bwd_reduce_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                     int64_t M, int C, const float* __restrict__ save_mean,
                     const float* __restrict__ save_invstd, const float* __restrict__ weight,
                     float* __restrict__ grad_weight, float* __restrict__ grad_bias,
                     float* __restrict__ k1, float* __restrict__ k2, float* __restrict__ k3,
                     float* __restrict__ partial, unsigned int* __restrict__ tickets) {
  const TileShape s = tile_shape(C);
  const int tx = threadIdx.x % s.tx, ty = threadIdx.x / s.tx;
  const int c0 = blockIdx.y * s.tile + tx * 8;
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float mu[8], sdy[8], sdx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { mu[i] = save_mean[c0 + i]; sdy[i] = 0.f; sdx[i] = 0.f; }
  for (int64_t r = r0 + ty; r < r1; r += s.ty) {
    float g[8], v[8];
    unpack8(ld_nc16(dy + r * C + c0), g);
    unpack8(ld_nc16(x + r * C + c0), v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sdy[i] += g[i];
      sdx[i] = fmaf(g[i], v[i] - mu[i], sdx[i]);
    }
  }
  __shared__ float s_dy[kBnThreads * 8], s_dx[kBnThreads * 8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s_dy[threadIdx.x * 8 + i] = sdy[i];
    s_dx[threadIdx.x * 8 + i] = sdx[i];
  }
  __syncthreads();
  if (ty == 0) {
    for (int k = 1; k < s.ty; ++k) {
      const int t = k * s.tx + tx;
#pragma unroll
      for (int i = 0; i < 8; ++i) { sdy[i] += s_dy[t * 8 + i]; sdx[i] += s_dx[t * 8 + i]; }
    }
    float* out = partial + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * (size_t)s.tile * 2;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      out[(tx * 8 + i) * 2 + 0] = sdy[i];
      out[(tx * 8 + i) * 2 + 1] = sdx[i];
    }
  }
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&tickets[blockIdx.y], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  {
    const int L = kBnThreads / s.tile;
    const int c = threadIdx.x % s.tile, lane = threadIdx.x / s.tile;
    float a = 0.f, b = 0.f;
    for (unsigned blk = lane; blk < gridDim.x; blk += L) {
      const float* p = partial + ((size_t)blockIdx.y * gridDim.x + blk) * (size_t)s.tile * 2 + (size_t)c * 2;
      a += __ldcg(p);
      b += __ldcg(p + 1);
    }
    __syncthreads();
    s_dy[threadIdx.x] = a;
    s_dx[threadIdx.x] = b;
    __syncthreads();
    if (lane == 0) {
      for (int l = 1; l < L; ++l) {
        a += s_dy[l * s.tile + c];
        b += s_dx[l * s.tile + c];
      }
      const int ch = blockIdx.y * s.tile + c;
      const float invstd = save_invstd[ch];
      const float w = weight != nullptr ? weight[ch] : 1.f;
      if (grad_bias != nullptr) grad_bias[ch] = a;
      if (grad_weight != nullptr) grad_weight[ch] = b * invstd;
      const float inv_m = 1.0f / (float)M;
      const float kk1 = invstd * w;
      const float kk2 = -invstd * invstd * invstd * w * b * inv_m;
      k1[ch] = kk1;
      k2[ch] = kk2;
      k3[ch] = -kk1 * a * inv_m - kk2 * save_mean[ch];
    }
  }
  if (threadIdx.x == 0) tickets[blockIdx.y] = 0u;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int sm_count_bn() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

int bn_row_blocks(int64_t M, int C) {
  const TileShape s = tile_shape(C);
  const int tiles = C / s.tile;
  int64_t want = (int64_t)sm_count_bn() * 4 / tiles;        // ~4 CTAs per SM in total
  const int64_t max_by_rows = (M + s.ty * 16 - 1) / (s.ty * 16);  // >= 16 rows per row lane
  if (want > max_by_rows) want = max_by_rows;
  if (want < 1) want = 1;
  return (int)want;
}

size_t bn_workspace_bytes(int64_t M, int C) {
  const int tiles = C / tile_shape(C).tile;
  return 256 + (size_t)bn_row_blocks(M, C) * (size_t)C * 3 * sizeof(float) + (size_t)tiles * 0;
}

cudaError_t launch_bn_fwd(const void* x, int64_t M, int C, const float* w, const float* b,
                          float* rm, float* rv, float momentum, float eps, float* save_mean,
                          float* save_invstd, float* scale_shift, void* y, void* ws,
                          cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const dim3 grid(bn_row_blocks(M, C), C / sh.tile);
  unsigned int* tickets = (unsigned int*)ws;
  float* partial = (float*)((char*)ws + 256);
  float* scale = scale_shift;
  float* shift = scale_shift + C;
  bn_fwd_reduce_kernel<<<grid, kBnThreads, 0, s>>>((const __nv_bfloat16*)x, M, C, w, b, rm, rv,
                                                   momentum, eps, save_mean, save_invstd, scale,
                                                   shift, partial, tickets);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t vecs = M * (C / 8);
  int64_t g = (vecs + kBnThreads - 1) / kBnThreads;
  const int64_t cap = (int64_t)sm_count_bn() * 8;
  if (g > cap) g = cap;
  bn_apply_kernel<false><<<(unsigned)g, kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)x, nullptr, M, C, scale, shift, nullptr, (__nv_bfloat16*)y);
  return cudaGetLastError();
}

cudaError_t launch_bn_bwd(const void* dy, const void* x, int64_t M, int C, const float* save_mean,
                          const float* save_invstd, const float* w, float* gw, float* gb,
                          float* coef, void* dx, void* ws, cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const dim3 grid(bn_row_blocks(M, C), C / sh.tile);
  unsigned int* tickets = (unsigned int*)ws;
  float* partial = (float*)((char*)ws + 256);
  bn_bwd_reduce_kernel<<<grid, kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, M, C, save_mean, save_invstd, w, gw, gb,
      coef, coef + C, coef + 2 * C, partial, tickets);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t vecs = M * (C / 8);
  int64_t g = (vecs + kBnThreads - 1) / kBnThreads;
  const int64_t cap = (int64_t)sm_count_bn() * 8;
  if (g > cap) g = cap;
  bn_apply_kernel<true><<<(unsigned)g, kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, M, C, coef, coef + C, coef + 2 * C,
      (__nv_bfloat16*)dx);
  return cudaGetLastError();
}

}  // namespace cs
