// crossover_bn.cu -- channels_last (NHWC) BatchNorm2d training kernels for the apps' compute.
//
// The ResNet-50 iteration the crossover step overlaps is ~51 % PyTorch channels_last BatchNorm
// kernels (profiles/r01_launches.md).  Six streaming kernels replace them (bf16 activations,
// fp32 weight / bias / statistics):
//
//   bn_fwd_partial   per (row block, channel tile): per-channel (count, mean, M2), Welford per
//                    thread over 4-row unrolled 16-byte loads, Chan merge across the CTA
//   bn_fwd_finalize  one warp per channel: Chan merge of all row blocks (lane-strided, then a
//                    fixed shuffle tree -> deterministic); mean, invstd, running stats (unbiased
//                    variance, nn.BatchNorm2d momentum), affine scale / shift
//   bn_apply<fwd>    y  = x * scale + shift                      (1 read + 1 write)
//   bn_bwd_partial   per-channel sum(dy), sum(dy * (x - mean))   (2 reads)
//   bn_bwd_finalize  grad_weight, grad_bias and the dx coefficients k1, k2, k3
//   bn_apply<bwd>    dx = dy * k1 + x * k2 + k3                  (2 reads + 1 write)
//
// Layout: row r, channel c at x[r * C + c]; every thread owns 8 consecutive channels (one
// 16-byte bf16x8 access); C % 8 == 0 and (C <= 256 or C % 256 == 0).  Apply kernels keep a
// thread's channel group fixed (grid stride is a multiple of C/8), so the per-channel
// coefficients are loaded once into registers.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"

namespace cs {

namespace {

constexpr int kBnThreads = 256;
constexpr int kBnMaxTile = 256;   // channels per CTA tile in the partial kernels
constexpr int kRowUnroll = 4;     // rows in flight per thread

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

__device__ __forceinline__ void welford8(const uint4& raw, float& n, float* mean, float* m2) {
  float v[8];
  unpack8(raw, v);
  n += 1.f;
  const float inv = 1.0f / n;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float d = v[i] - mean[i];
    mean[i] = fmaf(d, inv, mean[i]);
    m2[i] = fmaf(d, v[i] - mean[i], m2[i]);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// forward statistics
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBnThreads)
bn_fwd_partial_kernel(const __nv_bfloat16* __restrict__ x, int64_t M, int C,
                      float* __restrict__ partial) {
  const TileShape s = tile_shape(C);
  const int tx = threadIdx.x % s.tx, ty = threadIdx.x / s.tx;
  const int c0 = blockIdx.y * s.tile + tx * 8;
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;

  float n = 0.f, mean[8], m2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { mean[i] = 0.f; m2[i] = 0.f; }
  int64_t r = r0 + ty;
  for (; r + (kRowUnroll - 1) * s.ty < r1; r += kRowUnroll * s.ty) {
    uint4 raw[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) raw[u] = ld_nc16(x + (r + u * s.ty) * C + c0);
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) welford8(raw[u], n, mean, m2);
  }
  for (; r < r1; r += s.ty) welford8(ld_nc16(x + r * C + c0), n, mean, m2);

  // merge the ty row lanes of every channel (fixed order)
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
      const float nb = s_n[t];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float nn = n, mm = mean[i], qq = m2[i];
        chan_merge(nn, mm, qq, nb, s_mean[t * 8 + i], s_m2[t * 8 + i]);
        mean[i] = mm;
        m2[i] = qq;
      }
      n += nb;
    }
    // partial layout: [channel][row block][3]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float* out = partial + ((size_t)(c0 + i) * gridDim.x + blockIdx.x) * 3;
      out[0] = n;
      out[1] = mean[i];
      out[2] = m2[i];
    }
  }
}

// one warp per channel: lane-strided Chan merge, then a fixed shuffle tree
__global__ void __launch_bounds__(kBnThreads)
bn_fwd_finalize_kernel(const float* __restrict__ partial, int blocks, int C,
                       const float* __restrict__ weight, const float* __restrict__ bias,
                       float* __restrict__ running_mean, float* __restrict__ running_var,
                       float momentum, float eps, float* __restrict__ save_mean,
                       float* __restrict__ save_invstd, float* __restrict__ scale,
                       float* __restrict__ shift) {
  const int ch = blockIdx.x * (kBnThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ch >= C) return;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  for (int b = lane; b < blocks; b += 32) {
    const float* p = partial + ((size_t)ch * blocks + b) * 3;
    chan_merge(n, mean, m2, p[0], p[1], p[2]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float nb = __shfl_down_sync(0xffffffffu, n, o);
    const float mb = __shfl_down_sync(0xffffffffu, mean, o);
    const float qb = __shfl_down_sync(0xffffffffu, m2, o);
    chan_merge(n, mean, m2, nb, mb, qb);
  }
  if (lane == 0) {
    const float var = m2 / n;
    const float invstd = rsqrtf(var + eps);
    save_mean[ch] = mean;
    save_invstd[ch] = invstd;
    if (running_mean != nullptr) {
      const float unbiased = n > 1.f ? m2 / (n - 1.f) : var;
      running_mean[ch] = (1.f - momentum) * running_mean[ch] + momentum * mean;
      running_var[ch] = (1.f - momentum) * running_var[ch] + momentum * unbiased;
    }
    const float w = weight != nullptr ? weight[ch] : 1.f;
    const float b = bias != nullptr ? bias[ch] : 0.f;
    scale[ch] = invstd * w;
    shift[ch] = b - mean * invstd * w;
  }
}

template <bool kBwd>
__device__ __forceinline__ uint4 apply8(const uint4& ra, const uint4& rb, const float* q1,
                                        const float* q2, const float* q3) {
  float fa[8], o[8];
  unpack8(ra, fa);
  if (kBwd) {
    float fb[8];
    unpack8(rb, fb);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = fmaf(fa[i], q1[i], fmaf(fb[i], q2[i], q3[i]));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = fmaf(fa[i], q1[i], q2[i]);
  }
  return pack8(o);
}

// y = x * scale + shift  |  dx = dy * k1 + x * k2 + k3
template <bool kBwd>
__global__ void __launch_bounds__(kBnThreads)
bn_apply_kernel(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b,
                int64_t M, int C, const float* __restrict__ k1, const float* __restrict__ k2,
                const float* __restrict__ k3, __nv_bfloat16* __restrict__ out) {
  const int64_t vecs = M * (C / 8);
  const int cv = C / 8;
  const int64_t stride = (int64_t)gridDim.x * kBnThreads;   // multiple of cv (host guarantees)
  const int64_t v0 = (int64_t)blockIdx.x * kBnThreads + threadIdx.x;
  const int c = (int)(v0 % cv) * 8;
  float q1[8], q2[8], q3[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    q1[i] = k1[c + i];
    q2[i] = k2[c + i];
    q3[i] = kBwd ? k3[c + i] : 0.f;
  }
  const uint4 zero = make_uint4(0, 0, 0, 0);
  int64_t v = v0;
  for (; v + stride < vecs; v += 2 * stride) {
    const uint4 ra0 = ld_nc16(a + v * 8), ra1 = ld_nc16(a + (v + stride) * 8);
    const uint4 rb0 = kBwd ? ld_nc16(b + v * 8) : zero;
    const uint4 rb1 = kBwd ? ld_nc16(b + (v + stride) * 8) : zero;
    *reinterpret_cast<uint4*>(out + v * 8) = apply8<kBwd>(ra0, rb0, q1, q2, q3);
    *reinterpret_cast<uint4*>(out + (v + stride) * 8) = apply8<kBwd>(ra1, rb1, q1, q2, q3);
  }
  for (; v < vecs; v += stride) {
    const uint4 ra = ld_nc16(a + v * 8);
    const uint4 rb = kBwd ? ld_nc16(b + v * 8) : zero;
    *reinterpret_cast<uint4*>(out + v * 8) = apply8<kBwd>(ra, rb, q1, q2, q3);
  }
}

// ---------------------------------------------------------------------------
// backward: sum(dy), sum(dy * (x - mean)) per channel
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bwd_acc8(const uint4& rg, const uint4& rx, const float* mu,
                                         float* sdy, float* sdx) {
  float g[8], v[8];
  unpack8(rg, g);
  unpack8(rx, v);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sdy[i] += g[i];
    sdx[i] = fmaf(g[i], v[i] - mu[i], sdx[i]);
  }
}

__global__ void __launch_bounds__(kBnThreads)
bn_bwd_partial_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                      int64_t M, int C, const float* __restrict__ save_mean,
                      float* __restrict__ partial) {
  const TileShape s = tile_shape(C);
  const int tx = threadIdx.x % s.tx, ty = threadIdx.x / s.tx;
  const int c0 = blockIdx.y * s.tile + tx * 8;
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float mu[8], sdy[8], sdx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { mu[i] = save_mean[c0 + i]; sdy[i] = 0.f; sdx[i] = 0.f; }
  int64_t r = r0 + ty;
  for (; r + (kRowUnroll - 1) * s.ty < r1; r += kRowUnroll * s.ty) {
    uint4 rg[kRowUnroll], rx[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      rg[u] = ld_nc16(dy + (r + u * s.ty) * C + c0);
      rx[u] = ld_nc16(x + (r + u * s.ty) * C + c0);
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) bwd_acc8(rg[u], rx[u], mu, sdy, sdx);
  }
  for (; r < r1; r += s.ty) bwd_acc8(ld_nc16(dy + r * C + c0), ld_nc16(x + r * C + c0), mu, sdy, sdx);

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
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float* out = partial + ((size_t)(c0 + i) * gridDim.x + blockIdx.x) * 2;
      out[0] = sdy[i];
      out[1] = sdx[i];
    }
  }
}

__global__ void __launch_bounds__(kBnThreads)
bn_bwd_finalize_kernel(const float* __restrict__ partial, int blocks, int64_t M, int C,
                       const float* __restrict__ save_mean, const float* __restrict__ save_invstd,
                       const float* __restrict__ weight, float* __restrict__ grad_weight,
                       float* __restrict__ grad_bias, float* __restrict__ k1,
                       float* __restrict__ k2, float* __restrict__ k3) {
  const int ch = blockIdx.x * (kBnThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ch >= C) return;
  float a = 0.f, b = 0.f;
  for (int blk = lane; blk < blocks; blk += 32) {
    const float* p = partial + ((size_t)ch * blocks + blk) * 2;
    a += p[0];
    b += p[1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
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
  int64_t want = (int64_t)sm_count_bn() * 6 / tiles;                              // ~6 CTAs / SM
  const int64_t max_by_rows = (M + s.ty * 4 * kRowUnroll - 1) / (s.ty * 4 * kRowUnroll);
  if (want > max_by_rows) want = max_by_rows;
  if (want < 1) want = 1;
  return (int)want;
}

size_t bn_workspace_bytes(int64_t M, int C) {
  return 256 + (size_t)bn_row_blocks(M, C) * (size_t)C * 3 * sizeof(float);
}

static unsigned apply_grid(int64_t M, int C) {
  const int64_t vecs = M * (C / 8);
  const int cv = C / 8;
  int64_t g = (vecs + kBnThreads - 1) / kBnThreads;
  const int64_t cap = (int64_t)sm_count_bn() * 8;
  if (g > cap) g = cap;
  // grid * 256 must be a multiple of C/8 so a thread's channel group never changes
  if (cv > kBnThreads) {
    const int64_t m = cv / kBnThreads;
    g = (g + m - 1) / m * m;
  }
  return (unsigned)(g < 1 ? 1 : g);
}

cudaError_t launch_bn_fwd(const void* x, int64_t M, int C, const float* w, const float* b,
                          float* rm, float* rv, float momentum, float eps, float* save_mean,
                          float* save_invstd, float* scale_shift, void* y, void* ws,
                          cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const int blocks = bn_row_blocks(M, C);
  float* partial = (float*)((char*)ws + 256);
  bn_fwd_partial_kernel<<<dim3(blocks, C / sh.tile), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)x, M, C, partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  float* scale = scale_shift;
  float* shift = scale_shift + C;
  bn_fwd_finalize_kernel<<<(C + 7) / 8, kBnThreads, 0, s>>>(partial, blocks, C, w, b, rm, rv,
                                                             momentum, eps, save_mean, save_invstd,
                                                             scale, shift);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  bn_apply_kernel<false><<<apply_grid(M, C), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)x, nullptr, M, C, scale, shift, nullptr, (__nv_bfloat16*)y);
  return cudaGetLastError();
}

cudaError_t launch_bn_bwd(const void* dy, const void* x, int64_t M, int C, const float* save_mean,
                          const float* save_invstd, const float* w, float* gw, float* gb,
                          float* coef, void* dx, void* ws, cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const int blocks = bn_row_blocks(M, C);
  float* partial = (float*)((char*)ws + 256);
  bn_bwd_partial_kernel<<<dim3(blocks, C / sh.tile), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, M, C, save_mean, partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  bn_bwd_finalize_kernel<<<(C + 7) / 8, kBnThreads, 0, s>>>(partial, blocks, M, C, save_mean,
                                                             save_invstd, w, gw, gb, coef,
                                                             coef + C, coef + 2 * C);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  bn_apply_kernel<true><<<apply_grid(M, C), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, M, C, coef, coef + C, coef + 2 * C,
      (__nv_bfloat16*)dx);
  return cudaGetLastError();
}

}  // namespace cs
