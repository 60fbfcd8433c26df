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

int g_tune_bn_no_pdl = 0;   // 0: finalize / apply use programmatic dependent launch
int g_tune_bn_ctas_per_sm = 0;   // partial kernels: row-block CTAs per SM (0 = 3, the measured best)

namespace {

constexpr int kBnThreads = 256;

// Programmatic dependent launch (PDL) inside a BN op: finalize and apply are launched with
// programmatic stream serialization, so their CTAs are scheduled while the previous kernel of
// the chain drains; griddepcontrol.wait then blocks until that kernel has completed and its
// writes are visible (the ordering is unchanged, only the launch latency is hidden).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
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

// Shifted sums: per thread, s1 = sum(x - k), s2 = sum((x - k)^2) with k = the thread's first
// value of each channel (2 FMA-class ops per element instead of a Welford update); converted to
// (n, mean, M2) before the Chan merges.  |mean - k| ~ std for BN inputs, so s2 - s1^2/n keeps
// its precision.
__device__ __forceinline__ void shifted8(const uint4& raw, const float* k, float* s1, float* s2) {
  float v[8];
  unpack8(raw, v);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float d = v[i] - k[i];
    s1[i] += d;
    s2[i] = fmaf(d, d, s2[i]);
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

  constexpr int U = 2 * kRowUnroll;
  float k[8], s1[8], s2[8], mean[8], m2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { k[i] = 0.f; s1[i] = 0.f; s2[i] = 0.f; }
  int64_t r = r0 + ty;
  if (r < r1) unpack8(ld_nc16(x + r * C + c0), k);   // the shift
  for (; r + (U - 1) * s.ty < r1; r += U * s.ty) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) raw[u] = ld_nc16(x + (r + u * s.ty) * C + c0);
#pragma unroll
    for (int u = 0; u < U; ++u) shifted8(raw[u], k, s1, s2);
  }
  for (; r < r1; r += s.ty) shifted8(ld_nc16(x + r * C + c0), k, s1, s2);
  pdl_trigger();
  const int64_t my_rows = r1 > r0 + ty ? (r1 - (r0 + ty) + s.ty - 1) / s.ty : 0;
  float n = (float)my_rows;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float mu = n > 0.f ? s1[i] / n : 0.f;
    mean[i] = k[i] + mu;
    m2[i] = n > 0.f ? fmaxf(s2[i] - s1[i] * mu, 0.f) : 0.f;
  }

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
  pdl_trigger();
  pdl_wait();
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

// Fused epilogues: kRelu = max(., 0) after the affine map, kRes = + residual before it.
template <bool kRelu, bool kRes>
__device__ __forceinline__ void pre_act8(const uint4& rx, const uint4& rr, const float* sc,
                                         const float* sh, float* pre) {
  float fx[8];
  unpack8(rx, fx);
  if (kRes) {
    float fr[8];
    unpack8(rr, fr);
#pragma unroll
    for (int i = 0; i < 8; ++i) pre[i] = fmaf(fx[i], sc[i], sh[i]) + fr[i];
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) pre[i] = fmaf(fx[i], sc[i], sh[i]);
  }
}

// y = act(x * scale + shift [+ residual])
template <bool kRelu, bool kRes>
__global__ void __launch_bounds__(kBnThreads)
bn_fwd_apply_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ res,
                    int64_t M, int C, const float* __restrict__ scale,
                    const float* __restrict__ shift, __nv_bfloat16* __restrict__ y) {
  const int64_t vecs = M * (C / 8);
  const int cv = C / 8;
  const int64_t stride = (int64_t)gridDim.x * kBnThreads;   // multiple of cv (host guarantees)
  const int64_t v0 = (int64_t)blockIdx.x * kBnThreads + threadIdx.x;
  const int c = (int)(v0 % cv) * 8;
  pdl_wait();
  float sc[8], sh[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { sc[i] = scale[c + i]; sh[i] = shift[c + i]; }
  const uint4 zero = make_uint4(0, 0, 0, 0);
  int64_t v = v0;
  for (; v + stride < vecs; v += 2 * stride) {
    const uint4 rx0 = ld_nc16(x + v * 8), rx1 = ld_nc16(x + (v + stride) * 8);
    const uint4 rr0 = kRes ? ld_nc16(res + v * 8) : zero;
    const uint4 rr1 = kRes ? ld_nc16(res + (v + stride) * 8) : zero;
    float p[8];
    pre_act8<kRelu, kRes>(rx0, rr0, sc, sh, p);
    if (kRelu) for (int i = 0; i < 8; ++i) p[i] = fmaxf(p[i], 0.f);
    *reinterpret_cast<uint4*>(y + v * 8) = pack8(p);
    pre_act8<kRelu, kRes>(rx1, rr1, sc, sh, p);
    if (kRelu) for (int i = 0; i < 8; ++i) p[i] = fmaxf(p[i], 0.f);
    *reinterpret_cast<uint4*>(y + (v + stride) * 8) = pack8(p);
  }
  for (; v < vecs; v += stride) {
    const uint4 rx = ld_nc16(x + v * 8);
    const uint4 rr = kRes ? ld_nc16(res + v * 8) : zero;
    float p[8];
    pre_act8<kRelu, kRes>(rx, rr, sc, sh, p);
    if (kRelu) for (int i = 0; i < 8; ++i) p[i] = fmaxf(p[i], 0.f);
    *reinterpret_cast<uint4*>(y + v * 8) = pack8(p);
  }
}

// g = dy [+ dy2] masked by the forward activation (recomputed from x [, residual]; nothing
// stored).  kDy2: a second gradient of the same output delivered outside autograd (the next
// bottleneck block's identity path) is summed in fp32 instead of by a separate add kernel.
template <bool kRelu, bool kRes, bool kDy2>
__device__ __forceinline__ void masked_grad8(const uint4& rg, const uint4& rg2, const uint4& rx,
                                             const uint4& rr, const float* sc, const float* sh,
                                             float* g) {
  unpack8(rg, g);
  if (kDy2) {
    float g2[8];
    unpack8(rg2, g2);
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] += g2[i];
  }
  if (kRelu) {
    float p[8];
    pre_act8<kRelu, kRes>(rx, rr, sc, sh, p);
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = p[i] > 0.f ? g[i] : 0.f;
  }
}

// dx = g * k1 + x * k2 + k3 ; dres = g (kRes)
template <bool kRelu, bool kRes, bool kDy2>
__global__ void __launch_bounds__(kBnThreads)
bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dy2,
                    const __nv_bfloat16* __restrict__ x,
                    const __nv_bfloat16* __restrict__ res, int64_t M, int C,
                    const float* __restrict__ coef, const float* __restrict__ scale,
                    const float* __restrict__ shift, __nv_bfloat16* __restrict__ dx,
                    __nv_bfloat16* __restrict__ dres) {
  const int64_t vecs = M * (C / 8);
  const int cv = C / 8;
  const int64_t stride = (int64_t)gridDim.x * kBnThreads;
  const int64_t v0 = (int64_t)blockIdx.x * kBnThreads + threadIdx.x;
  const int c = (int)(v0 % cv) * 8;
  pdl_wait();
  float q1[8], q2[8], q3[8], sc[8], sh[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    q1[i] = coef[c + i];
    q2[i] = coef[C + c + i];
    q3[i] = coef[2 * C + c + i];
    sc[i] = kRelu ? scale[c + i] : 0.f;
    sh[i] = kRelu ? shift[c + i] : 0.f;
  }
  const uint4 zero = make_uint4(0, 0, 0, 0);
  for (int64_t v = v0; v < vecs; v += stride) {
    const uint4 rg = ld_nc16(dy + v * 8);
    const uint4 rg2 = kDy2 ? ld_nc16(dy2 + v * 8) : zero;
    const uint4 rx = ld_nc16(x + v * 8);
    const uint4 rr = (kRes && kRelu) ? ld_nc16(res + v * 8) : zero;
    float g[8], fx[8], o[8];
    masked_grad8<kRelu, kRes, kDy2>(rg, rg2, rx, rr, sc, sh, g);
    unpack8(rx, fx);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = fmaf(g[i], q1[i], fmaf(fx[i], q2[i], q3[i]));
    *reinterpret_cast<uint4*>(dx + v * 8) = pack8(o);
    if (kRes) *reinterpret_cast<uint4*>(dres + v * 8) = pack8(g);
  }
}

// ---------------------------------------------------------------------------
// backward: sum(dy), sum(dy * (x - mean)) per channel
// ---------------------------------------------------------------------------
template <bool kRelu, bool kRes, bool kDy2>
__device__ __forceinline__ void bwd_acc8(const uint4& rg, const uint4& rg2, const uint4& rx,
                                         const uint4& rr, const float* mu, const float* sc,
                                         const float* sh, float* sdy, float* sdx) {
  float g[8], v[8];
  masked_grad8<kRelu, kRes, kDy2>(rg, rg2, rx, rr, sc, sh, g);
  unpack8(rx, v);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sdy[i] += g[i];
    sdx[i] = fmaf(g[i], v[i] - mu[i], sdx[i]);
  }
}

template <bool kRelu, bool kRes, bool kDy2>
__global__ void __launch_bounds__(kBnThreads)
bn_bwd_partial_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dy2,
                      const __nv_bfloat16* __restrict__ x,
                      const __nv_bfloat16* __restrict__ res, int64_t M, int C,
                      const float* __restrict__ save_mean, const float* __restrict__ scale,
                      const float* __restrict__ shift, float* __restrict__ partial) {
  const TileShape s = tile_shape(C);
  const int tx = threadIdx.x % s.tx, ty = threadIdx.x / s.tx;
  const int c0 = blockIdx.y * s.tile + tx * 8;
  const int64_t rows_per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
  float mu[8], sdy[8], sdx[8], sc[8], sh[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mu[i] = save_mean[c0 + i]; sdy[i] = 0.f; sdx[i] = 0.f;
    sc[i] = kRelu ? scale[c0 + i] : 0.f;
    sh[i] = kRelu ? shift[c0 + i] : 0.f;
  }
  const uint4 zero = make_uint4(0, 0, 0, 0);
  constexpr bool kLoadRes = kRes && kRelu;
  int64_t r = r0 + ty;
  for (; r + (kRowUnroll - 1) * s.ty < r1; r += kRowUnroll * s.ty) {
    uint4 rg[kRowUnroll], rg2[kRowUnroll], rx[kRowUnroll], rr[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      rg[u] = ld_nc16(dy + (r + u * s.ty) * C + c0);
      rg2[u] = kDy2 ? ld_nc16(dy2 + (r + u * s.ty) * C + c0) : zero;
      rx[u] = ld_nc16(x + (r + u * s.ty) * C + c0);
      rr[u] = kLoadRes ? ld_nc16(res + (r + u * s.ty) * C + c0) : zero;
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u)
      bwd_acc8<kRelu, kRes, kDy2>(rg[u], rg2[u], rx[u], rr[u], mu, sc, sh, sdy, sdx);
  }
  for (; r < r1; r += s.ty)
    bwd_acc8<kRelu, kRes, kDy2>(ld_nc16(dy + r * C + c0), kDy2 ? ld_nc16(dy2 + r * C + c0) : zero,
                                ld_nc16(x + r * C + c0), kLoadRes ? ld_nc16(res + r * C + c0) : zero,
                                mu, sc, sh, sdy, sdx);
  pdl_trigger();

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
  pdl_trigger();
  pdl_wait();
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
  // ~3 CTAs / SM: with 8 rows of 16-byte loads in flight per thread that keeps >= 64 KB per SM
  // outstanding, and halves the partials the finalize kernels must merge (vs 6 / SM)
  const int per_sm = g_tune_bn_ctas_per_sm > 0 ? g_tune_bn_ctas_per_sm : 3;
  int64_t want = (int64_t)sm_count_bn() * per_sm / tiles;
  const int64_t max_by_rows = (M + s.ty * 4 * kRowUnroll - 1) / (s.ty * 4 * kRowUnroll);
  if (want > max_by_rows) want = max_by_rows;
  if (want < 1) want = 1;
  return (int)want;
}

size_t bn_workspace_bytes(int64_t M, int C) {
  return 256 + (size_t)bn_row_blocks(M, C) * (size_t)C * 3 * sizeof(float);
}

// launch with programmatic stream serialization (cs_tune("bn_no_pdl", 1) turns it off)
template <typename... KArgs, typename... Args>
static cudaError_t launch_dependent(void (*kernel)(KArgs...), dim3 grid, cudaStream_t s,
                                    Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kBnThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_tune_bn_no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
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

template <bool kRelu, bool kRes>
static void fwd_apply(const void* x, const void* res, int64_t M, int C, const float* scale,
                      const float* shift, void* y, cudaStream_t s) {
  launch_dependent(bn_fwd_apply_kernel<kRelu, kRes>, dim3(apply_grid(M, C)), s,
                   (const __nv_bfloat16*)x, (const __nv_bfloat16*)res, M, C, scale, shift,
                   (__nv_bfloat16*)y);
}

cudaError_t launch_bn_fwd(const void* x, const void* res, int64_t M, int C, const float* w,
                          const float* b, float* rm, float* rv, float momentum, float eps,
                          float* save_mean, float* save_invstd, float* scale_shift, void* y,
                          void* ws, int flags, cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const int blocks = bn_row_blocks(M, C);
  float* partial = (float*)((char*)ws + 256);
  bn_fwd_partial_kernel<<<dim3(blocks, C / sh.tile), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)x, M, C, partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  float* scale = scale_shift;
  float* shift = scale_shift + C;
  e = launch_dependent(bn_fwd_finalize_kernel, dim3((C + 7) / 8), s, (const float*)partial, blocks,
                       C, w, b, rm, rv, momentum, eps, save_mean, save_invstd, scale, shift);
  if (e != cudaSuccess) return e;
  const bool relu = flags & CS_BN_RELU, resid = flags & CS_BN_RESIDUAL;
  if (relu && resid) fwd_apply<true, true>(x, res, M, C, scale, shift, y, s);
  else if (relu) fwd_apply<true, false>(x, res, M, C, scale, shift, y, s);
  else if (resid) fwd_apply<false, true>(x, res, M, C, scale, shift, y, s);
  else fwd_apply<false, false>(x, res, M, C, scale, shift, y, s);
  return cudaGetLastError();
}

template <bool kRelu, bool kRes, bool kDy2>
static cudaError_t bwd_impl(const void* dy, const void* dy2, const void* x, const void* res,
                            int64_t M, int C, const float* save_mean, const float* save_invstd,
                            const float* scale_shift, const float* w, float* gw, float* gb,
                            float* coef, void* dx, void* dres, void* ws, cudaStream_t s) {
  const TileShape sh = tile_shape(C);
  const int blocks = bn_row_blocks(M, C);
  float* partial = (float*)((char*)ws + 256);
  const float* scale = scale_shift;
  const float* shift = scale_shift ? scale_shift + C : nullptr;
  bn_bwd_partial_kernel<kRelu, kRes, kDy2><<<dim3(blocks, C / sh.tile), kBnThreads, 0, s>>>(
      (const __nv_bfloat16*)dy, (const __nv_bfloat16*)dy2, (const __nv_bfloat16*)x,
      (const __nv_bfloat16*)res, M, C, save_mean, scale, shift, partial);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = launch_dependent(bn_bwd_finalize_kernel, dim3((C + 7) / 8), s, (const float*)partial, blocks,
                       M, C, save_mean, save_invstd, w, gw, gb, coef, coef + C, coef + 2 * C);
  if (e != cudaSuccess) return e;
  return launch_dependent(bn_bwd_apply_kernel<kRelu, kRes, kDy2>, dim3(apply_grid(M, C)), s,
                          (const __nv_bfloat16*)dy, (const __nv_bfloat16*)dy2,
                          (const __nv_bfloat16*)x, (const __nv_bfloat16*)res, M, C,
                          (const float*)coef, scale, shift, (__nv_bfloat16*)dx,
                          (__nv_bfloat16*)dres);
}

template <bool kDy2>
static cudaError_t bwd_dispatch(const void* dy, const void* dy2, const void* x, const void* res,
                                int64_t M, int C, const float* save_mean,
                                const float* save_invstd, const float* scale_shift, const float* w,
                                float* gw, float* gb, float* coef, void* dx, void* dres, void* ws,
                                int flags, cudaStream_t s) {
  const bool relu = flags & CS_BN_RELU, resid = flags & CS_BN_RESIDUAL;
  if (relu && resid)
    return bwd_impl<true, true, kDy2>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, s);
  if (relu)
    return bwd_impl<true, false, kDy2>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, s);
  if (resid)
    return bwd_impl<false, true, kDy2>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, s);
  return bwd_impl<false, false, kDy2>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, s);
}

cudaError_t launch_bn_bwd(const void* dy, const void* dy2, const void* x, const void* res, int64_t M,
                          int C, const float* save_mean, const float* save_invstd,
                          const float* scale_shift, const float* w, float* gw, float* gb,
                          float* coef, void* dx, void* dres, void* ws, int flags, cudaStream_t s) {
  if (dy2 != nullptr)
    return bwd_dispatch<true>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, flags, s);
  return bwd_dispatch<false>(dy, dy2, x, res, M, C, save_mean, save_invstd, scale_shift, w, gw, gb, coef, dx, dres, ws, flags, s);
}

}  // namespace cs
