// crossover_pool.cu -- channels_last max pooling for the apps' compute (ResNet stem).
//
// ATen's NHWC max_pool2d kernels took ~2.5 ms of every ResNet-50 bs256 iteration
// (profiles/r01_launches_fastbn.md) and save int64 indices (8 bytes per output element).
// Here the forward stores the argmax as a uint8 window offset (kh*kw <= 255) and the backward
// is a gather: every input element sums dy over the (at most ceil(k/s)^2) windows that
// selected it.  Scan order and comparison match ATen (row-major window scan, first strictly
// greater value wins, NaN propagates), so the selected positions -- and therefore dx -- are
// identical.  8 channels (16 bytes of bf16) per thread.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"

namespace cs {

namespace {
constexpr int kPoolThreads = 256;

__device__ __forceinline__ void unpack8p(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ uint4 pack8p(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
}  // namespace

struct PoolShape {
  int N, H, W, C, OH, OW, kh, kw, sh, sw, ph, pw;
};

// 3x3 windows (the ResNet stem): all nine 16-byte loads issued before the first compare.
// Idx = int when the element count fits (the host picks it): the per-thread index
// decomposition is then 32-bit division, several times cheaper than 64-bit.
template <typename Idx>
__global__ void __launch_bounds__(kPoolThreads)
maxpool3_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                    uint8_t* __restrict__ arg, PoolShape s) {
  const int cv = s.C / 8;
  const Idx total = (Idx)s.N * s.OH * s.OW * cv;
  for (Idx i = (Idx)blockIdx.x * kPoolThreads + threadIdx.x; i < total;
       i += (Idx)gridDim.x * kPoolThreads) {
    const int c8 = (int)(i % cv);
    Idx t = i / cv;
    const int ow = (int)(t % s.OW);
    t /= s.OW;
    const int oh = (int)(t % s.OH);
    const int n = (int)(t / s.OH);
    const int h0 = oh * s.sh - s.ph, w0 = ow * s.sw - s.pw;
    uint4 raw[9];
    bool ok[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int ih = h0 + a, iw = w0 + b;
        ok[a * 3 + b] = ih >= 0 && ih < s.H && iw >= 0 && iw < s.W;
        raw[a * 3 + b] = ok[a * 3 + b]
            ? __ldg(reinterpret_cast<const uint4*>(x + (((int64_t)n * s.H + ih) * s.W + iw) * s.C + c8 * 8))
            : make_uint4(0, 0, 0, 0);
      }
    float best[8];
    uint8_t idx[8];
    const uint8_t first = (uint8_t)(max(0, -h0) * 3 + max(0, -w0));
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; idx[k] = first; }
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      if (!ok[o]) continue;
      float v[8];
      unpack8p(raw[o], v);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (v[k] > best[k] || isnan(v[k])) { best[k] = v[k]; idx[k] = (uint8_t)o; }   // ATen's rule
    }
    *reinterpret_cast<uint4*>(y + i * 8) = pack8p(best);
    uint2 packed;
    packed.x = idx[0] | (idx[1] << 8) | (idx[2] << 16) | ((uint32_t)idx[3] << 24);
    packed.y = idx[4] | (idx[5] << 8) | (idx[6] << 16) | ((uint32_t)idx[7] << 24);
    *reinterpret_cast<uint2*>(arg + i * 8) = packed;
  }
}

__global__ void __launch_bounds__(kPoolThreads)
maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                   uint8_t* __restrict__ arg, PoolShape s) {
  const int cv = s.C / 8;
  const int64_t total = (int64_t)s.N * s.OH * s.OW * cv;
  for (int64_t i = (int64_t)blockIdx.x * kPoolThreads + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * kPoolThreads) {
    const int c8 = (int)(i % cv);
    int64_t t = i / cv;
    const int ow = (int)(t % s.OW);
    t /= s.OW;
    const int oh = (int)(t % s.OH);
    const int n = (int)(t / s.OH);
    float best[8];
    uint8_t idx[8];
    const int h0 = oh * s.sh - s.ph, w0 = ow * s.sw - s.pw;
    // ATen starts from the first in-bounds position of the window
    const uint8_t first = (uint8_t)(max(0, -h0) * s.kw + max(0, -w0));
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; idx[k] = first; }
    for (int a = 0; a < s.kh; ++a) {
      const int ih = h0 + a;
      if (ih < 0 || ih >= s.H) continue;
      for (int b = 0; b < s.kw; ++b) {
        const int iw = w0 + b;
        if (iw < 0 || iw >= s.W) continue;
        float v[8];
        unpack8p(*reinterpret_cast<const uint4*>(x + (((int64_t)n * s.H + ih) * s.W + iw) * s.C + c8 * 8), v);
        const uint8_t o = (uint8_t)(a * s.kw + b);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (v[k] > best[k] || isnan(v[k])) { best[k] = v[k]; idx[k] = o; }   // ATen's rule
      }
    }
    *reinterpret_cast<uint4*>(y + i * 8) = pack8p(best);
    uint2 packed;
    packed.x = idx[0] | (idx[1] << 8) | (idx[2] << 16) | ((uint32_t)idx[3] << 24);
    packed.y = idx[4] | (idx[5] << 8) | (idx[6] << 16) | ((uint32_t)idx[7] << 24);
    *reinterpret_cast<uint2*>(arg + i * 8) = packed;
  }
}

template <typename Idx>
__global__ void __launch_bounds__(kPoolThreads)
maxpool_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
                   __nv_bfloat16* __restrict__ dx, PoolShape s) {
  const int cv = s.C / 8;
  const Idx total = (Idx)s.N * s.H * s.W * cv;
  for (Idx i = (Idx)blockIdx.x * kPoolThreads + threadIdx.x; i < total;
       i += (Idx)gridDim.x * kPoolThreads) {
    const int c8 = (int)(i % cv);
    Idx t = i / cv;
    const int iw = (int)(t % s.W);
    t /= s.W;
    const int ih = (int)(t % s.H);
    const int n = (int)(t / s.H);
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    // output windows containing (ih, iw): oh*sh - ph <= ih < oh*sh - ph + kh
    const int oh_lo = max(0, (ih + s.ph - s.kh + s.sh) / s.sh);
    const int oh_hi = min(s.OH - 1, (ih + s.ph) / s.sh);
    const int ow_lo = max(0, (iw + s.pw - s.kw + s.sw) / s.sw);
    const int ow_hi = min(s.OW - 1, (iw + s.pw) / s.sw);
    if (oh_hi - oh_lo <= 1 && ow_hi - ow_lo <= 1) {
      // common case (kernel <= 2 * stride): up to 2x2 windows, loads issued together
      uint4 rg[4];
      uint2 ra[4];
      uint8_t me[4];
      bool use[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int oh = oh_lo + (q >> 1), ow = ow_lo + (q & 1);
        const int a = ih - (oh * s.sh - s.ph), b = iw - (ow * s.sw - s.pw);
        use[q] = oh <= oh_hi && ow <= ow_hi && a >= 0 && a < s.kh && b >= 0 && b < s.kw;
        me[q] = (uint8_t)(a * s.kw + b);
        const int64_t o = (((int64_t)n * s.OH + oh) * s.OW + ow) * cv + c8;
        rg[q] = use[q] ? __ldg(reinterpret_cast<const uint4*>(dy + o * 8)) : make_uint4(0, 0, 0, 0);
        ra[q] = use[q] ? __ldg(reinterpret_cast<const uint2*>(arg + o * 8)) : make_uint2(0, 0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!use[q]) continue;
        float g[8];
        unpack8p(rg[q], g);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t word = k < 4 ? ra[q].x : ra[q].y;
          if (((word >> (8 * (k & 3))) & 0xffu) == me[q]) acc[k] += g[k];
        }
      }
    } else {
      for (int oh = oh_lo; oh <= oh_hi; ++oh) {
        const int a = ih - (oh * s.sh - s.ph);
        if (a < 0 || a >= s.kh) continue;
        for (int ow = ow_lo; ow <= ow_hi; ++ow) {
          const int b = iw - (ow * s.sw - s.pw);
          if (b < 0 || b >= s.kw) continue;
          const int64_t o = (((int64_t)n * s.OH + oh) * s.OW + ow) * cv + c8;
          const uint2 packed = *reinterpret_cast<const uint2*>(arg + o * 8);
          const uint8_t mine = (uint8_t)(a * s.kw + b);
          float g[8];
          unpack8p(*reinterpret_cast<const uint4*>(dy + o * 8), g);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t word = k < 4 ? packed.x : packed.y;
            if (((word >> (8 * (k & 3))) & 0xffu) == mine) acc[k] += g[k];
          }
        }
      }
    }
    *reinterpret_cast<uint4*>(dx + i * 8) = pack8p(acc);
  }
}

// The ResNet stem's pool (3x3, stride 2, padding 1, C = 8 * kCV): one CTA per row and the
// channel-vector count a compile-time constant, so the per-thread index arithmetic is shifts and
// masks (the generic kernels spend most of their time in runtime integer division).
template <int kCV>
__global__ void __launch_bounds__(128)
maxpool_k3s2_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                        uint8_t* __restrict__ arg, PoolShape s) {
  const int row = blockIdx.x;                 // n * OH + oh
  const int n = row / s.OH, oh = row - n * s.OH;
  const int h0 = 2 * oh - 1;
  const __nv_bfloat16* img = x + (int64_t)n * s.H * s.W * (kCV * 8);
  for (int v = threadIdx.x; v < s.OW * kCV; v += blockDim.x) {
    const int ow = v / kCV, c8 = v % kCV;
    const int w0 = 2 * ow - 1;
    uint4 raw[9];
    bool ok[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int ih = h0 + a, iw = w0 + b;
        ok[a * 3 + b] = (unsigned)ih < (unsigned)s.H && (unsigned)iw < (unsigned)s.W;
        raw[a * 3 + b] = ok[a * 3 + b]
            ? __ldg(reinterpret_cast<const uint4*>(img + ((int64_t)ih * s.W + iw) * (kCV * 8) + c8 * 8))
            : make_uint4(0, 0, 0, 0);
      }
    float best[8];
    uint8_t idx[8];
    const uint8_t first = (uint8_t)(max(0, -h0) * 3 + max(0, -w0));
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; idx[k] = first; }
#pragma unroll
    for (int o = 0; o < 9; ++o) {
      if (!ok[o]) continue;
      float f[8];
      unpack8p(raw[o], f);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (f[k] > best[k] || isnan(f[k])) { best[k] = f[k]; idx[k] = (uint8_t)o; }   // ATen's rule
    }
    const int64_t out = ((int64_t)row * s.OW + ow) * kCV + c8;
    *reinterpret_cast<uint4*>(y + out * 8) = pack8p(best);
    uint2 packed;
    packed.x = idx[0] | (idx[1] << 8) | (idx[2] << 16) | ((uint32_t)idx[3] << 24);
    packed.y = idx[4] | (idx[5] << 8) | (idx[6] << 16) | ((uint32_t)idx[7] << 24);
    *reinterpret_cast<uint2*>(arg + out * 8) = packed;
  }
}

template <int kCV>
__global__ void __launch_bounds__(128)
maxpool_k3s2_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
                        __nv_bfloat16* __restrict__ dx, PoolShape s) {
  const int row = blockIdx.x;                 // n * H + ih
  const int n = row / s.H, ih = row - n * s.H;
  // windows oh with 2*oh - 1 <= ih <= 2*oh + 1
  const int oh_lo = ih >> 1, oh_hi = min(s.OH - 1, (ih + 1) >> 1);
  for (int v = threadIdx.x; v < s.W * kCV; v += blockDim.x) {
    const int iw = v / kCV, c8 = v % kCV;
    const int ow_lo = iw >> 1, ow_hi = min(s.OW - 1, (iw + 1) >> 1);
    uint4 rg[4];
    uint2 ra[4];
    uint8_t me[4];
    bool use[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int oh = oh_lo + (q >> 1), ow = ow_lo + (q & 1);
      use[q] = oh <= oh_hi && ow <= ow_hi;
      me[q] = (uint8_t)((ih - (2 * oh - 1)) * 3 + (iw - (2 * ow - 1)));
      const int64_t o = (((int64_t)n * s.OH + oh) * s.OW + ow) * kCV + c8;
      rg[q] = use[q] ? __ldg(reinterpret_cast<const uint4*>(dy + o * 8)) : make_uint4(0, 0, 0, 0);
      ra[q] = use[q] ? __ldg(reinterpret_cast<const uint2*>(arg + o * 8)) : make_uint2(0, 0);
    }
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!use[q]) continue;
      float g[8];
      unpack8p(rg[q], g);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t word = k < 4 ? ra[q].x : ra[q].y;
        if (((word >> (8 * (k & 3))) & 0xffu) == me[q]) acc[k] += g[k];
      }
    }
    const int64_t out = ((int64_t)row * s.W + iw) * kCV + c8;
    *reinterpret_cast<uint4*>(dx + out * 8) = pack8p(acc);
  }
}

// Backward of the stem pool for even H, W with OH = H/2, OW = W/2: one thread per 2x2 input
// block (2a..2a+1, 2b..2b+1) x 8 channels.  The block's 4 dx vectors are covered by exactly the
// windows (a, b), (a, b+1), (a+1, b), (a+1, b+1), so every window's dy / argmax is loaded once
// instead of ~2.25 times; window offsets of the 4 positions are compile-time constants.
template <int kCV>
__global__ void __launch_bounds__(128)
maxpool_k3s2_bwd_2x2_kernel(const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
                            __nv_bfloat16* __restrict__ dx, PoolShape s) {
  const int row = blockIdx.x;                 // n * OH + a
  const int n = row / s.OH, a = row - n * s.OH;
  for (int v = threadIdx.x; v < s.OW * kCV; v += blockDim.x) {
    const int b = v / kCV, c8 = v % kCV;
    uint4 rg[4];
    uint2 ra[4];
    bool use[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {               // q = 2 * dh + dw: window (a + dh, b + dw)
      const int oh = a + (q >> 1), ow = b + (q & 1);
      use[q] = oh < s.OH && ow < s.OW;
      const int64_t o = (((int64_t)n * s.OH + oh) * s.OW + ow) * kCV + c8;
      rg[q] = use[q] ? __ldg(reinterpret_cast<const uint4*>(dy + o * 8)) : make_uint4(0, 0, 0, 0);
      ra[q] = use[q] ? __ldg(reinterpret_cast<const uint2*>(arg + o * 8)) : make_uint2(0, 0);
    }
    float g[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q) unpack8p(rg[q], g[q]);
    // position p = 2 * di + dj (input (2a + di, 2b + dj)); for window q its offset in the 3x3
    // window is (di - 2*(q>>1) + 1) * 3 + (dj - 2*(q&1) + 1) when inside, else not covered
#pragma unroll
    for (int pos = 0; pos < 4; ++pos) {
      const int di = pos >> 1, dj = pos & 1;
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = di - 2 * (q >> 1) + 1, c = dj - 2 * (q & 1) + 1;
        if (r < 0 || r > 2 || c < 0 || c > 2) continue;          // compile-time after unrolling
        if (!use[q]) continue;
        const uint32_t me = (uint32_t)(r * 3 + c);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t word = k < 4 ? ra[q].x : ra[q].y;
          if (((word >> (8 * (k & 3))) & 0xffu) == me) acc[k] += g[q][k];
        }
      }
      const int ih = 2 * a + di, iw = 2 * b + dj;
      const int64_t out = (((int64_t)n * s.H + ih) * s.W + iw) * kCV + c8;
      *reinterpret_cast<uint4*>(dx + out * 8) = pack8p(acc);
    }
  }
}

static bool stem_pool(const PoolShape& s) {
  return s.kh == 3 && s.kw == 3 && s.sh == 2 && s.sw == 2 && s.ph == 1 && s.pw == 1 && s.C == 64;
}

static unsigned pool_grid(int64_t total) {
  int64_t g = (total + kPoolThreads - 1) / kPoolThreads;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

cudaError_t launch_maxpool_fwd(const void* x, void* y, void* arg, const int* shape, cudaStream_t st) {
  PoolShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5],
              shape[6], shape[7], shape[8], shape[9], shape[10], shape[11]};
  const int64_t total = (int64_t)s.N * s.OH * s.OW * (s.C / 8);
  const bool narrow = (int64_t)s.N * s.H * s.W * s.C < INT32_MAX;   // every flat index fits int
  if (stem_pool(s))
    maxpool_k3s2_fwd_kernel<8><<<(unsigned)(s.N * s.OH), 128, 0, st>>>(
        (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)arg, s);
  else if (s.kh == 3 && s.kw == 3 && narrow)
    maxpool3_fwd_kernel<int><<<pool_grid(total), kPoolThreads, 0, st>>>(
        (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)arg, s);
  else if (s.kh == 3 && s.kw == 3)
    maxpool3_fwd_kernel<int64_t><<<pool_grid(total), kPoolThreads, 0, st>>>(
        (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)arg, s);
  else
    maxpool_fwd_kernel<<<pool_grid(total), kPoolThreads, 0, st>>>(
        (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)arg, s);
  return cudaGetLastError();
}

cudaError_t launch_maxpool_bwd(const void* dy, const void* arg, void* dx, const int* shape,
                               cudaStream_t st) {
  PoolShape s{shape[0], shape[1], shape[2], shape[3], shape[4], shape[5],
              shape[6], shape[7], shape[8], shape[9], shape[10], shape[11]};
  const int64_t total = (int64_t)s.N * s.H * s.W * (s.C / 8);
  if (stem_pool(s) && s.H == 2 * s.OH && s.W == 2 * s.OW)
    maxpool_k3s2_bwd_2x2_kernel<8><<<(unsigned)(s.N * s.OH), 128, 0, st>>>(
        (const __nv_bfloat16*)dy, (const uint8_t*)arg, (__nv_bfloat16*)dx, s);
  else if (stem_pool(s))
    maxpool_k3s2_bwd_kernel<8><<<(unsigned)(s.N * s.H), 128, 0, st>>>(
        (const __nv_bfloat16*)dy, (const uint8_t*)arg, (__nv_bfloat16*)dx, s);
  else if ((int64_t)s.N * s.H * s.W * s.C < INT32_MAX)
    maxpool_bwd_kernel<int><<<pool_grid(total), kPoolThreads, 0, st>>>(
        (const __nv_bfloat16*)dy, (const uint8_t*)arg, (__nv_bfloat16*)dx, s);
  else
    maxpool_bwd_kernel<int64_t><<<pool_grid(total), kPoolThreads, 0, st>>>(
        (const __nv_bfloat16*)dy, (const uint8_t*)arg, (__nv_bfloat16*)dx, s);
  return cudaGetLastError();
}

}  // namespace cs
