// crossover_im2col.cu -- patch matrix of an NHWC image batch for the models' RGB stem convolution.
//
// cuDNN runs the ResNet-50 stem (7x7 / 2, 3 -> 64 channels, channels_last bf16) at ~46 TFLOP/s:
// with C = 3 it pads the input and falls back to sm80-era fprop / wgrad kernels, ~2.6 ms of a
// ~24 ms bs-256 iteration (tools/stem_bench.py).  The stem becomes two plain GEMMs instead
// (stem.py): y[M, O] = P[M, KP] . W[O, KP]^T and dW = dy^T . P, with P written here once per
// forward and kept for the weight gradient.  cuBLAS runs the GEMMs on the tensor cores.
//
// P row m = output pixel (n, oh, ow) (m = (n * OH + oh) * OW + ow, so P . W^T is NHWC = the
// channels_last output); column j < K = KH*KW*C holds x[n, oh*SH - PH + kh, ow*SW - PW + kw, c]
// with (kh, kw, c) = (j / (KW*C), (j / C) % KW, j % C), zero outside the image; columns K..KP-1
// are zero (KP % 8 == 0 keeps every row 16-byte aligned for 128-bit stores and the GEMM).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"
#include "crossover_internal.h"

namespace cs {

namespace {

struct Im2colShape {
  int N, H, W, C, OH, OW, KH, KW, SH, SW, PH, PW, KP;
};

// one thread = 8 consecutive columns (one 16-byte store) of one patch row.  The filter geometry
// is a template (the two RGB stems the apps use) so the per-column (kh, kw, c) decomposition is
// multiply-shift arithmetic; kGeneric = 1 is the runtime-shaped fallback.
template <int kC, int kKH, int kKW, int kSH, int kSW, int kKP, int kGeneric>
__global__ void __launch_bounds__(256)
im2col_nhwc_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ p,
                   const Im2colShape s, int rows) {
  const int C = kGeneric ? s.C : kC, KW = kGeneric ? s.KW : kKW, KH = kGeneric ? s.KH : kKH;
  const int SH = kGeneric ? s.SH : kSH, SW = kGeneric ? s.SW : kSW, KP = kGeneric ? s.KP : kKP;
  const int groups = KP / 8;
  const int K = KH * KW * C;
  const int total = rows * groups;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int m = t / groups;
    const int j0 = (t - m * groups) * 8;
    const int ow = m % s.OW;
    const int q = m / s.OW;
    const int oh = q % s.OH;
    const int n = q / s.OH;
    const int ih0 = oh * SH - s.PH, iw0 = ow * SW - s.PW;
    const __nv_bfloat16* img = x + (int64_t)n * s.H * s.W * C;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      __nv_bfloat16 val = __float2bfloat16(0.f);
      if (j < K) {
        const int c = j % C;
        const int kw = (j / C) % KW;
        const int kh = j / (C * KW);
        const int ih = ih0 + kh, iw = iw0 + kw;
        if ((unsigned)ih < (unsigned)s.H && (unsigned)iw < (unsigned)s.W)
          val = __ldg(img + (ih * s.W + iw) * C + c);
      }
      v[i] = val;
    }
    *reinterpret_cast<uint4*>(p + (int64_t)m * KP + j0) = *reinterpret_cast<const uint4*>(v);
  }
}

// One CTA per output row (n, oh): the KH input rows the row's windows touch are staged in shared
// memory with 16-byte loads (an NHWC input row is W*C contiguous bf16), then the CTA writes its
// OW consecutive patch rows -- one contiguous block of P -- with 16-byte stores.  The gather is
// served from shared memory instead of 2-byte global loads.
template <int kC, int kKH, int kKW, int kSH, int kSW, int kKP>
__global__ void __launch_bounds__(256)
im2col_rows_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ p,
                   const Im2colShape s) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* tile = reinterpret_cast<__nv_bfloat16*>(smem_raw);   // [kKH][W * kC]
  const int row = blockIdx.x;                  // n * OH + oh
  const int n = row / s.OH, oh = row - n * s.OH;
  const int rowlen = s.W * kC;                 // bf16 per input row (multiple of 8: host checked)
  const int vecs = rowlen / 8;
  for (int t = threadIdx.x; t < kKH * vecs; t += blockDim.x) {
    const int kh = t / vecs, v = t - kh * vecs;
    const int ih = oh * kSH - s.PH + kh;
    uint4 val = make_uint4(0, 0, 0, 0);
    if ((unsigned)ih < (unsigned)s.H)
      val = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)n * s.H + ih) * rowlen) + v);
    reinterpret_cast<uint4*>(tile + kh * rowlen)[v] = val;
  }
  __syncthreads();
  constexpr int kGroups = kKP / 8;
  constexpr int kK = kKH * kKW * kC;
  constexpr int kRowsPerPass = 256 / kGroups;    // blockDim = kGroups * kRowsPerPass (host)
  __nv_bfloat16* out = p + (int64_t)row * s.OW * kKP;
  // each thread owns one fixed 8-column group of every patch row it writes: the (kh, kw, c)
  // decomposition of its 8 columns is done once, the row loop is a shared-memory gather
  const int g = threadIdx.x % kGroups, r0 = threadIdx.x / kGroups;
  if (r0 >= kRowsPerPass) return;
  int off[8], kwv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = g * 8 + i;
    const int c = j % kC, kw = (j / kC) % kKW, kh = j / (kC * kKW);
    off[i] = j < kK ? kh * rowlen + kw * kC + c : -1;
    kwv[i] = j < kK ? kw : -1 - s.W;              // never in range for padding columns
  }
  for (int ow = r0; ow < s.OW; ow += kRowsPerPass) {
    const int iw0 = ow * kSW - s.PW;
    __align__(16) __nv_bfloat16 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int iw = iw0 + kwv[i];
      v[i] = (unsigned)iw < (unsigned)s.W ? tile[off[i] + iw0 * kC] : __float2bfloat16(0.f);
    }
    *reinterpret_cast<uint4*>(out + (int64_t)ow * kKP + g * 8) = *reinterpret_cast<const uint4*>(v);
  }
}

int sm_count_im2col() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

cudaError_t launch_im2col_nhwc(const void* x, void* p, const int* shape, cudaStream_t stream) {
  Im2colShape s{shape[0], shape[1], shape[2],  shape[3],  shape[4],  shape[5], shape[6],
                shape[7], shape[8], shape[9], shape[10], shape[11], shape[12]};
  const int rows = s.N * s.OH * s.OW;            // host checked: rows * KP / 8 < 2^31
  const int64_t total = (int64_t)rows * (s.KP / 8);
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)sm_count_im2col() * 16;
  if (grid > cap) grid = cap;
  const unsigned g = (unsigned)(grid < 1 ? 1 : grid);
  const auto* xi = (const __nv_bfloat16*)x;
  auto* po = (__nv_bfloat16*)p;
  // 16-byte staging of whole input rows: row length and base address must be 16-byte multiples
  const bool rows_ok = (s.W * s.C) % 8 == 0 && ((uintptr_t)xi & 15u) == 0;
  if (rows_ok && s.C == 3 && s.KH == 7 && s.KW == 7 && s.SH == 2 && s.SW == 2 && s.KP == 152)
    im2col_rows_kernel<3, 7, 7, 2, 2, 152><<<(unsigned)(s.N * s.OH), 19 * (256 / 19), 7 * s.W * 3 * 2, stream>>>(
        xi, po, s);                                                                        // ResNet stem
  else if (rows_ok && s.C == 3 && s.KH == 3 && s.KW == 3 && s.SH == 1 && s.SW == 1 && s.KP == 32)
    im2col_rows_kernel<3, 3, 3, 1, 1, 32><<<(unsigned)(s.N * s.OH), 4 * (256 / 4), 3 * s.W * 3 * 2, stream>>>(
        xi, po, s);                                                                        // VGG stem
  else if (s.C == 3 && s.KH == 7 && s.KW == 7 && s.SH == 2 && s.SW == 2 && s.KP == 152)
    im2col_nhwc_kernel<3, 7, 7, 2, 2, 152, 0><<<g, 256, 0, stream>>>(xi, po, s, rows);
  else if (s.C == 3 && s.KH == 3 && s.KW == 3 && s.SH == 1 && s.SW == 1 && s.KP == 32)
    im2col_nhwc_kernel<3, 3, 3, 1, 1, 32, 0><<<g, 256, 0, stream>>>(xi, po, s, rows);
  else
    im2col_nhwc_kernel<1, 1, 1, 1, 1, 8, 1><<<g, 256, 0, stream>>>(xi, po, s, rows);
  return cudaGetLastError();
}

}  // namespace cs
