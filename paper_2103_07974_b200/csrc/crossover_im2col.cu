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
  if (s.C == 3 && s.KH == 7 && s.KW == 7 && s.SH == 2 && s.SW == 2 && s.KP == 152)
    im2col_nhwc_kernel<3, 7, 7, 2, 2, 152, 0><<<g, 256, 0, stream>>>(xi, po, s, rows);   // ResNet stem
  else if (s.C == 3 && s.KH == 3 && s.KW == 3 && s.SH == 1 && s.SW == 1 && s.KP == 32)
    im2col_nhwc_kernel<3, 3, 3, 1, 1, 32, 0><<<g, 256, 0, stream>>>(xi, po, s, rows);     // VGG stem
  else
    im2col_nhwc_kernel<1, 1, 1, 1, 1, 8, 1><<<g, 256, 0, stream>>>(xi, po, s, rows);
  return cudaGetLastError();
}

}  // namespace cs
