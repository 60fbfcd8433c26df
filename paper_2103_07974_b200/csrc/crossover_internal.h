// crossover_internal.h -- launch-parameter layouts shared by the kernels and the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "crossover.h"

namespace cs {

constexpr int kThreads = 256;                      // 8 warps per CTA
constexpr int kStatsMaxGrid = 148 * 8;             // fixed -> deterministic partial order

// descriptor capacities per launch (kernel parameters are <= 32 KB on sm_70+)
constexpr int kCapSmall = 16;
constexpr int kCapMid = 128;
constexpr int kCapLarge = 512;

template <int CAP>
struct PackArgs {
  int n;
  int total_chunks;
  int chunk_begin[CAP + 1];
  const float* src[CAP];
  float* dst[CAP];
  int64_t numel[CAP];
};

template <int CAP>
struct UpdateArgs {
  int n;
  int total_chunks;
  int nsrc;
  int pad_;
  float* snapshot;
  uint64_t base[CS_MAX_SOURCES];
  cs_sgd_hyper h;
  int chunk_begin[CAP + 1];
  float* param[CAP];
  float* mom[CAP];
  uint64_t grad_off[CAP];
  uint64_t snap_off[CAP];
  int64_t numel[CAP];
};

static_assert(sizeof(PackArgs<kCapLarge>) < 32000, "pack args exceed kernel param space");
static_assert(sizeof(UpdateArgs<kCapLarge>) < 32000, "update args exceed kernel param space");

template <int CAP>
cudaError_t launch_pack(const PackArgs<CAP>& a, int max_ctas, cudaStream_t s);
template <int CAP>
cudaError_t launch_unpack_sgd(const UpdateArgs<CAP>& a, bool mom, int max_ctas, cudaStream_t s);
int reg_pack_chunk();
int reg_update_chunk();
extern int g_tune_reg_shape;
extern int g_tune_sync_ctas;
extern int g_tune_p2p_ctas;
extern int g_tune_p2p_bulk;
extern int g_tune_bn_no_pdl;
extern int g_tune_bn_ctas_per_sm;
cudaError_t launch_p2p(const cs_p2p_desc& d, const cs_sgd_hyper& h, cudaStream_t s);
int64_t p2p_gather_chunk_elems(int nranks);
cudaError_t launch_p2p_gather(const cs_p2p_desc* chunks, int64_t nchunks, int nranks, int max_ctas,
                              const cs_sgd_hyper& h, cudaStream_t s);
int bn_row_blocks(int64_t M, int C);
cudaError_t launch_im2col_nhwc(const void* x, void* p, const int* shape, cudaStream_t stream);
size_t bn_workspace_bytes(int64_t M, int C);
cudaError_t launch_bn_fwd(const void* x, const void* res, int64_t M, int C, const float* w,
                          const float* b, float* rm, float* rv, float momentum, float eps,
                          float* save_mean, float* save_invstd, float* scale_shift, void* y,
                          void* ws, int flags, cudaStream_t s);
cudaError_t launch_bn_bwd(const void* dy, const void* dy2, const void* x, const void* res, int64_t M, int C,
                          const float* save_mean, const float* save_invstd,
                          const float* scale_shift, const float* w, float* gw, float* gb,
                          float* coef, void* dx, void* dres, void* ws, int flags, cudaStream_t s);
cudaError_t launch_maxpool_fwd(const void* x, void* y, void* arg, const int* shape, cudaStream_t st);
cudaError_t launch_maxpool_bwd(const void* dy, const void* arg, void* dx, const int* shape,
                               cudaStream_t st);
cudaError_t launch_stats(const float* data, int64_t numel, double* out, void* ws,
                         cudaStream_t s);
int stats_grid(int64_t numel);
cudaError_t launch_spin_ns(uint64_t ns, cudaStream_t s);

// thread-local error reporting shared by every translation unit of the library
int set_error(int code, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

}  // namespace cs
