// crossover_abi.cu -- extern "C" entry points of libcrossover.so (see include/crossover.h).
//
// Host-side work per call is O(n_tensors): validate, build the chunk prefix,
// copy descriptors into a by-value kernel-parameter block, launch.  No device
// allocation, no synchronisation, no host<->device copies.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "crossover.h"
#include "crossover_internal.h"

namespace cs {
thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return 0;
  return set_error((int)e, "%s: %s", where, cudaGetErrorString(e));
}

static int64_t chunks_of(int64_t numel, int chunk) { return (numel + chunk - 1) / chunk; }

template <int CAP>
static int pack_batch(const cs_pack_desc* d, int n, int max_ctas, cudaStream_t s) {
  static thread_local PackArgs<CAP> a;  // ~28 KB for the large capacity: keep off the stack
  a.n = n;
  const int chunk = reg_pack_chunk();
  int64_t c = 0;
  for (int i = 0; i < n; ++i) {
    a.chunk_begin[i] = (int)c;
    a.src[i] = d[i].src;
    a.dst[i] = d[i].dst;
    a.numel[i] = d[i].numel;
    c += chunks_of(d[i].numel, chunk);
  }
  a.chunk_begin[n] = (int)c;
  if (c > INT32_MAX) return set_error(CS_ERR_ARG, "cs_pack: %lld chunks exceed grid limit", (long long)c);
  a.total_chunks = (int)c;
  return cuda_status(launch_pack<CAP>(a, max_ctas, s), "cs_pack launch");
}

template <int CAP>
static int update_batch(const cs_update_desc* d, int n, const uint64_t* sources, int nsrc,
                        float* snapshot, const cs_sgd_hyper* h, int max_ctas, cudaStream_t s) {
  static thread_local UpdateArgs<CAP> a;
  a.n = n;
  a.nsrc = nsrc;
  a.pad_ = 0;
  a.snapshot = snapshot;
  for (int k = 0; k < CS_MAX_SOURCES; ++k) a.base[k] = k < nsrc ? sources[k] : 0;
  a.h = *h;
  const bool mom = h->momentum != 0.0f;
  const int chunk = reg_update_chunk();
  int64_t c = 0;
  for (int i = 0; i < n; ++i) {
    a.chunk_begin[i] = (int)c;
    a.param[i] = d[i].param;
    a.mom[i] = d[i].momentum_buf;
    a.grad_off[i] = d[i].grad_offset;
    a.snap_off[i] = d[i].snap_offset;
    a.numel[i] = d[i].numel;
    c += chunks_of(d[i].numel, chunk);
  }
  a.chunk_begin[n] = (int)c;
  if (c > INT32_MAX) return set_error(CS_ERR_ARG, "cs_unpack_sgd: %lld chunks exceed grid limit", (long long)c);
  a.total_chunks = (int)c;
  return cuda_status(launch_unpack_sgd<CAP>(a, mom, max_ctas, s), "cs_unpack_sgd launch");
}

}  // namespace cs

using namespace cs;

extern "C" {

int cs_abi_version(void) { return CS_ABI_VERSION; }

const char* cs_last_error(void) { return g_last_error.c_str(); }

int cs_tune(const char* key, int value) {
  if (key == nullptr || value < 0) return set_error(CS_ERR_ARG, "cs_tune: invalid arguments");
  const std::string k(key);
  if (k == "reg_shape" && value <= 4) g_tune_reg_shape = value;
  else if (k == "p2p_ctas" && value <= 65536) g_tune_p2p_ctas = value;
  else if (k == "p2p_bulk" && value <= 1) g_tune_p2p_bulk = value;
  else if (k == "sync_ctas" && value <= 65536) g_tune_sync_ctas = value;
  else if (k == "bn_no_pdl" && value <= 1) g_tune_bn_no_pdl = value;
  else if (k == "bn_ctas_per_sm" && value <= 8) g_tune_bn_ctas_per_sm = value;
  else return set_error(CS_ERR_ARG, "cs_tune: unknown key or bad value (%s=%d)", key, value);
  return 0;
}

int cs_pack(const cs_pack_desc* descs, int n, int max_ctas, void* stream) {
  if (n < 0 || (n > 0 && descs == nullptr))
    return set_error(CS_ERR_ARG, "cs_pack: invalid descriptor array (n=%d)", n);
  if (max_ctas < 0) return set_error(CS_ERR_ARG, "cs_pack: max_ctas < 0");
  for (int i = 0; i < n; ++i) {
    if (descs[i].numel < 0)
      return set_error(CS_ERR_ARG, "cs_pack: tensor %d has negative numel", i);
    if (descs[i].numel > 0 && (descs[i].src == nullptr || descs[i].dst == nullptr))
      return set_error(CS_ERR_ARG, "cs_pack: tensor %d has a null pointer", i);
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (int b = 0; b < n; b += kCapLarge) {
    const int m = std::min(kCapLarge, n - b);
    int rc = m <= kCapSmall ? pack_batch<kCapSmall>(descs + b, m, max_ctas, s)
           : m <= kCapMid   ? pack_batch<kCapMid>(descs + b, m, max_ctas, s)
                            : pack_batch<kCapLarge>(descs + b, m, max_ctas, s);
    if (rc) return rc;
  }
  return 0;
}

int cs_unpack_sgd(const cs_update_desc* descs, int n, const uint64_t* sources,
                  int n_sources, float* snapshot, const cs_sgd_hyper* hyper, int max_ctas,
                  void* stream) {
  if (n < 0 || (n > 0 && descs == nullptr))
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: invalid descriptor array (n=%d)", n);
  if (max_ctas < 0) return set_error(CS_ERR_ARG, "cs_unpack_sgd: max_ctas < 0");
  if (hyper == nullptr) return set_error(CS_ERR_ARG, "cs_unpack_sgd: hyper is NULL");
  if (n_sources < 1 || n_sources > CS_MAX_SOURCES || sources == nullptr)
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: n_sources=%d outside [1, %d]", n_sources,
                     CS_MAX_SOURCES);
  if (hyper->divisor < 1)
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: divisor must be >= 1 (got %d)", hyper->divisor);
  if (!(hyper->lr > 0.0f))
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: learning rate must be > 0");
  if (hyper->rounding != CS_ROUND_REFERENCE && hyper->rounding != CS_ROUND_TORCH)
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: unknown rounding mode %d", hyper->rounding);
  if (hyper->rounding == CS_ROUND_REFERENCE &&
      (hyper->momentum != 0.0f || hyper->weight_decay != 0.0f))
    return set_error(CS_ERR_ARG,
                     "cs_unpack_sgd: reference rounding has no momentum / weight decay");
  if (hyper->nesterov && (hyper->momentum <= 0.0f || hyper->dampening_complement != 1.0f))
    return set_error(CS_ERR_ARG, "cs_unpack_sgd: nesterov needs momentum > 0 and dampening 0");
  const bool mom = hyper->momentum != 0.0f;
  for (int i = 0; i < n; ++i) {
    if (descs[i].numel < 0)
      return set_error(CS_ERR_ARG, "cs_unpack_sgd: tensor %d has negative numel", i);
    if (descs[i].numel > 0 && (descs[i].param == nullptr || (mom && descs[i].momentum_buf == nullptr)))
      return set_error(CS_ERR_ARG, "cs_unpack_sgd: tensor %d has a null pointer", i);
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (int b = 0; b < n; b += kCapLarge) {
    const int m = std::min(kCapLarge, n - b);
    int rc = m <= kCapSmall ? update_batch<kCapSmall>(descs + b, m, sources, n_sources, snapshot, hyper, max_ctas, s)
           : m <= kCapMid   ? update_batch<kCapMid>(descs + b, m, sources, n_sources, snapshot, hyper, max_ctas, s)
                            : update_batch<kCapLarge>(descs + b, m, sources, n_sources, snapshot, hyper, max_ctas, s);
    if (rc) return rc;
  }
  return 0;
}

int cs_p2p_reduce_sgd_bcast(const cs_p2p_desc* d, const cs_sgd_hyper* h, void* stream) {
  if (d == nullptr || h == nullptr) return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: NULL argument");
  if (d->nranks < 1 || d->nranks > CS_MAX_SOURCES)
    return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: nranks=%d outside [1, %d]", d->nranks,
                     CS_MAX_SOURCES);
  if (d->numel < 0 || (d->numel > 0 && d->param == nullptr))
    return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: bad shard");
  if (d->max_ctas < 0) return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: max_ctas < 0");
  if (h->divisor != d->nranks)
    return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: divisor %d != nranks %d", h->divisor, d->nranks);
  if (!(h->lr > 0.0f)) return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: learning rate must be > 0");
  if (h->rounding == CS_ROUND_REFERENCE && (h->momentum != 0.0f || h->weight_decay != 0.0f))
    return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: reference rounding has no momentum / weight decay");
  if (h->momentum != 0.0f && d->momentum_buf == nullptr)
    return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: momentum buffer is NULL");
  uintptr_t al = (uintptr_t)d->param | (uintptr_t)d->momentum_buf;
  for (int r = 0; r < d->nranks; ++r) {
    if (d->src[r] == 0 || d->dst[r] == 0)
      return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: NULL peer address for rank %d", r);
    al |= (uintptr_t)d->src[r] | (uintptr_t)d->dst[r];
  }
  if (al & 15u) return set_error(CS_ERR_ARG, "cs_p2p_reduce_sgd_bcast: shards must be 16-byte aligned");
  return cuda_status(launch_p2p(*d, *h, (cudaStream_t)stream), "cs_p2p_reduce_sgd_bcast launch");
}

int cs_device_alloc(size_t bytes, void** ptr) {
  if (ptr == nullptr || bytes == 0) return set_error(CS_ERR_ARG, "cs_device_alloc: invalid arguments");
  int rc = cuda_status(cudaMalloc(ptr, bytes), "cudaMalloc");
  if (rc) return rc;
  return cuda_status(cudaMemset(*ptr, 0, bytes), "cudaMemset");
}

int cs_device_free(void* ptr) {
  if (ptr == nullptr) return 0;
  return cuda_status(cudaFree(ptr), "cudaFree");
}

int cs_ipc_get_handle(void* ptr, uint8_t* out) {
  if (ptr == nullptr || out == nullptr) return set_error(CS_ERR_ARG, "cs_ipc_get_handle: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == CS_IPC_HANDLE_BYTES, "IPC handle size changed");
  cudaIpcMemHandle_t h;
  int rc = cuda_status(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
  if (rc) return rc;
  std::memcpy(out, &h, sizeof(h));
  return 0;
}

int cs_ipc_open_handle(const uint8_t* handle, void** ptr) {
  if (ptr == nullptr || handle == nullptr) return set_error(CS_ERR_ARG, "cs_ipc_open_handle: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int cs_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  if (dst == nullptr || src == nullptr) return set_error(CS_ERR_ARG, "cs_copy_async: NULL pointer");
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  if (e == cudaSuccess) return 0;
  cudaGetLastError();
  return set_error((int)e, "cs_copy_async(dst=%p, src=%p, %zu bytes): %s", dst, src, bytes,
                   cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// SM-free cross-rank barrier: stream memory operations (executed by the GPU front end, no
// kernel).  The driver entry points come from cudaGetDriverEntryPointByVersion, so the library
// does not link libcuda and still loads on a host without a driver.
// ---------------------------------------------------------------------------
namespace {
typedef CUresult (*PFN_memop32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_memop32 g_wait32 = nullptr, g_write32 = nullptr;
std::once_flag g_memops_once;
int g_memops_status = (int)cudaErrorNotSupported;

void load_memops() {
  cudaDriverEntryPointQueryResult q1, q2;
  cudaError_t e1 = cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", (void**)&g_wait32, 12000,
                                                    cudaEnableDefault, &q1);
  cudaError_t e2 = cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", (void**)&g_write32, 12000,
                                                    cudaEnableDefault, &q2);
  if (e1 == cudaSuccess && e2 == cudaSuccess && q1 == cudaDriverEntryPointSuccess &&
      q2 == cudaDriverEntryPointSuccess && g_wait32 && g_write32)
    g_memops_status = 0;
  else
    g_memops_status = (int)cudaErrorNotSupported;
  cudaGetLastError();
}
}  // namespace

int cs_stream_memops_supported(void) {
  // 32-bit wait / write stream memory operations (the v2 API) are part of the CUDA 12 driver on
  // every supported GPU; the legacy CAN_USE_STREAM_MEM_OPS_V1 attribute describes the v1 API
  // only, so availability = the entry points resolve.
  std::call_once(g_memops_once, load_memops);
  return g_memops_status == 0 ? 1 : 0;
}

int cs_flag_barrier(const uint64_t* peer_rows, uint64_t local_row, int rank, int nranks,
                    void* stream) {
  if (peer_rows == nullptr || local_row == 0 || nranks < 1 || nranks > CS_MAX_SOURCES ||
      rank < 0 || rank >= nranks)
    return set_error(CS_ERR_ARG, "cs_flag_barrier: invalid arguments");
  for (int p = 0; p < nranks; ++p)
    if (p != rank && peer_rows[p] == 0)
      return set_error(CS_ERR_ARG, "cs_flag_barrier: NULL flag row of rank %d", p);
  std::call_once(g_memops_once, load_memops);
  if (g_memops_status)
    return set_error(g_memops_status, "cs_flag_barrier: stream memory operations unavailable");
  CUstream s = (CUstream)stream;
  // When the device can flush remote writes, each wait also makes every write that reached this
  // GPU before the flag (a peer's NVLink stores into my parameters) visible to the work queued
  // behind it.  Without the attribute the ordering comes from the writer: its flag write is
  // preceded by a system-scope fence, so its earlier peer stores land first.
  static int flush_cache[64] = {0};   // per device: 0 unknown, 1 no, 2 yes
  int dev = 0, can_flush = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
    if (flush_cache[dev] == 0) {
      int v = 0;
      if (cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, dev) != cudaSuccess) {
        cudaGetLastError();
        v = 0;
      }
      flush_cache[dev] = v ? 2 : 1;
    }
    can_flush = flush_cache[dev] == 2;
  }
  const unsigned int wait_flags = CU_STREAM_WAIT_VALUE_EQ | (can_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0u);
  // arrive: 1 into my slot of every peer's row (a system-scope fence precedes each write, so
  // everything this stream did before is visible to the peer that observes the flag)
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    CUresult r = g_write32(s, (CUdeviceptr)(peer_rows[p] + 4u * (uint64_t)rank), 1u, 0);
    if (r != CUDA_SUCCESS) return set_error((int)r, "cs_flag_barrier: write to rank %d failed (%d)", p, (int)r);
  }
  // wait: every peer's slot in my row is 1
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    CUresult r = g_wait32(s, (CUdeviceptr)(local_row + 4u * (uint64_t)p), 1u, wait_flags);
    if (r != CUDA_SUCCESS) return set_error((int)r, "cs_flag_barrier: wait on rank %d failed (%d)", p, (int)r);
  }
  // reset my row (only this rank reads it, in stream order; the v2 write API has no
  // no-barrier flag, so each reset carries the default fence)
  for (int p = 0; p < nranks; ++p) {
    if (p == rank) continue;
    CUresult r = g_write32(s, (CUdeviceptr)(local_row + 4u * (uint64_t)p), 0u, 0);
    if (r != CUDA_SUCCESS) return set_error((int)r, "cs_flag_barrier: reset of slot %d failed (%d)", p, (int)r);
  }
  return 0;
}

int cs_host_register(void* ptr, size_t bytes, void** dev_ptr) {
  if (ptr == nullptr || bytes == 0 || dev_ptr == nullptr)
    return set_error(CS_ERR_ARG, "cs_host_register: invalid arguments");
  int rc = cuda_status(cudaHostRegister(ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable),
                       "cudaHostRegister");
  if (rc) return rc;
  rc = cuda_status(cudaHostGetDevicePointer(dev_ptr, ptr, 0), "cudaHostGetDevicePointer");
  if (rc) cudaHostUnregister(ptr);
  return rc;
}

int cs_host_unregister(void* ptr) {
  if (ptr == nullptr) return 0;
  return cuda_status(cudaHostUnregister(ptr), "cudaHostUnregister");
}

int cs_ipc_close_handle(void* ptr) {
  if (ptr == nullptr) return 0;
  return cuda_status(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

int cs_ipc_base_of(const void* ptr, void** base, size_t* size) {
  if (ptr == nullptr || base == nullptr || size == nullptr)
    return set_error(CS_ERR_ARG, "cs_ipc_base_of: NULL argument");
  typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", (void**)&range, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      range = nullptr;
    cudaGetLastError();
  });
  if (range == nullptr) return set_error((int)cudaErrorNotSupported, "cs_ipc_base_of: no cuMemGetAddressRange");
  CUdeviceptr b = 0;
  size_t n = 0;
  const CUresult r = range(&b, &n, (CUdeviceptr)ptr);
  if (r != CUDA_SUCCESS) return set_error((int)r, "cs_ipc_base_of(%p): cuMemGetAddressRange failed (%d)", ptr, (int)r);
  *base = (void*)b;
  *size = n;
  return 0;
}

int64_t cs_p2p_gather_chunk_elems(int nranks) {
  if (nranks < 1 || nranks > CS_MAX_SOURCES) return 0;
  return p2p_gather_chunk_elems(nranks);
}

int cs_p2p_gather_check(const cs_p2p_desc* chunks, int64_t nchunks, int nranks, int momentum) {
  if ((nchunks > 0 && chunks == nullptr) || nchunks < 0) return set_error(CS_ERR_ARG, "cs_p2p_gather_check: bad table");
  if (nranks < 1 || nranks > CS_MAX_SOURCES)
    return set_error(CS_ERR_ARG, "cs_p2p_gather_check: nranks=%d outside [1, %d]", nranks, CS_MAX_SOURCES);
  const int64_t ch = p2p_gather_chunk_elems(nranks);
  for (int64_t i = 0; i < nchunks; ++i) {
    const cs_p2p_desc& d = chunks[i];
    if (d.nranks != nranks || d.numel <= 0 || d.numel > ch || d.param == nullptr ||
        (momentum && d.momentum_buf == nullptr))
      return set_error(CS_ERR_ARG, "cs_p2p_gather_check: chunk %lld malformed", (long long)i);
    uintptr_t al = (uintptr_t)d.param | (uintptr_t)d.momentum_buf;
    for (int r = 0; r < nranks; ++r) {
      if (d.src[r] == 0 || d.dst[r] == 0)
        return set_error(CS_ERR_ARG, "cs_p2p_gather_check: chunk %lld: NULL address of rank %d", (long long)i, r);
      al |= (uintptr_t)d.src[r] | (uintptr_t)d.dst[r];
    }
    if (al & 15u) return set_error(CS_ERR_ARG, "cs_p2p_gather_check: chunk %lld not 16-byte aligned", (long long)i);
  }
  return 0;
}

int cs_p2p_gather_reduce_sgd_bcast(const cs_p2p_desc* chunks_dev, int64_t nchunks, int nranks, int max_ctas,
                                   const cs_sgd_hyper* h, void* stream) {
  if (h == nullptr || (nchunks > 0 && chunks_dev == nullptr) || nchunks < 0)
    return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: NULL argument");
  if (((uintptr_t)chunks_dev & 15u) != 0)
    return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: chunk table not 16-byte aligned");
  if (nranks < 1 || nranks > CS_MAX_SOURCES || max_ctas < 0)
    return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: bad nranks / max_ctas");
  if (h->divisor != nranks)
    return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: divisor %d != nranks %d", h->divisor, nranks);
  if (!(h->lr > 0.0f)) return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: learning rate must be > 0");
  if (h->rounding == CS_ROUND_REFERENCE && (h->momentum != 0.0f || h->weight_decay != 0.0f))
    return set_error(CS_ERR_ARG, "cs_p2p_gather_reduce_sgd_bcast: reference rounding has no momentum / weight decay");
  return cuda_status(launch_p2p_gather(chunks_dev, nchunks, nranks, max_ctas, *h, (cudaStream_t)stream),
                     "cs_p2p_gather_reduce_sgd_bcast launch");
}

size_t cs_bn_workspace_bytes(int64_t M, int C) {
  if (M <= 0 || C <= 0 || C % 8) return 0;
  return bn_workspace_bytes(M, C);
}

static bool bn_shape_ok(int64_t M, int C) {
  return M > 0 && C > 0 && C % 8 == 0 && (C <= 256 || C % 256 == 0);
}

int cs_bn_forward(const void* x, const void* residual, int64_t M, int C, const float* weight,
                  const float* bias, float* running_mean, float* running_var, float momentum,
                  float eps, float* save_mean, float* save_invstd, float* scale_shift, void* y,
                  void* workspace, int flags, void* stream) {
  const bool resid = flags & CS_BN_RESIDUAL;
  if (x == nullptr || y == nullptr || save_mean == nullptr || save_invstd == nullptr ||
      scale_shift == nullptr || workspace == nullptr || !bn_shape_ok(M, C) ||
      (flags & ~(CS_BN_RELU | CS_BN_RESIDUAL)) || (resid && residual == nullptr) ||
      (((uintptr_t)x | (uintptr_t)y | (uintptr_t)residual) & 15u) ||
      ((running_mean == nullptr) != (running_var == nullptr)))
    return set_error(CS_ERR_ARG, "cs_bn_forward: invalid arguments (M=%lld C=%d flags=%d)",
                     (long long)M, C, flags);
  return cuda_status(launch_bn_fwd(x, residual, M, C, weight, bias, running_mean, running_var,
                                   momentum, eps, save_mean, save_invstd, scale_shift, y,
                                   workspace, flags, (cudaStream_t)stream),
                     "cs_bn_forward launch");
}

int cs_bn_backward2(const void* dy, const void* dy2, const void* x, const void* residual, int64_t M,
                    int C, const float* save_mean, const float* save_invstd,
                    const float* scale_shift, const float* weight, float* grad_weight,
                    float* grad_bias, float* coef, void* dx, void* dresidual, void* workspace,
                    int flags, void* stream) {
  const bool relu = flags & CS_BN_RELU, resid = flags & CS_BN_RESIDUAL;
  if (dy == nullptr || x == nullptr || dx == nullptr || save_mean == nullptr ||
      save_invstd == nullptr || coef == nullptr || workspace == nullptr || !bn_shape_ok(M, C) ||
      (flags & ~(CS_BN_RELU | CS_BN_RESIDUAL)) || (relu && scale_shift == nullptr) ||
      (resid && (dresidual == nullptr || (relu && residual == nullptr))) ||
      (((uintptr_t)dy | (uintptr_t)dy2 | (uintptr_t)x | (uintptr_t)dx | (uintptr_t)residual |
        (uintptr_t)dresidual) & 15u))
    return set_error(CS_ERR_ARG, "cs_bn_backward: invalid arguments (M=%lld C=%d flags=%d)",
                     (long long)M, C, flags);
  return cuda_status(launch_bn_bwd(dy, dy2, x, residual, M, C, save_mean, save_invstd, scale_shift,
                                   weight, grad_weight, grad_bias, coef, dx, dresidual, workspace,
                                   flags, (cudaStream_t)stream),
                     "cs_bn_backward launch");
}

int cs_bn_backward(const void* dy, const void* x, const void* residual, int64_t M, int C,
                   const float* save_mean, const float* save_invstd, const float* scale_shift,
                   const float* weight, float* grad_weight, float* grad_bias, float* coef,
                   void* dx, void* dresidual, void* workspace, int flags, void* stream) {
  return cs_bn_backward2(dy, nullptr, x, residual, M, C, save_mean, save_invstd, scale_shift, weight,
                         grad_weight, grad_bias, coef, dx, dresidual, workspace, flags, stream);
}

static bool pool_shape_ok(const int* s) {
  if (s == nullptr) return false;
  for (int i = 0; i < 10; ++i)
    if (s[i] <= 0) return false;
  if (s[10] < 0 || s[11] < 0 || s[3] % 8 || s[6] * s[7] > 256) return false;
  return s[4] == (s[1] + 2 * s[10] - s[6]) / s[8] + 1 && s[5] == (s[2] + 2 * s[11] - s[7]) / s[9] + 1;
}

int cs_maxpool2d_forward(const void* x, void* y, uint8_t* argmax, const int* shape, void* stream) {
  if (x == nullptr || y == nullptr || argmax == nullptr || !pool_shape_ok(shape) ||
      (((uintptr_t)x | (uintptr_t)y) & 15u) || ((uintptr_t)argmax & 7u))
    return set_error(CS_ERR_ARG, "cs_maxpool2d_forward: invalid arguments");
  return cuda_status(launch_maxpool_fwd(x, y, argmax, shape, (cudaStream_t)stream),
                     "cs_maxpool2d_forward launch");
}

int cs_im2col_nhwc(const void* x, void* patches, const int* s, void* stream) {
  bool ok = x != nullptr && patches != nullptr && s != nullptr && !(((uintptr_t)patches) & 15u);
  if (ok) {
    for (int i = 0; i < 10; ++i) ok = ok && s[i] > 0;
    ok = ok && s[10] >= 0 && s[11] >= 0 && s[12] > 0 && s[12] % 8 == 0 && s[12] >= s[3] * s[6] * s[7] &&
         s[4] == (s[1] + 2 * s[10] - s[6]) / s[8] + 1 && s[5] == (s[2] + 2 * s[11] - s[7]) / s[9] + 1 &&
         (int64_t)s[0] * s[4] * s[5] * (s[12] / 8) < (int64_t)INT32_MAX &&
         (int64_t)s[0] * s[1] * s[2] * s[3] < (int64_t)INT32_MAX * 8;
  }
  if (!ok) return set_error(CS_ERR_ARG, "cs_im2col_nhwc: invalid arguments");
  return cuda_status(launch_im2col_nhwc(x, patches, s, (cudaStream_t)stream), "cs_im2col_nhwc launch");
}

int cs_maxpool2d_backward(const void* dy, const uint8_t* argmax, void* dx, const int* shape,
                          void* stream) {
  if (dy == nullptr || dx == nullptr || argmax == nullptr || !pool_shape_ok(shape) ||
      (((uintptr_t)dy | (uintptr_t)dx) & 15u) || ((uintptr_t)argmax & 7u))
    return set_error(CS_ERR_ARG, "cs_maxpool2d_backward: invalid arguments");
  return cuda_status(launch_maxpool_bwd(dy, argmax, dx, shape, (cudaStream_t)stream),
                     "cs_maxpool2d_backward launch");
}

// ---- streams and events: the pipeline primitives for hosts without torch ----
int cs_stream_create(int priority, void** stream) {
  if (stream == nullptr) return set_error(CS_ERR_ARG, "cs_stream_create: NULL argument");
  cudaStream_t s = nullptr;
  int rc = cuda_status(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority),
                       "cudaStreamCreateWithPriority");
  if (rc) return rc;
  *stream = (void*)s;
  return 0;
}

int cs_stream_destroy(void* stream) {
  if (stream == nullptr) return 0;
  return cuda_status(cudaStreamDestroy((cudaStream_t)stream), "cudaStreamDestroy");
}

int cs_stream_synchronize(void* stream) {
  return cuda_status(cudaStreamSynchronize((cudaStream_t)stream), "cudaStreamSynchronize");
}

int cs_event_create(int timing, void** event) {
  if (event == nullptr) return set_error(CS_ERR_ARG, "cs_event_create: NULL argument");
  cudaEvent_t e = nullptr;
  int rc = cuda_status(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming),
                       "cudaEventCreateWithFlags");
  if (rc) return rc;
  *event = (void*)e;
  return 0;
}

int cs_event_destroy(void* event) {
  if (event == nullptr) return 0;
  return cuda_status(cudaEventDestroy((cudaEvent_t)event), "cudaEventDestroy");
}

int cs_event_record(void* event, void* stream) {
  if (event == nullptr) return set_error(CS_ERR_ARG, "cs_event_record: NULL event");
  return cuda_status(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream), "cudaEventRecord");
}

int cs_stream_wait_event(void* stream, void* event) {
  if (event == nullptr) return set_error(CS_ERR_ARG, "cs_stream_wait_event: NULL event");
  return cuda_status(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0),
                     "cudaStreamWaitEvent");
}

int cs_event_query(void* event) {
  if (event == nullptr) return set_error(CS_ERR_ARG, "cs_event_query: NULL event");
  const cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaSuccess) return 1;
  if (e == cudaErrorNotReady) { cudaGetLastError(); return 0; }
  return cuda_status(e, "cudaEventQuery");
}

int cs_event_elapsed_ns(void* start, void* end, int64_t* ns) {
  if (start == nullptr || end == nullptr || ns == nullptr)
    return set_error(CS_ERR_ARG, "cs_event_elapsed_ns: NULL argument");
  float ms = 0.f;
  int rc = cuda_status(cudaEventElapsedTime(&ms, (cudaEvent_t)start, (cudaEvent_t)end),
                       "cudaEventElapsedTime");
  if (rc) return rc;
  *ns = (int64_t)llround((double)ms * 1e6);
  return 0;
}

int cs_spin_ns(uint64_t ns, void* stream) {
  if (ns > 60ull * 1000000000ull) return set_error(CS_ERR_ARG, "cs_spin_ns: more than 60 s");
  return cuda_status(launch_spin_ns(ns, (cudaStream_t)stream), "cs_spin_ns launch");
}

size_t cs_gradient_stats_workspace_bytes(int64_t numel) {
  return 256 + (size_t)stats_grid(numel) * 2 * sizeof(double);
}

int cs_gradient_stats(const float* data, int64_t numel, double* out, void* workspace,
                      void* stream) {
  if (numel < 0 || out == nullptr || workspace == nullptr || (numel > 0 && data == nullptr))
    return set_error(CS_ERR_ARG, "cs_gradient_stats: invalid arguments");
  return cuda_status(launch_stats(data, numel, out, workspace, (cudaStream_t)stream),
                     "cs_gradient_stats launch");
}

}  // extern "C"
