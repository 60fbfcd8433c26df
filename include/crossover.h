/*
 * crossover.h -- C-ABI of libcrossover.so, the B200-native crossover step.
 *
 * The reference (colosim, /root/reference/pkg/src/colosim) is pure Python and
 * has no FFI.  These entry points are the calls its Python API would bind
 * (ctypes) to execute the crossover step on the device instead of pricing it:
 *
 *   cs_pack            replaces  workload.fuse_gradients     (workload.py:94-101)
 *                                the payload sum becomes a real gather of every
 *                                gradient tensor into one contiguous bucket.
 *   cs_unpack_sgd      replaces  equivalence.average_gradients (equivalence.py:150-160)
 *                           +    equivalence.sgd_step          (equivalence.py:163-168)
 *                                fixed left-to-right sum over sources, divide by
 *                                the worker count, SGD(-momentum) update, in place.
 *   cs_nccl_*          replaces  comm.comm_time_allreduce       (comm.py:87-99)
 *                                the alpha-beta price becomes a measured NCCL
 *                                all-reduce on the caller's comm stream.
 *   cs_gradient_stats  new       warp-reduced sum of squares / non-finite count
 *                                over a bucket (gradient health, checksums).
 *
 * Conventions
 *   - Ownership: every device buffer (gradients, buckets, parameters, momentum
 *     buffers, snapshots) is allocated and owned by the caller.  The library
 *     never allocates on the step path and never frees caller memory.
 *   - Streams: `stream` is a cudaStream_t passed as void*; NULL = legacy default.
 *     Every call is an asynchronous enqueue; nothing blocks the host.
 *   - Descriptor arrays are HOST memory; they are copied into kernel parameters
 *     at launch (no device-side tables, no per-step H2D copies).
 *   - Errors: 0 on success; CS_ERR_ARG (<0) for invalid arguments; otherwise a
 *     cudaError_t value or CS_ERR_NCCL_BASE + ncclResult_t.  cs_last_error()
 *     returns a thread-local message for the last failure on this thread.
 *   - Threading: one host thread per process (one process per GPU).  Calls on
 *     distinct streams are reentrant.
 */
#ifndef CROSSOVER_H_
#define CROSSOVER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CS_API __attribute__((visibility("default")))
#else
#define CS_API
#endif

#define CS_ABI_VERSION 3
#define CS_ERR_ARG (-1)
#define CS_ERR_NCCL_BASE 10000
#define CS_NCCL_UNIQUE_ID_BYTES 128
#define CS_MAX_SOURCES 8

/* One gradient tensor to gather: src[0:numel) -> dst[0:numel). */
typedef struct cs_pack_desc {
  const float* src;   /* device pointer of the gradient tensor (contiguous fp32) */
  float* dst;         /* device pointer inside the bucket (bucket + offset)      */
  int64_t numel;      /* elements; 0 is allowed (skipped)                         */
} cs_pack_desc;

/* One parameter tensor to update from the reduced gradient. */
typedef struct cs_update_desc {
  float* param;          /* device pointer, updated in place                      */
  float* momentum_buf;   /* device pointer or NULL when momentum == 0             */
  uint64_t grad_offset;  /* byte offset added to every source base (see below)    */
  uint64_t snap_offset;  /* byte offset into `snapshot` (ignored if snapshot NULL) */
  int64_t numel;
} cs_update_desc;

/* Update rule.  rounding = CS_ROUND_REFERENCE reproduces equivalence.sgd_step's
 * `p - lr * avg` (two roundings, no FMA; momentum/weight_decay must be 0).
 * rounding = CS_ROUND_TORCH reproduces torch.optim.SGD's single-tensor update
 * (weight decay, momentum/dampening/nesterov, `p.add_(d, alpha=-lr)` as FMA). */
enum { CS_ROUND_REFERENCE = 0, CS_ROUND_TORCH = 1 };

typedef struct cs_sgd_hyper {
  float lr;
  float momentum;
  float dampening_complement;  /* 1 - dampening, rounded once from double (ATen's alpha) */
  float weight_decay;
  int32_t nesterov;
  int32_t first_step;  /* momentum buffer is initialised to the gradient      */
  int32_t divisor;     /* worker count W: the summed gradient is divided by W */
  int32_t rounding;    /* CS_ROUND_REFERENCE or CS_ROUND_TORCH                */
} cs_sgd_hyper;

CS_API int cs_abi_version(void);
CS_API const char* cs_last_error(void);

/* Launch-shape knobs (0 restores the built-in default): of the register K1/K2 "reg_shape"
 * (0..4: unroll x CTAs/SM); of the fused P2P kernel: "p2p_ctas" (persistent grid cap, 0 = default
 * 2 CTAs per SM) and "p2p_bulk" (1, the default: a launch with max_ctas > 0 streams tiles through
 * shared memory with cp.async.bulk; 0: the register kernel); of the K1/K2: "sync_ctas" (persistent grid cap, default 0 = one CTA per chunk) -- a
 * sync that overlaps another app's compute with slack can trade speed for fewer SMs; of the BN
 * kernels: "bn_no_pdl" (1 = launch finalize / apply without programmatic dependent launch),
 * "bn_ctas_per_sm" (row-block CTAs per SM of the partial kernels, 0 = 3; changes the partial
 * merge tree, so results are deterministic per setting but not bitwise across settings).
 * Results never depend on them (except bn_ctas_per_sm, see above). */
CS_API int cs_tune(const char* key, int value);

/* Streams and events -- the crossover pipeline's primitives for hosts without torch
 * (reference lanes / events, engine.py:62-86): gpu0 = compute stream, nic0 = comm stream,
 * COMPUTE_DONE / COMM_DONE = recorded events, span times = cs_event_elapsed_ns against an
 * origin event.  cs_event_query returns 1 (complete), 0 (pending) or an error code. */
CS_API int cs_stream_create(int priority, void** stream);
CS_API int cs_stream_destroy(void* stream);
CS_API int cs_stream_synchronize(void* stream);
CS_API int cs_event_create(int timing, void** event);
CS_API int cs_event_destroy(void* event);
CS_API int cs_event_record(void* event, void* stream);
CS_API int cs_stream_wait_event(void* stream, void* event);
CS_API int cs_event_query(void* event);
CS_API int cs_event_elapsed_ns(void* start, void* end, int64_t* ns);

/* K1: gather n tensors into the bucket (128-bit vector path when src and dst
 * are 16-byte aligned, scalar otherwise).  Bit-exact copy.
 * max_ctas: 0 = one CTA per 4096-element chunk (or the cs_tune("sync_ctas") cap); > 0 = a
 * persistent grid of at most max_ctas CTAs -- what a sync overlapping another app's compute on a
 * high-priority stream should use, so the other stream's CTAs are not held back behind thousands of
 * pending high-priority ones.  Results never depend on it (same for cs_unpack_sgd). */
CS_API int cs_pack(const cs_pack_desc* descs, int n, int max_ctas, void* stream);

/* K2: for every tensor i and element k
 *     acc  = 0 + g_0 + g_1 + ... + g_{S-1}   (left to right over sources)
 *     avg  = acc / divisor                      (IEEE division, == equivalence.py:160)
 *     param, momentum_buf <- SGD(param, avg)   (see cs_sgd_hyper)
 * where g_s = *(const float*)(sources[s] + descs[i].grad_offset + 4k).
 * `sources` is a HOST array of n_sources (1..CS_MAX_SOURCES) device byte
 * addresses: a reduced bucket (after all-reduce), the rows of a simulated-worker
 * staging buffer, or {0} with grad_offset = raw gradient pointer (W = 1, no bucket).
 * If snapshot != NULL the updated parameter is also written to
 * snapshot + snap_offset (per-iteration weight capture for parity). */
CS_API int cs_unpack_sgd(const cs_update_desc* descs, int n, const uint64_t* sources,
                  int n_sources, float* snapshot, const cs_sgd_hyper* hyper, int max_ctas,
                  void* stream);

/* Gradient health over a contiguous fp32 range: out[0] += sum of squares
 * (fp64), out[1] += count of non-finite values.  Deterministic: per-CTA
 * partials are reduced in a fixed order by the last CTA.  `workspace` must hold
 * cs_gradient_stats_workspace_bytes(numel) bytes (device, caller-owned, zeroed
 * once before first use; the kernel leaves it zeroed again). */
CS_API size_t cs_gradient_stats_workspace_bytes(int64_t numel);
CS_API int cs_gradient_stats(const float* data, int64_t numel, double* out,
                      void* workspace, void* stream);

/* A compute phase of known device duration: one thread on one SM spins on %globaltimer for `ns`
 * nanoseconds (no memory traffic).  The fixed compute kernel of the comm/comp sweep and of the
 * timing-level schedule tests (reference: JobProfile.forward_time / backward_time as durations,
 * workload.py:43-56).  At most 60 s. */
CS_API int cs_spin_ns(uint64_t ns, void* stream);

/* Collective-fused update over NVLink peer memory (replaces reduce-scatter + K2 +
 * all-gather).  For this rank's shard of an app's flat parameters:
 *   acc = 0 + src[0][k] + ... + src[W-1][k]   (rank order == equivalence.py:156-159)
 *   p   = SGD(p, acc / W)                      (cs_sgd_hyper rules; momentum shard local)
 *   dst[r][k] = p  for every rank r            (fused all-gather; remote NVLink stores)
 * src[r] / dst[r] are rank r's bucket shard / flat-parameter shard as mapped in THIS
 * process (cs_ipc_open_handle for peers).  The caller orders it between two barriers. */
typedef struct cs_p2p_desc {
  uint64_t src[CS_MAX_SOURCES];
  uint64_t dst[CS_MAX_SOURCES];
  float* param;          /* this rank's parameter shard (== dst[rank]) */
  float* momentum_buf;   /* this rank's momentum shard, NULL when momentum == 0 */
  int64_t numel;         /* shard length (fp32 elements) */
  int32_t nranks;        /* W, 2..CS_MAX_SOURCES */
  int32_t max_ctas;      /* persistent grid cap for this launch; 0 = cs_tune("p2p_ctas") or
                            2 CTAs per SM.  A sync that overlaps another app's compute with slack
                            should hold few SMs (the scheduler uses 32 under crossover). */
} cs_p2p_desc;
CS_API int cs_p2p_reduce_sgd_bcast(const cs_p2p_desc* desc, const cs_sgd_hyper* hyper,
                                   void* stream);

/* The same update without K1 ("p2p_gather"): every rank's GRADIENT TENSORS are read in place over
 * NVLink (no bucket, no pack).  This rank's shard of the bucket layout is cut into chunks that
 * never cross a gradient tensor, at most cs_p2p_gather_chunk_elems(nranks) elements each; chunk i
 * is a cs_p2p_desc whose src[r] points at the chunk inside rank r's gradient tensor (mapped in
 * this process), dst[r] / param / momentum_buf at the chunk's place in the flat parameters /
 * momentum shard, numel its length.  Arithmetic and sum order are cs_p2p_reduce_sgd_bcast's, so
 * the result is bit-identical to it (and to K1 + p2p).  Gradients must stay at these addresses
 * while syncs run (CUDA-graphed backward passes).  cs_p2p_gather_check validates a host copy of
 * the table; the launch takes a device copy (16-byte aligned). */
CS_API int64_t cs_p2p_gather_chunk_elems(int nranks);
CS_API int cs_p2p_gather_check(const cs_p2p_desc* chunks, int64_t nchunks, int nranks, int momentum);
CS_API int cs_p2p_gather_reduce_sgd_bcast(const cs_p2p_desc* chunks_dev, int64_t nchunks, int nranks,
                                          int max_ctas, const cs_sgd_hyper* hyper, void* stream);

/* Collective-fused update through NVSwitch multicast (NVLS): same contract as
 * cs_p2p_reduce_sgd_bcast, but the W-rank sum is a multimem.ld_reduce on the multicast mapping of
 * the buckets (the switch adds; its order is unspecified, so results match the rank-order
 * transports within fp32 rounding, not bitwise) and the new shard is a multimem.st into the
 * multicast mapping of the flat parameters (the switch writes every rank's copy).
 * mc_bucket / mc_param: this rank's shard in the multicast mappings; param: the same shard in the
 * local (unicast) mapping.  numel % 4 == 0.  The caller orders it between two barriers. */
typedef struct cs_nvls_desc {
  const float* mc_bucket;
  float* mc_param;
  float* param;
  float* momentum_buf;   /* this rank's momentum shard, NULL when momentum == 0 */
  int64_t numel;
  int32_t nranks;
  int32_t max_ctas;      /* persistent grid cap, 0 = 2 CTAs per SM */
} cs_nvls_desc;
CS_API int cs_nvls_reduce_sgd_bcast(const cs_nvls_desc* desc, const cs_sgd_hyper* hyper, void* stream);
/* Multicast objects and the physical memory bound to them (driver entry points resolved at run
 * time).  Rank 0 creates the object and exports it as a POSIX file descriptor; the other ranks
 * import it; every rank adds its device, then (after all ranks added theirs) allocates, binds and
 * maps its memory twice: unicast (uc_ptr, local accesses) and multicast (mc_ptr, multimem ops). */
CS_API int cs_nvls_supported(int device);
CS_API int cs_nvls_granularity(int nranks, size_t bytes, size_t* gran);
CS_API int cs_nvls_create(int nranks, size_t bytes, uint64_t* mc, int* fd);
CS_API int cs_nvls_import(int fd, uint64_t* mc);
CS_API int cs_nvls_add_device(uint64_t mc, int device);
CS_API int cs_nvls_alloc_bind(uint64_t mc, int device, size_t bytes, size_t gran, uint64_t* phys,
                              void** uc_ptr, void** mc_ptr);
CS_API int cs_nvls_free(uint64_t mc, int device, uint64_t phys, void* uc_ptr, void* mc_ptr, size_t bytes);
CS_API int cs_nvls_release(uint64_t mc);

/* IPC-capable device memory (cudaMalloc'd, zero-filled) and its peer mapping. */
#define CS_IPC_HANDLE_BYTES 64
CS_API int cs_device_alloc(size_t bytes, void** ptr);
CS_API int cs_device_free(void* ptr);
CS_API int cs_ipc_get_handle(void* ptr, uint8_t* out /* CS_IPC_HANDLE_BYTES */);
CS_API int cs_ipc_open_handle(const uint8_t* handle, void** ptr);
CS_API int cs_ipc_close_handle(void* ptr);
/* Base address and size of the device allocation that contains ptr (cuMemGetAddressRange): the
 * IPC handle of a tensor inside a caching allocator's segment is its segment's handle plus the
 * offset ptr - base. */
CS_API int cs_ipc_base_of(const void* ptr, void** base, size_t* size);
/* Stream-ordered copy by the copy engines (cudaMemcpyAsync, cudaMemcpyDefault): src / dst may be
 * local or peer-mapped (IPC) device memory, so a pull from a peer crosses NVLink without
 * occupying any SM -- the transport of the "ce" sync mode. */
CS_API int cs_copy_async(void* dst, const void* src, size_t bytes, void* stream);
/* Cross-rank barrier without SMs: stream memory operations on uint32 flag rows (host shared
 * memory registered with cs_host_register, or IPC-mapped device memory), constant values only, so
 * the same sequence can be captured into a CUDA graph and replayed:
 *   arrive  write 1 into slot `rank` of every peer's row (peer_rows[p] = rank p's row as mapped
 *           here; a system-scope fence orders all earlier work of the stream before each write)
 *   wait    until every peer's slot in this rank's row (local_row) is 1
 *   reset   write 0 into this rank's row
 * A transport that needs two barriers per sync (p2p, ce) uses two separate rows ("phases") per
 * rank and always passes them in the same order: a peer can only arrive at phase X again after
 * passing the other phase, which this rank enters only after it reset phase X -- so no arrival
 * is lost and no reset erases a fresh one.  Replaces the 1-element NCCL all-reduce barriers, whose
 * kernels need a free SM while the other app's GEMMs occupy them. */
CS_API int cs_stream_memops_supported(void);
/* Page-locked, device-mapped host memory for the flag arrays (cudaHostRegister, mapped +
 * portable).  The p2p / ce transports keep their barrier flags in one host shared-memory segment
 * mapped by every rank of the node, so a host can release every rank's pending waits on failure
 * (keep writing 1 into the segment until the streams drained) without issuing any GPU work. */
CS_API int cs_host_register(void* ptr, size_t bytes, void** dev_ptr);
CS_API int cs_host_unregister(void* ptr);
CS_API int cs_flag_barrier(const uint64_t* peer_rows, uint64_t local_row, int rank, int nranks,
                           void* stream);

/* channels_last BatchNorm2d (training) for the apps' compute: x / y / dy / dx / residual are
 * bf16 [M, C] row-major (M = N*H*W, C % 8 == 0, C <= 256 or C % 256 == 0), weight / bias /
 * running stats / saved stats fp32 [C].
 * Forward: per-channel mean / biased var (Welford + fixed-order Chan merge), running stats
 * updated with the unbiased variance (nn.BatchNorm2d momentum semantics), then the fused
 * epilogue y = act((x - mean) * invstd * w + b [+ residual]) with flags
 * CS_BN_RELU (act = max(., 0)) and CS_BN_RESIDUAL (add `residual` before the activation).
 * scale_shift: fp32 [2C] written by the forward (scale, shift) and read by the backward.
 * Backward: g = dy masked by the recomputed activation; grad_weight = sum(g * xhat),
 * grad_bias = sum(g), dx per torch's formula, dresidual = g (CS_BN_RESIDUAL).
 * coef: fp32 [3C] scratch.  workspace: cs_bn_workspace_bytes(M, C) bytes (caller-owned).
 * weight / bias / running stats / grads may be NULL. */
#define CS_BN_RELU 1
#define CS_BN_RESIDUAL 2
CS_API size_t cs_bn_workspace_bytes(int64_t M, int C);
CS_API int cs_bn_forward(const void* x, const void* residual, int64_t M, int C,
                         const float* weight, const float* bias, float* running_mean,
                         float* running_var, float momentum, float eps, float* save_mean,
                         float* save_invstd, float* scale_shift, void* y, void* workspace,
                         int flags, void* stream);
CS_API int cs_bn_backward(const void* dy, const void* x, const void* residual, int64_t M, int C,
                          const float* save_mean, const float* save_invstd,
                          const float* scale_shift, const float* weight, float* grad_weight,
                          float* grad_bias, float* coef, void* dx, void* dresidual,
                          void* workspace, int flags, void* stream);
/* cs_bn_backward with a second incoming gradient of the same output (dy2, bf16 [M, C], may be
 * NULL): g = (dy + dy2) is formed in fp32 inside the kernels, before the activation mask.  The
 * ResNet bottleneck delivers the identity-path gradient of a block's input this way instead of
 * materialising the autograd sum (one elementwise add kernel per block). */
CS_API int cs_bn_backward2(const void* dy, const void* dy2, const void* x, const void* residual,
                           int64_t M, int C, const float* save_mean, const float* save_invstd,
                           const float* scale_shift, const float* weight, float* grad_weight,
                           float* grad_bias, float* coef, void* dx, void* dresidual,
                           void* workspace, int flags, void* stream);

/* channels_last max pooling (bf16, C % 8 == 0, no dilation / ceil mode).
 * shape = {N, H, W, C, OH, OW, kh, kw, sh, sw, ph, pw}; argmax: uint8 [N*OH*OW*C] window
 * offsets (kh*kw <= 256) written by the forward, read by the backward (dx is fully written). */
CS_API int cs_maxpool2d_forward(const void* x, void* y, uint8_t* argmax, const int* shape,
                                void* stream);
CS_API int cs_maxpool2d_backward(const void* dy, const uint8_t* argmax, void* dx,
                                 const int* shape, void* stream);

/* Patch matrix of an NHWC bf16 image batch for a convolution as a GEMM (the models' RGB stem):
 * shape = {N, H, W, C, OH, OW, kh, kw, sh, sw, ph, pw, KP}; patches: bf16 [N*OH*OW, KP],
 * row m = output pixel (n, oh, ow), column j < kh*kw*C = x[n, oh*sh-ph+j/(kw*C), ow*sw-pw+(j/C)%kw,
 * j%C] (0 outside the image), columns >= kh*kw*C zero; KP % 8 == 0, patches 16-byte aligned. */
CS_API int cs_im2col_nhwc(const void* x, void* patches, const int* shape, void* stream);

/* NCCL communicator over NVLink / NVSwitch (one per process, one per job set).
 * min_ctas / max_ctas <= 0 leave NCCL's defaults. */
CS_API int cs_nccl_version(void);
CS_API int cs_nccl_get_unique_id(uint8_t* out /* CS_NCCL_UNIQUE_ID_BYTES */);
CS_API int cs_nccl_init(void** comm, int nranks, int rank, const uint8_t* id,
                 int min_ctas, int max_ctas);
CS_API int cs_nccl_allreduce_sum_f32(void* comm, const float* send, float* recv,
                              size_t count, void* stream);
CS_API int cs_nccl_reduce_scatter_sum_f32(void* comm, const float* send, float* recv,
                                   size_t recv_count, void* stream);
CS_API int cs_nccl_all_gather_f32(void* comm, const float* send, float* recv,
                           size_t send_count, void* stream);
CS_API int cs_nccl_async_error(void* comm);
CS_API int cs_nccl_abort(void* comm);   /* failure path: unblocks work waiting on a dead peer */
CS_API int cs_nccl_destroy(void* comm);

#ifdef __cplusplus
}
#endif

#endif /* CROSSOVER_H_ */
