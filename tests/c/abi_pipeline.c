/* A host with no torch driving the crossover step through libcrossover.so alone.
 *
 *   gcc -O2 -I include tests/c/abi_pipeline.c -L paper_2103_07974_b200 -lcrossover \
 *       -Wl,-rpath,paper_2103_07974_b200 -L/usr/local/cuda/lib64 -lcudart -o abi_pipeline
 *
 * Two apps, one worker each (W = 1), three iterations in the crossover order: the "compute"
 * of app j is a host-written gradient copied to the device on the compute stream; its sync is
 * K1 pack -> K2 update on the comm stream, gated by events exactly like the Python pipeline.
 * The result is compared with the same arithmetic on the host (reference rounding: two
 * roundings, p - lr * (g / 1)), which must match bit for bit.  Exit 0 = pass.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "crossover.h"

#define CK(x) do { int rc_ = (x); if (rc_) { fprintf(stderr, "%s -> %d: %s\n", #x, rc_, cs_last_error()); return 1; } } while (0)
#define CU(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

enum { APPS = 2, T = 3, N0 = 1000, N1 = 4099 };

int main(void) {
  const int64_t numel[2] = {N0, N1};
  float *param[APPS][2], *grad[APPS][2], *bucket[APPS];
  static float host_p[APPS][2][N1], host_g[N1];
  void *cs, *ms, *bwd_done[APPS], *update_done[APPS];
  CK(cs_stream_create(0, &cs));
  CK(cs_stream_create(-1, &ms));
  for (int j = 0; j < APPS; ++j) {
    CK(cs_event_create(0, &bwd_done[j]));
    CK(cs_event_create(0, &update_done[j]));
    CU(cudaMalloc((void**)&bucket[j], (N0 + N1 + 64) * sizeof(float)));
    for (int t = 0; t < 2; ++t) {
      CU(cudaMalloc((void**)&param[j][t], numel[t] * sizeof(float)));
      CU(cudaMalloc((void**)&grad[j][t], numel[t] * sizeof(float)));
      for (int64_t k = 0; k < numel[t]; ++k) host_p[j][t][k] = 0.001f * (float)(k % 97) - 0.05f * j;
      CU(cudaMemcpy(param[j][t], host_p[j][t], numel[t] * sizeof(float), cudaMemcpyHostToDevice));
    }
  }
  const float lr = 0.125f;
  for (int it = 1; it <= T; ++it) {
    for (int j = 0; j < APPS; ++j) {            /* rotation slot (scheduler.py:106-122) */
      if (it > 1) CK(cs_stream_wait_event(cs, update_done[j]));  /* Alg. 1 readiness */
      for (int t = 0; t < 2; ++t) {
        for (int64_t k = 0; k < numel[t]; ++k) host_g[k] = 0.01f * (float)((k * (it + 3) + j) % 13) - 0.06f;
        CU(cudaMemcpyAsync(grad[j][t], host_g, numel[t] * sizeof(float), cudaMemcpyHostToDevice,
                           (cudaStream_t)cs));
        CU(cudaStreamSynchronize((cudaStream_t)cs));   /* host_g is reused */
        for (int64_t k = 0; k < numel[t]; ++k)      /* host mirror of K2 (reference rounding) */
          host_p[j][t][k] = host_p[j][t][k] - lr * (host_g[k] / 1.0f);
      }
      CK(cs_event_record(bwd_done[j], cs));
      CK(cs_stream_wait_event(ms, bwd_done[j]));
      cs_pack_desc pd[2] = {{grad[j][0], bucket[j], N0}, {grad[j][1], bucket[j] + 1024, N1}};
      CK(cs_pack(pd, 2, 0, ms));
      cs_update_desc ud[2];
      memset(ud, 0, sizeof(ud));
      ud[0].param = param[j][0]; ud[0].grad_offset = 0; ud[0].numel = N0;
      ud[1].param = param[j][1]; ud[1].grad_offset = 1024 * sizeof(float); ud[1].numel = N1;
      uint64_t src = (uint64_t)(uintptr_t)bucket[j];
      cs_sgd_hyper h;
      memset(&h, 0, sizeof(h));
      h.lr = lr; h.dampening_complement = 1.0f; h.divisor = 1; h.rounding = CS_ROUND_REFERENCE;
      CK(cs_unpack_sgd(ud, 2, &src, 1, NULL, &h, 0, ms));
      CK(cs_event_record(update_done[j], ms));
    }
  }
  CK(cs_stream_synchronize(ms));
  static float back[N1];
  for (int j = 0; j < APPS; ++j)
    for (int t = 0; t < 2; ++t) {
      CU(cudaMemcpy(back, param[j][t], numel[t] * sizeof(float), cudaMemcpyDeviceToHost));
      if (memcmp(back, host_p[j][t], numel[t] * sizeof(float)) != 0) {
        fprintf(stderr, "mismatch app %d tensor %d\n", j, t);
        return 1;
      }
    }
  int64_t ns = -1;
  void *e0, *e1;
  CK(cs_event_create(1, &e0));
  CK(cs_event_create(1, &e1));
  CK(cs_event_record(e0, ms));
  CK(cs_event_record(e1, ms));
  CK(cs_stream_synchronize(ms));
  CK(cs_event_elapsed_ns(e0, e1, &ns));
  if (ns < 0 || cs_event_query(e1) != 1) return 1;
  printf("abi_pipeline ok: %d apps x %d iterations bit-exact vs host, event clock %lld ns\n", APPS, T,
         (long long)ns);
  return 0;
}
