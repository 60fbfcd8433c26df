// crossover_sgd.cuh -- the per-element update rule shared by every K2 variant.
#pragma once
#include <cuda_runtime.h>

#include "crossover.h"

namespace cs {

struct Rule {
  float lr, mu, one_minus_damp, wd;
  int nesterov, first, rounding;
  float divisor;
  float inv_divisor;   // exact 1/W when W is a power of two
  int div_mode;        // 0: W == 1, 1: W == 2^k (multiply by the exact reciprocal), 2: divide
  int has_mom;
};

// One element of the update.  Returns the new parameter and updates *buf.
__device__ __forceinline__ float sgd_elem(const Rule& r, float acc, float p, float* buf) {
  // equivalence.py:160  acc / len(grads).  For W = 2^k the product with the exact
  // reciprocal is the same correctly rounded value as the IEEE quotient (no FTZ), so
  // the slow division sequence only runs for other worker counts.
  float d = r.div_mode == 0 ? acc : r.div_mode == 1 ? __fmul_rn(acc, r.inv_divisor)
                                                    : __fdiv_rn(acc, r.divisor);
  if (r.rounding == CS_ROUND_REFERENCE) {
    // equivalence.py:167  parameters - learning_rate * averaged  (two roundings)
    return __fsub_rn(p, __fmul_rn(r.lr, d));
  }
  // torch.optim.SGD (_single_tensor_sgd): grad.add(param, alpha=wd);
  // buf.mul_(mu).add_(grad, alpha=1-damp); grad = grad.add(buf, alpha=mu) | buf;
  // param.add_(grad, alpha=-lr).  add(x, alpha=a) is one FMA in ATen (vec::fmadd).
  if (r.wd != 0.0f) d = __fmaf_rn(r.wd, p, d);
  if (r.has_mom) {
    float b = r.first ? d : __fmaf_rn(r.one_minus_damp, d, __fmul_rn(r.mu, *buf));
    *buf = b;
    d = r.nesterov ? __fmaf_rn(r.mu, b, d) : b;
  }
  return __fmaf_rn(-r.lr, d, p);
}

__device__ __forceinline__ Rule make_rule(const cs_sgd_hyper& h, bool has_mom) {
  Rule r;
  r.lr = h.lr;
  r.mu = h.momentum;
  r.one_minus_damp = h.dampening_complement;
  r.wd = h.weight_decay;
  r.nesterov = h.nesterov;
  r.first = h.first_step;
  r.rounding = h.rounding;
  r.divisor = (float)h.divisor;
  const bool pow2 = (h.divisor & (h.divisor - 1)) == 0;
  r.div_mode = h.divisor == 1 ? 0 : pow2 ? 1 : 2;
  r.inv_divisor = pow2 ? 1.0f / (float)h.divisor : 0.0f;
  r.has_mom = has_mom;
  return r;
}

}  // namespace cs
