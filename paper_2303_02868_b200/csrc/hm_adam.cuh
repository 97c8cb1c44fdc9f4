// The per-element Adam chain shared by the page-Adam kernels: the reference's
// numpy expression (hiermem/lockfree.py:135-141) one correctly rounded binary32
// op per operator, in its order, no contraction.
#pragma once
#include "hm_device.cuh"

namespace hm {

struct AdamScalars {
  float lr, b1, ob1, b2, ob2, eps, bc1, bc2, gscale;
};

__device__ __forceinline__ AdamScalars make_scalars(const hm_adam_hyper& h, const hm_group_rt& r) {
  AdamScalars s;
  s.lr = h.lr;
  s.b1 = h.beta1;
  s.ob1 = h.one_minus_beta1;
  s.b2 = h.beta2;
  s.ob2 = h.one_minus_beta2;
  s.eps = h.eps;
  s.bc1 = r.bc1;
  s.bc2 = r.bc2;
  s.gscale = r.gscale;
  return s;
}

__device__ __forceinline__ void adam_elem(const AdamScalars& s, float g, float& p, float& m,
                                          float& v) {
  g = __fmul_rn(g, s.gscale);  // x * 1.0f == x exactly: identity for parity runs
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.ob1, g));                  // lockfree.py:135
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(s.ob2, __fmul_rn(g, g)));    // :136
  const float mh = __fdiv_rn(m, s.bc1);                                    // :139
  const float vh = __fdiv_rn(v, s.bc2);                                    // :140
  const float den = __fadd_rn(__fsqrt_rn(vh), s.eps);                      // :141
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(s.lr, mh), den));
}

}  // namespace hm
