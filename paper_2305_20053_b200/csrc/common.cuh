// common.cuh -- shared device helpers for the SAA engine (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define SDN_DEV __device__ __forceinline__

namespace sdn {

// ---------------------------------------------------------------------------
// activations (reference: ouukit surrogate.py:42-63; ELU is the BASELINE gap)
enum Act : int { ACT_IDENTITY = 0, ACT_TANH = 1, ACT_SOFTPLUS = 2, ACT_SIGMOID = 3, ACT_ELU = 4,
                 ACT_SOFTMAX = 5 /* per-layer vector softmax: row kernels, not elementwise */ };

// value and derivative of the activation at pre-activation s
SDN_DEV void act_eval(int act, float s, float& a, float& d) {
  switch (act) {
    case ACT_TANH: {
      a = tanhf(s);
      d = 1.0f - a * a;
      break;
    }
    case ACT_SOFTPLUS: {                 // log(1 + e^s), stable; d = sigmoid(s)
      a = fmaxf(s, 0.0f) + log1pf(expf(-fabsf(s)));
      d = 0.5f * (1.0f + tanhf(0.5f * s));
      break;
    }
    case ACT_SIGMOID: {
      a = 0.5f * (1.0f + tanhf(0.5f * s));
      d = a * (1.0f - a);
      break;
    }
    case ACT_ELU: {
      if (s > 0.0f) { a = s; d = 1.0f; }
      else { a = expm1f(s); d = expf(s); }
      break;
    }
    default: { a = s; d = 1.0f; }
  }
}

SDN_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SDN_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// smoothed plus (reference riskopt.py:26-49), evaluated in fp64
SDN_DEV double splus_d(double x, double eps) {
  if (x < 0.0) return 0.0;
  if (x >= eps) return x - 0.5 * eps;
  return x * x * x / (eps * eps) - x * x * x * x / (2.0 * eps * eps * eps);
}
SDN_DEV double splus_d1_d(double x, double eps) {
  if (x < 0.0) return 0.0;
  if (x >= eps) return 1.0;
  return 3.0 * x * x / (eps * eps) - 2.0 * x * x * x / (eps * eps * eps);
}

// order-preserving uint64 key of a double (larger value -> larger key);
// NaN maps above +inf so non-finite samples surface in the CVaR tail.
SDN_DEV uint64_t dkey(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v);
  if (v != v) return 0xFFFFFFFFFFFFFFFFull;
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// inverse of dkey (the NaN key maps back to a NaN)
SDN_DEV double dkey_inv(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

// activations in fp64 (Q refinement chain; oracle act_value)
SDN_DEV double act64(int act, double s) {
  switch (act) {
    case ACT_TANH: return tanh(s);
    case ACT_SOFTPLUS: return fmax(s, 0.0) + log1p(exp(-fabs(s)));
    case ACT_SIGMOID: return 1.0 / (1.0 + exp(-s));
    case ACT_ELU: return s > 0.0 ? s : expm1(s);
    default: return s;
  }
}

}  // namespace sdn
