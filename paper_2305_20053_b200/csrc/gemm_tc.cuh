// gemm_tc.cuh -- tcgen05 (TMEM accumulator, TMA-fed) GEMM back end.
// Interfaces used by engine.cu.  (Staged: this revision keeps the tensor-core
// path disabled; the SIMT back end serves every shape.)
#pragma once
#include "common.cuh"
#include <cuda_bf16.h>
#include <vector>

namespace sdn {

// a bf16x3-split operand: hi = bf16(x), lo = bf16(x - hi), row-major
struct TcOperand {
  __nv_bfloat16* hi = nullptr;
  __nv_bfloat16* lo = nullptr;
  int64_t rows = 0;
  int cols = 0;
};

struct TcWeights {
  bool enabled = false;
  std::vector<TcOperand> fwd, bwd;   // per layer: W (K-major) and W^T (K-major)
  TcOperand act[2];                  // activation / backward operands (ping-pong)
  TcOperand seed;                    // reverse-sweep seed E
  TcOperand mr;                      // encoded samples (layer-0 A operand)
};

// epilogue side-output: split the next-GEMM operand into bf16 hi/lo
struct TcEpiSplit {
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
  int64_t ld;
  TcEpiSplit(const TcOperand* op) : hi(op ? op->hi : nullptr), lo(op ? op->lo : nullptr), ld(op ? op->cols : 0) {}
  SDN_DEV void store(int64_t r, int c, float4 v) const {
    __nv_bfloat16 h0 = __float2bfloat16_rn(v.x), h1 = __float2bfloat16_rn(v.y);
    __nv_bfloat16 h2 = __float2bfloat16_rn(v.z), h3 = __float2bfloat16_rn(v.w);
    __nv_bfloat16 l0 = __float2bfloat16_rn(v.x - __bfloat162float(h0));
    __nv_bfloat16 l1 = __float2bfloat16_rn(v.y - __bfloat162float(h1));
    __nv_bfloat16 l2 = __float2bfloat16_rn(v.z - __bfloat162float(h2));
    __nv_bfloat16 l3 = __float2bfloat16_rn(v.w - __bfloat162float(h3));
    __nv_bfloat162* ph = reinterpret_cast<__nv_bfloat162*>(hi + r * ld + c);
    __nv_bfloat162* pl = reinterpret_cast<__nv_bfloat162*>(lo + r * ld + c);
    ph[0] = __halves2bfloat162(h0, h1); ph[1] = __halves2bfloat162(h2, h3);
    pl[0] = __halves2bfloat162(l0, l1); pl[1] = __halves2bfloat162(l2, l3);
  }
};

template <class Epi>
struct TcChain {
  Epi base;
  TcEpiSplit split;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float4 o = base.apply(r, c, v);
    if (split.hi) split.store(r, c, o);
  }
};

inline bool tc_gemm_supported(int64_t, int, int) { return false; }

template <class Epi>
inline int tc_gemm(cudaStream_t, int64_t, const int*, int, int, const TcOperand&, const TcOperand&, Epi) {
  return -1;
}

template <class H> inline int tc_alloc(H*, TcWeights& t) { t.enabled = false; return 0; }
inline void tc_free(TcWeights&) {}
template <class H> inline int tc_set_weights(H*, TcWeights&) { return 0; }
template <class H> inline int tc_set_samples(H*, TcWeights&, const float*, int64_t) { return 0; }
template <class H> inline int tc_split_seed(H*, TcWeights&, const float*, int64_t, const int*) { return 0; }

}  // namespace sdn
