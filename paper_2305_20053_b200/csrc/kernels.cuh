// kernels.cuh -- QoI, risk moments, sample weights, compaction, radix
// selection and the gradient reductions of the SAA engine.
//
// Determinism: every reduction runs in a fixed order for a given sample
// count (fixed grids, fixed-order block combines, no float atomics), so the
// same inputs give bit-identical outputs run to run.
#pragma once
#include "common.cuh"
#include <cuda_bf16.h>

namespace sdn {

enum RiskKind : int { RISK_MEAN = 0, RISK_CVAR_SMOOTH = 1, RISK_MEANVAR = 2, RISK_CVAR_EXACT = 3,
                      RISK_UNIT = 100 /* per-sample G: w_i = 1 */,
                      RISK_BAND = 101, RISK_BAND_EXACT = 102 /* refinement band flags */ };

constexpr int STATS_LEN = 8;   // [n, sum q~, sum q~^2, sum splus, sum d1, n_active, 0, 0]

// Last-block reduction (fuses the k_sum_rows pass into the producing kernel):
// every block has written its w-wide partial row; the last block to finish
// sums the nb rows in a fixed order into out and re-arms the counter.  All
// threads of every block must call it.
SDN_DEV void last_block_sum(int* counter, int nb, int w, const double* part, double* out) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(counter, 1) == nb - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // one warp per field, lanes stride the rows, fixed butterfly (as k_sum_rows)
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int f = threadIdx.x >> 5; f < w; f += nw) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(part + (int64_t)b * w + f);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[f] = s;
  }
  if (threadIdx.x == 0) *counter = 0;
}

// zb = b1 + Pz z  (first-layer control contribution, W1_z V_z^T z, shared by
// every sample of the evaluation -- SURVEY 2.2 K2)
// one warp per output c, lanes over k (row c of Pz is contiguous)
__global__ void __launch_bounds__(256)
k_zbias(int h1, int d_z, const double* __restrict__ Pz, const double* __restrict__ z,
        const float* __restrict__ b1, float* __restrict__ zb, double* __restrict__ zb64 = nullptr) {
  // programmatic dependent launch on both sides (no-ops in a plain launch): the forward chain behind this kernel
  // may set itself up now, and -- launched behind the z fetch kernel -- this row's Pz entries (the cold HBM
  // reads) are in registers before z is waited for
  asm volatile("griddepcontrol.launch_dependents;");
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  double pz[4] = {0.0, 0.0, 0.0, 0.0};
  if (c < h1) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (lane + 32 * u < d_z) pz[u] = Pz[(int64_t)c * d_z + lane + 32 * u];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (c >= h1) return;
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (lane + 32 * u < d_z) s += pz[u] * z[lane + 32 * u];
  for (int k = lane + 128; k < d_z; k += 32) s += Pz[(int64_t)c * d_z + k] * z[k];
  s = warp_sum(s);
  if (lane == 0) {
    zb[c] = (float)(s + (double)b1[c]);
    if (zb64) zb64[c] = s + (double)b1[c];
  }
}

// unit-seed coefficients of the fused output-layer epilogue (reduced frame):
// seed = 2 sigma (phi + c) = a2 phi + b2
__global__ void k_seedcoef(int r_u, const float* __restrict__ ostd, const float* __restrict__ c,
                           float* __restrict__ a2, float* __restrict__ b2) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < r_u; j += gridDim.x * blockDim.x) {
    a2[j] = (float)(2.0 * (double)ostd[j]);
    b2[j] = (float)(2.0 * (double)ostd[j] * (double)c[j]);
  }
}

// X = [m_r, z_row, 0-pad]  (forward_batch / jacobian rows with per-row z)
__global__ void k_build_x(int64_t n, int r_m, int d_z, int ldx, const float* __restrict__ mr,
                          const float* __restrict__ z, float* __restrict__ X) {
  int64_t i = blockIdx.x;
  for (int c = threadIdx.x; c < ldx; c += blockDim.x) {
    float v = 0.0f;
    if (c < r_m) v = mr[i * r_m + c];
    else if (c < r_m + d_z) v = z[i * d_z + (c - r_m)];
    X[i * ldx + c] = v;
  }
}

// Per-sample QoI (reference riskopt.py:187-189 / pod.py:56-58):
//   reduced: Q = phi.phi + 2 phi.c + q0
//   gram   : Q = phi.(K phi) + 2 phi.c + q0  (decoded frame, K = U^T M U)
// accumulated in fp64; plus per-block fp64 partial moments.
// the warp's moments: lanes 0..3 each accumulated every fourth row of the
// warp; added in lane order (k_qoi and k_moments share this order)
SDN_DEV void qoi_lane_combine(const double (&acc)[6], double* dst, int lane) {
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const double a1 = __shfl_sync(0xffffffffu, acc[f], 1), a2 = __shfl_sync(0xffffffffu, acc[f], 2),
                 a3 = __shfl_sync(0xffffffffu, acc[f], 3);
    if (lane == 0) dst[f] = ((acc[f] + a1) + a2) + a3;
  }
}
// One warp per row, grid-stride, four rows in flight per warp (their 16-byte
// loads are issued before the first fp64 reduction); block partials in fixed
// order (rows of a warp are accumulated in ascending order).
__global__ void __launch_bounds__(256)
k_qoi(int64_t n, int r_u, const float* __restrict__ phi, const float* __restrict__ kphi,
      const float* __restrict__ c, double q0, double shift, double t, double eps,
      double* __restrict__ Q, double* __restrict__ part, const double* __restrict__ tp = nullptr,
      int* __restrict__ counter = nullptr, double* __restrict__ out = nullptr, double* __restrict__ Q2 = nullptr) {
  if (tp) t = *tp;                     // device-side t (graph replay)
  __shared__ double sp[8][6];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * 8;
  const bool vec = (r_u & 3) == 0;     // rows start 16-byte aligned (cudaMalloc base, r_u % 4 == 0)
  for (int64_t i0 = (int64_t)blockIdx.x * 8 + warp; i0 < n; i0 += 4 * stride) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (vec) {
      for (int j = 4 * lane; j < r_u; j += 128) {
        const float4 c4 = __ldg(reinterpret_cast<const float4*>(c + j));
        float4 p4[4], k4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + u * stride;
          p4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (i < n) p4[u] = __ldg(reinterpret_cast<const float4*>(phi + i * r_u + j));
          k4[u] = p4[u];
          if (kphi && i < n) k4[u] = __ldg(reinterpret_cast<const float4*>(kphi + i * r_u + j));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s[u] += (double)p4[u].x * ((double)k4[u].x + 2.0 * (double)c4.x);
          s[u] += (double)p4[u].y * ((double)k4[u].y + 2.0 * (double)c4.y);
          s[u] += (double)p4[u].z * ((double)k4[u].z + 2.0 * (double)c4.z);
          s[u] += (double)p4[u].w * ((double)k4[u].w + 2.0 * (double)c4.w);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= n) break;
        const float* p = phi + i * r_u;
        const float* kp = kphi ? kphi + i * r_u : p;
        for (int j = lane; j < r_u; j += 32) {
          double pj = p[j];
          s[u] += pj * ((double)kp[j] + 2.0 * (double)c[j]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = warp_sum(s[u]);
    if (lane < 4) {                      // lane u finishes row u (the smoothed-plus terms are fp64 exp/log work)
      const int64_t i = i0 + lane * stride;
      if (i < n) {
        const double q = (lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3]) + q0;
        Q[i] = q;
        if (Q2) Q2[i] = q;             // the exact-CVaR selection's own copy (sel_q)
        double qs = q - shift, x = q - t;
        double d1 = splus_d1_d(x, eps);
        acc[0] += 1.0; acc[1] += qs; acc[2] += qs * qs;
        acc[3] += splus_d(x, eps); acc[4] += d1; acc[5] += (d1 > 0.0) ? 1.0 : 0.0;
      }
    }
  }
  qoi_lane_combine(acc, sp[warp], lane);
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sp[w][threadIdx.x];
    part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = s;
  }
  if (threadIdx.x == 6 || threadIdx.x == 7) part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = 0.0;
  if (counter) last_block_sum(counter, gridDim.x, STATS_LEN, part, out);
}

// QoI from the output layer's fused chunk partials (EpiAffineSeed::qp,
// gemm_tc.cuh): Q_i = q0 + sum over the row's 16-column chunks in order, then
// the moments exactly as k_qoi takes them.  One thread per row (coalesced
// chunk planes), fixed butterfly per warp, warps in order, last block sums.
__global__ void __launch_bounds__(128)
k_qoi_part(int64_t n, int nch, const double* __restrict__ P, int64_t ld, double q0, double shift, double t,
           double eps, double* __restrict__ Q, double* __restrict__ part, const double* __restrict__ tp = nullptr,
           int* __restrict__ counter = nullptr, double* __restrict__ out = nullptr, double* __restrict__ Q2 = nullptr) {
  if (tp) t = *tp;                     // device-side t (graph replay)
  __shared__ double sp[4][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 128) {
    double s = 0.0;
#pragma unroll 8
    for (int ch = 0; ch < nch; ++ch) s += P[(int64_t)ch * ld + i];
    const double q = s + q0;
    Q[i] = q;
    if (Q2) Q2[i] = q;                 // the exact-CVaR selection's own copy (sel_q)
    const double qs = q - shift, x = q - t;
    const double d1 = splus_d1_d(x, eps);
    acc[0] += 1.0; acc[1] += qs; acc[2] += qs * qs;
    acc[3] += splus_d(x, eps); acc[4] += d1; acc[5] += (d1 > 0.0) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const double v = warp_sum(acc[f]);
    if (lane == 0) sp[warp][f] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int w = 0; w < 4; ++w) s += sp[w][threadIdx.x];
    part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = s;
  }
  if (threadIdx.x == 6 || threadIdx.x == 7) part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = 0.0;
  if (counter) last_block_sum(counter, gridDim.x, STATS_LEN, part, out);
}

// fixed-order sum of nb rows of width w (fp64) -> out (w): one warp per
// column, lanes stride the rows, then a fixed butterfly (deterministic)
__global__ void __launch_bounds__(256)
k_sum_rows(int nb, int w, const double* __restrict__ part, double* __restrict__ out) {
  const int f = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (f >= w) return;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)b * w + f];
  s = warp_sum(s);
  if (lane == 0) out[f] = s;
}

// ---- Q refinement band (the fp64 re-evaluation is refine.cuh).
// REFINE_REL bounds the chain's Q error with ~6x margin over the largest
// measured (1.7e-5 relative at c3).
constexpr double REFINE_REL = 1e-4;
constexpr int REFINE_ROWS = 4096;     // band rows per k_refine row chunk (larger bands run in several chunks)
SDN_DEV bool in_band(double q, double t, double eps) {       // smoothed CVaR window
  double d = REFINE_REL * fabs(q) + 1e-300;
  double x = q - t;
  return x >= -d && x <= eps + d;
}
SDN_DEV bool in_band_exact(double q, double thr) {            // exact-CVaR threshold
  return fabs(q - thr) <= 2.0 * REFINE_REL * fabs(q) + 1e-300 || q != q || thr != thr;
}

// block moments of k_qoi recomputed from Q (after refinement)
__global__ void __launch_bounds__(256)
k_moments(int64_t n, const double* __restrict__ Q, double shift, double t, double eps,
          double* __restrict__ part, const double* __restrict__ tp = nullptr) {
  if (tp) t = *tp;
  __shared__ double sp[8][6];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  // same row -> (block, warp, lane) assignment and order as k_qoi
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t i0 = (int64_t)blockIdx.x * 8 + warp; i0 < n; i0 += 4 * stride) {
    const int64_t i = i0 + lane * stride;
    if (lane < 4 && i < n) {
      double q = Q[i], qs = q - shift, x = q - t;
      double d1 = splus_d1_d(x, eps);
      acc[0] += 1.0; acc[1] += qs; acc[2] += qs * qs;
      acc[3] += splus_d(x, eps); acc[4] += d1; acc[5] += (d1 > 0.0) ? 1.0 : 0.0;
    }
  }
  qoi_lane_combine(acc, sp[warp], lane);
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sp[w][threadIdx.x];
    part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = s;
  }
  if (threadIdx.x == 6 || threadIdx.x == 7) part[(int64_t)blockIdx.x * STATS_LEN + threadIdx.x] = 0.0;
}

// results of an evaluation straight into host-mapped pinned memory (zero
// copy): one small kernel instead of three device-to-host copy nodes
__global__ void __launch_bounds__(256)
k_export(const double* __restrict__ stats, double* __restrict__ hstats, int nstats, const double* __restrict__ part,
         double* __restrict__ hpart, int npart, const int* __restrict__ band, int* __restrict__ hband, int nband) {
  for (int i = threadIdx.x; i < nstats; i += blockDim.x) hstats[i] = stats[i];
  for (int i = threadIdx.x; i < npart; i += blockDim.x) hpart[i] = part[i];
  for (int i = threadIdx.x; i < nband; i += blockDim.x) hband[i] = band[i];
}

// sample weight w_i of the risk functional:
//   mean: 1/n; meanvar: (1 + 2 beta (Q_i - Qbar))/n; smoothed CVaR (riskopt.py:238-241):
//   splus'(Q_i - t)/(n (1-beta)); exact CVaR: 1/k on the selection; unit: 1.
SDN_DEV double sample_weight(int kind, double q, const double* st, double shift, double beta,
                             double eps, double t, double kinv) {
  double n = st[0];
  switch (kind) {
    case RISK_MEAN: return 1.0 / n;
    case RISK_MEANVAR: {
      double qbar = shift + st[1] / n;
      return (1.0 + 2.0 * beta * (q - qbar)) / n;
    }
    case RISK_CVAR_SMOOTH: return splus_d1_d(q - t, eps) / (n * (1.0 - beta));
    case RISK_CVAR_EXACT: return kinv;
    default: return 1.0;
  }
}

// active-row flags for compaction: smoothed CVaR -> splus'(Q - t) > 0;
// exact CVaR -> selection mask; RISK_BAND -> Q within the refinement band.
SDN_DEV bool row_flag(int kind, const double* Q, const uint8_t* sel, int64_t i, double t, double eps,
                      const double* tdev) {
  if (kind == RISK_CVAR_EXACT) return sel[i] != 0;
  if (kind == RISK_BAND) return in_band(Q[i], t, eps);
  if (kind == RISK_BAND_EXACT) return in_band_exact(Q[i], *tdev);
  return splus_d1_d(Q[i] - t, eps) > 0.0;
}
// Per 1024-row block: count.
__global__ void __launch_bounds__(1024)
k_flag_count(int64_t n, int kind, const double* __restrict__ Q, const uint8_t* __restrict__ sel,
             double t, double eps, const double* __restrict__ tdev, int* __restrict__ counts) {
  __shared__ int wc[32];
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  bool f = false;
  if (i < n) f = row_flag(kind, Q, sel, i, t, eps, tdev);
  unsigned b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 32; ++w) s += wc[w];
    counts[blockIdx.x] = s;
  }
}

// ordered compaction of a selection mask in ONE block (n up to 64 K rows):
// thread t owns the rows [t per, (t + 1) per), counts, a block-wide exclusive
// scan, then writes its rows' indices in order; total -> *n_act.  Replaces the
// count / scan / compact chain (three dependent launches) behind the exact-CVaR
// selection, which sits on the evaluation's critical path at c2.
constexpr int64_t COMPACT1_MAX = 65536;
__global__ void __launch_bounds__(1024)
k_compact_mask1(int64_t n, const uint8_t* __restrict__ sel, int* __restrict__ rowidx, int* __restrict__ n_act) {
  __shared__ int wsum[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (int)((n + 1023) / 1024);
  const int64_t lo = min((int64_t)t * per, n), hi = min(lo + per, n);
  int c = 0;
  for (int64_t i = lo; i < hi; ++i) c += sel[i] != 0;
  int inc = c;                                     // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    wsum[lane] = wi - w;                           // exclusive warp offsets
    if (lane == 31) *n_act = wi;
  }
  __syncthreads();
  int off = wsum[warp] + inc - c;
  for (int64_t i = lo; i < hi; ++i)
    if (sel[i] != 0) rowidx[off++] = (int)i;
}

// exclusive scan of nb block counts (single block); total -> *n_act
__global__ void k_scan_counts(int nb, const int* __restrict__ counts, int* __restrict__ offs,
                              int* __restrict__ n_act) {
  if (threadIdx.x != 0) return;
  int s = 0;
  for (int b = 0; b < nb; ++b) { offs[b] = s; s += counts[b]; }
  *n_act = s;
}

// ordered compaction: rowidx[offs[b] + rank-in-block] = i for flagged rows
__global__ void __launch_bounds__(1024)
k_compact(int64_t n, int kind, const double* __restrict__ Q, const uint8_t* __restrict__ sel,
          double t, double eps, const double* __restrict__ tdev, const int* __restrict__ offs,
          int* __restrict__ rowidx) {
  __shared__ int wbase[32];
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  bool f = false;
  if (i < n) f = row_flag(kind, Q, sel, i, t, eps, tdev);
  unsigned b = __ballot_sync(0xffffffffu, f);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wbase[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 32; ++w) { int c = wbase[w]; wbase[w] = s; s += c; }
  }
  __syncthreads();
  if (f) rowidx[offs[blockIdx.x] + wbase[warp] + __popc(b & ((1u << lane) - 1u))] = (int)i;
}

// seed of the reverse sweep on y (pre-output-scaling), compacted rows:
//   E[r] = w_i * out_std * dQ/dphi,  dQ/dphi = 2 (phi + c)  (reduced, pod.py:60-62)
//                                     or 2 (K phi + c)       (decoded frame)
// rowidx null = identity; n_act_dev null = all n rows.
__global__ void __launch_bounds__(256)
k_seed(int64_t n, const int* __restrict__ n_act_dev, const int* __restrict__ rowidx, int r_u,
       const float* __restrict__ phi, const float* __restrict__ kphi, const float* __restrict__ c,
       const float* __restrict__ ostd, const double* __restrict__ Q, const double* __restrict__ st,
       int kind, double shift, double beta, double eps, double t, double kinv,
       float* __restrict__ E, __nv_bfloat16* __restrict__ Ehi = nullptr, __nv_bfloat16* __restrict__ Elo = nullptr) {
  int64_t nr = n_act_dev ? (int64_t)*n_act_dev : n;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < nr; r += (int64_t)gridDim.x * 8) {
    int64_t i = rowidx ? (int64_t)rowidx[r] : r;
    const double w = (kind == RISK_UNIT) ? 1.0 : sample_weight(kind, Q[i], st, shift, beta, eps, t, kinv);
    const float* p = (kphi ? kphi : phi) + i * r_u;
    for (int j = lane; j < r_u; j += 32)
    {
      const float e = (float)(w * 2.0 * ((double)p[j] + (double)c[j]) * (double)ostd[j]);
      E[r * r_u + j] = e;
      if (Ehi) {   // bf16x3 split for the tensor-core sweep (its first A operand)
        const __nv_bfloat16 hi = __float2bfloat16_rn(e);
        Ehi[r * r_u + j] = hi;
        Elo[r * r_u + j] = __float2bfloat16_rn(e - __bfloat162float(hi));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Unified reverse sweep: one sweep with unit seeds gives the
// per-sample VJPs u0_i = dQ_i/dS1; every risk's gradient is the weighted
// column sum sum_i w_i^(r) u0_i (fp64), so all risks of an evaluation share
// one sweep and the weights are only needed at the last reduction.
constexpr int SDN_RMAX = 8;

struct RiskSet {
  int R;
  int kind[SDN_RMAX];
  double beta[SDN_RMAX], eps[SDN_RMAX], t[SDN_RMAX], kinv[SDN_RMAX];
  const uint8_t* mask[SDN_RMAX];     // exact CVaR selection masks (sample rows)
  const double* tdev;                // per-risk t on the device (graph replay), else t[] by value
};
SDN_DEV double risk_t(const RiskSet& rs, int r) { return rs.tdev ? rs.tdev[r] : rs.t[r]; }

SDN_DEV double risk_weight(const RiskSet& rs, int r, int64_t i, double q, const double* st, double shift) {
  // (an exact-CVaR risk without a mask is deferred: its sums are taken later
  // over the selected rows' stored u, k_sel_colsum)
  if (rs.kind[r] == RISK_CVAR_EXACT) return (rs.mask[r] && rs.mask[r][i]) ? rs.kinv[r] : 0.0;
  return sample_weight(rs.kind[r], q, st, shift, rs.beta[r], rs.eps[r], risk_t(rs, r), 0.0);
}

SDN_DEV bool risk_active(const RiskSet& rs, int64_t i, double q) {
  bool a = false;
  for (int r = 0; r < rs.R; ++r) {
    if (rs.kind[r] == RISK_CVAR_EXACT) a |= rs.mask[r][i] != 0;
    else if (rs.kind[r] == RISK_CVAR_SMOOTH) a |= splus_d1_d(q - risk_t(rs, r), rs.eps[r]) > 0.0;
    else a = true;
  }
  return a;
}

// ordered compaction of the union of the risks' active rows (same scheme as
// k_flag_count / k_compact)
__global__ void __launch_bounds__(1024)
k_union_count(int64_t n, RiskSet rs, const double* __restrict__ Q, int* __restrict__ counts) {
  __shared__ int wc[32];
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const bool f = i < n && risk_active(rs, i, Q[i]);
  unsigned b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 32; ++w) s += wc[w];
    counts[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(1024)
k_union_compact(int64_t n, RiskSet rs, const double* __restrict__ Q, const int* __restrict__ offs,
                int* __restrict__ rowidx) {
  __shared__ int wbase[32];
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const bool f = i < n && risk_active(rs, i, Q[i]);
  unsigned b = __ballot_sync(0xffffffffu, f);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wbase[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 32; ++w) { int c = wbase[w]; wbase[w] = s; s += c; }
  }
  __syncthreads();
  if (f) rowidx[offs[blockIdx.x] + wbase[warp] + __popc(b & ((1u << lane) - 1u))] = (int)i;
}

// per-row risk weights of the sweep rows, W[j * R + r] (j = sweep row, i =
// rowidx ? rowidx[j] : j), and per-block fixed-order partials of
// sum_{w != 0} Q_i and #{w != 0} per risk (exact CVaR: the selection sum)
__global__ void __launch_bounds__(256)
k_weights(int64_t nsw, const int* __restrict__ n_act_dev, const int* __restrict__ rowidx, RiskSet rs,
          const double* __restrict__ Q, const double* __restrict__ st, double shift, double* __restrict__ W,
          double* __restrict__ part, int* __restrict__ counter = nullptr, double* __restrict__ out = nullptr) {
  __shared__ double sp[8][2 * SDN_RMAX];
  const int64_t nr = n_act_dev ? (int64_t)*n_act_dev : nsw;
  double acc[2 * SDN_RMAX];
#pragma unroll
  for (int f = 0; f < 2 * SDN_RMAX; ++f) acc[f] = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x; j < nr; j += (int64_t)gridDim.x * 256) {
    const int64_t i = rowidx ? (int64_t)rowidx[j] : j;
    const double q = Q[i];
#pragma unroll
    for (int r = 0; r < SDN_RMAX; ++r) {
      if (r < rs.R) {
        const double w = risk_weight(rs, r, i, q, st, shift);
        W[j * rs.R + r] = w;
        if (w != 0.0) { acc[2 * r] += q; acc[2 * r + 1] += 1.0; }
      }
    }
  }
  // fixed-order block reduction: lanes (butterfly), then warps in order
#pragma unroll
  for (int f = 0; f < 2 * SDN_RMAX; ++f) acc[f] = warp_sum(acc[f]);
  if (lane == 0)
    for (int f = 0; f < 2 * SDN_RMAX; ++f) sp[warp][f] = acc[f];
  __syncthreads();
  if (threadIdx.x < 2 * SDN_RMAX) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sp[w][threadIdx.x];
    part[(int64_t)blockIdx.x * 2 * SDN_RMAX + threadIdx.x] = s;
  }
  if (counter) last_block_sum(counter, gridDim.x, 2 * SDN_RMAX, part, out);
}

// weighted column sums of U (n_act x w): part[r][by][c] = sum_rows W[row][r] U[row][c]
__global__ void __launch_bounds__(256)
k_colsum_w(int64_t n, const int* __restrict__ n_act_dev, int w, const float* __restrict__ U,
           const double* __restrict__ Wt, int R, double* __restrict__ part) {
  __shared__ double s[8][33];
  const int64_t nr = n_act_dev ? (int64_t)*n_act_dev : n;
  const int c = blockIdx.x * 32 + threadIdx.x;
  for (int r = 0; r < R; ++r) {
    double acc = 0.0;
    if (c < w)
      for (int64_t j = (int64_t)blockIdx.y * 8 + threadIdx.y; j < nr; j += (int64_t)gridDim.y * 8)
        acc += Wt[j * R + r] * (double)U[j * w + c];
    s[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && c < w) {
      double t = 0.0;
      for (int y = 0; y < 8; ++y) t += s[y][threadIdx.x];
      part[((int64_t)r * gridDim.y + blockIdx.y) * w + c] = t;
    }
    __syncthreads();
  }
}

// per-risk finalisation (blockIdx.y = risk): A = sum_rb part_r[rb][:];
// out_r[k] = sum_c PzT[k][c] A[c]; out_r[d_z], out_r[d_z+1] = vsum[2r], vsum[2r+1]
__global__ void __launch_bounds__(256)
k_finalize_multi(int nrb, int64_t plane, int h1, int d_z, const double* __restrict__ part,
                 const double* __restrict__ PzT, const double* __restrict__ vsum, int plen,
                 double* __restrict__ out) {
  extern __shared__ double A[];
  const int r = blockIdx.y;
  const double* pr = part ? part + (int64_t)r * plane : nullptr;
  for (int c = threadIdx.x; c < h1; c += blockDim.x) {
    double s = 0.0;
    if (pr)
      for (int b = 0; b < nrb; ++b) s += pr[(int64_t)b * h1 + c];
    A[c] = s;
  }
  __syncthreads();
  double* o = out + (int64_t)r * plen;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = blockIdx.x * nw + warp; k < d_z; k += gridDim.x * nw) {
    double s = 0.0;
#pragma unroll 8
    for (int c = lane; c < h1; c += 32) s += __ldg(PzT + (int64_t)k * h1 + c) * A[c];
    s = warp_sum(s);
    if (lane == 0) o[k] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    o[d_z] = vsum[2 * r];
    o[d_z + 1] = vsum[2 * r + 1];
  }
}

// deferred exact-CVaR sums: out[c] = kinv * sum_{j < k} u[rows[j], c] (fp64,
// fixed order: thread rows j = y, y + 32, ..., then the 32 row groups in
// order) and the value partials vs = (sum_j Q[rows[j]], k)
__global__ void __launch_bounds__(1024)
k_sel_colsum(int64_t k, const int* __restrict__ rows, int w, const float* __restrict__ u, int64_t ld, double kinv,
             const double* __restrict__ Q, double* __restrict__ out, double* __restrict__ vs) {
  __shared__ double s[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  double acc = 0.0;
  if (c < w) {
#pragma unroll 4
    for (int64_t j = threadIdx.y; j < k; j += 32) acc += (double)u[(int64_t)__ldg(rows + j) * ld + c];
  }
  s[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < w) {
    double t = 0.0;
    for (int y = 0; y < 32; ++y) t += s[y][threadIdx.x];
    out[c] = kinv * t;
  }
  if (blockIdx.x == 0 && threadIdx.y == 1) {       // one warp: lane-strided, fixed butterfly
    double qs = 0.0;
    for (int64_t j = threadIdx.x; j < k; j += 32) qs += Q[rows[j]];
    qs = warp_sum(qs);
    if (threadIdx.x == 0) {
      vs[0] = qs;
      vs[1] = (double)k;
    }
  }
}

// column sums of fp64 partial rows (nrb rows, bounded by the device row count
// for compacted sweeps: 4 partial rows per 128-row tile), fixed order
__global__ void __launch_bounds__(1024)
k_colsum64(int nrb, const int* __restrict__ n_act_dev, int w, const double* __restrict__ part,
           double* __restrict__ out, int64_t plane = 0) {
  __shared__ double s[32][33];
  part += blockIdx.y * plane;          // gridDim.y = risks (one partial plane each)
  out += (int64_t)blockIdx.y * w;
  if (n_act_dev) nrb = min(nrb, ((*n_act_dev + 127) / 128) * 4);
  const int c = blockIdx.x * 32 + threadIdx.x;
  double acc = 0.0;
  if (c < w) {
#pragma unroll 8
    for (int r = threadIdx.y; r < nrb; r += 32) acc += part[(int64_t)r * w + c];
  }
  s[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < w) {
    double t = 0.0;
    for (int y = 0; y < 32; ++y) t += s[y][threadIdx.x];
    out[c] = t;
  }
}

// ---- short tail of an evaluation (graph path).  The deferred exact-CVaR
// sums over the k selected rows of the stored u are taken by row slices
// (k_sel_colsum_sl: S x w/32 blocks instead of w/32; 13.7 -> ~4 us at c2), and
// one kernel finalises every risk from its own list of partial rows and --
// every block writing its own outputs -- puts the results in host-mapped memory
// (k_finalize_export: what k_finalize_multi + k_export did in two dependent
// launches).  Variants that finished in ONE block (all projections, or only
// the export behind an atomic ticket) were slower, profiles/README.md.
// out[s][c] = sum over slice s of the selected rows of u[rows[j], c] (fp64,
// fixed order: thread rows j = lo + y, lo + y + 32, ..., then the 32 row groups
// in order); the value partials vs = (sum_j Q[rows[j]], k) by block (0, 0)
__global__ void __launch_bounds__(1024)
k_sel_colsum_sl(int64_t k, const int* __restrict__ rows, int w, const float* __restrict__ u, int64_t ld,
                const double* __restrict__ Q, double* __restrict__ out, double* __restrict__ vs) {
  asm volatile("griddepcontrol.launch_dependents;");       // k_finalize_export prefetches its PzT rows meanwhile
  __shared__ double s[32][33];
  const int c = blockIdx.x * 32 + threadIdx.x, S = gridDim.y, sl = blockIdx.y;
  const int64_t per = (k + S - 1) / S, lo = sl * per, hi = min(k, lo + per);
  double acc = 0.0;
  if (c < w) {
#pragma unroll 4
    for (int64_t j = lo + threadIdx.y; j < hi; j += 32) acc += (double)u[(int64_t)__ldg(rows + j) * ld + c];
  }
  s[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < w) {
    double t = 0.0;
    for (int y = 0; y < 32; ++y) t += s[y][threadIdx.x];
    out[(int64_t)sl * w + c] = t;
  }
  if (blockIdx.x == 0 && sl == 0 && threadIdx.y == 1) {       // one warp: lane-strided, fixed butterfly
    double qs = 0.0;
    for (int64_t j = threadIdx.x; j < k; j += 32) qs += Q[rows[j]];
    qs = warp_sum(qs);
    if (threadIdx.x == 0) {
      vs[0] = qs;
      vs[1] = (double)k;
    }
  }
}
struct FinRisk {
  const double* part;    // nrb partial rows of h1 (null: zero gradient)
  int nrb;
  double scale;          // applied to the summed rows (1/k for the deferred exact-CVaR sums)
};
struct FinArgs {
  int h1, d_z, plen;
  FinRisk risk[SDN_RMAX];
  const double* PzT;
  const double* vsum;
  double* out;           // [R][plen]
  const double* stats; double* hstats; int nstats;      // export to host-mapped memory (hstats null: none)
  double* hpart; int npart;
  const int* band; int* hband; int nband;
};
// per-risk finalisation (blockIdx.y = risk): A = scale * sum_b part[b][:];
// out_r[k] = sum_c PzT[k][c] A[c]; out_r[d_z], out_r[d_z+1] = vsum[2r], vsum[2r+1].
// With hstats set every block also writes its outputs straight to the
// host-mapped result buffers (block (0, 0): the moments and the band log too),
// so no export kernel follows and no block waits for another.
__global__ void __launch_bounds__(256)
k_finalize_export(const FinArgs a) {
  extern __shared__ double A[];
  const int r = blockIdx.y, h1 = a.h1, d_z = a.d_z;
  const FinRisk& fr = a.risk[r];
  // launched programmatically behind the last sum kernel (a no-op in a plain launch): this block's PzT rows
  // (static, cold in L2 after the evaluation's traffic) are on their way before the sums are waited for
  for (int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < d_z; k += gridDim.x * (blockDim.x >> 5))
    for (int o = (threadIdx.x & 31) * 128; o < h1 * 8; o += 32 * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.PzT + (int64_t)k * h1) + o));
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int c = threadIdx.x; c < h1; c += blockDim.x) {
    double s = 0.0;
    if (fr.part)
      for (int b = 0; b < fr.nrb; ++b) s += fr.part[(int64_t)b * h1 + c];
    A[c] = fr.scale * s;
  }
  __syncthreads();
  double* o = a.out + (int64_t)r * a.plen;
  double* ho = a.hstats ? a.hpart + (int64_t)r * a.plen : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = blockIdx.x * nw + warp; k < d_z; k += gridDim.x * nw) {
    double s = 0.0;
#pragma unroll 8
    for (int c = lane; c < h1; c += 32) s += __ldg(a.PzT + (int64_t)k * h1 + c) * A[c];
    s = warp_sum(s);
    if (lane == 0) {
      o[k] = s;
      if (ho) ho[k] = s;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double v0 = a.vsum[2 * r], v1 = a.vsum[2 * r + 1];
    o[d_z] = v0;
    o[d_z + 1] = v1;
    if (ho) { ho[d_z] = v0; ho[d_z + 1] = v1; }
  }
  if (a.hstats && blockIdx.x == 0 && blockIdx.y == 0) {
    for (int i = threadIdx.x; i < a.nstats; i += blockDim.x) a.hstats[i] = a.stats[i];
    for (int i = threadIdx.x; i < a.nband; i += blockDim.x) a.hband[i] = a.band[i];
  }
}

// histogram increment (plain shared atomics measured faster than warp
// aggregation with __match_any_sync on B200 for these key distributions)
SDN_DEV void hist_add(unsigned* hist, bool m, unsigned d) {
  if (m) atomicAdd(&hist[d], 1u);
}

// ---------------------------------------------------------------------------
// Exact top-k selection (value desc, then global index asc).
// Single-CTA 8-pass MSD radix select over order-preserving 64-bit keys,
// then an index-ordered tie resolution at the threshold key.  `gidx` (double,
// may be null = position) supplies the global index used for ordering and
// marks padding (gidx < 0 -> never selected).  Output: mask (n).
__global__ void __launch_bounds__(1024)
k_topk_select(int64_t n, int64_t k, const double* __restrict__ vals, const double* __restrict__ gidx,
              uint8_t* __restrict__ mask, double* __restrict__ thr) {
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ long long s_krem;
  __shared__ int wsum[32];
  __shared__ long long s_run;
  const int tid = threadIdx.x;
  if (tid == 0) { s_prefix = 0; s_krem = k; }
  uint64_t himask = 0;
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int d = tid; d < 256; d += blockDim.x) hist[d] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int64_t base = 0; base < n; base += blockDim.x) {
      const int64_t i = base + tid;
      bool m = false;
      unsigned d = 0;
      if (i < n && !(gidx && gidx[i] < 0.0)) {
        const uint64_t key = dkey(vals[i]);
        m = (key & himask) == prefix;
        d = (unsigned)(key >> shift) & 255u;
      }
      hist_add(hist, m, d);
    }
    __syncthreads();
    if (tid == 0) {
      long long krem = s_krem, cum = 0;
      int d = 255;
      for (; d > 0; --d) {
        if (cum + (long long)hist[d] >= krem) break;
        cum += hist[d];
      }
      s_krem = krem - cum;
      s_prefix = prefix | ((uint64_t)d << shift);
    }
    himask |= (0xFFull << shift);
    __syncthreads();
  }
  const uint64_t T = s_prefix;
  const long long need = s_krem;       // how many threshold-equal keys to take
  if (thr && tid == 0) *thr = dkey_inv(T);
  if (tid == 0) s_run = 0;
  __syncthreads();
  // rows in ascending global index order: positions are index-ordered for
  // the local case; candidate arrays are concatenated in rank order, and each
  // rank's candidates are index-ordered, so position order == global order.
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t i = base + tid;
    bool valid = i < n && !(gidx && gidx[i] < 0.0);
    uint64_t key = valid ? dkey(vals[i]) : 0;
    bool eq = valid && key == T;
    unsigned b = __ballot_sync(0xffffffffu, eq);
    int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) wsum[warp] = __popc(b);
    __syncthreads();
    if (tid == 0) {
      int s = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { int c = wsum[w]; wsum[w] = s; s += c; }
    }
    __syncthreads();
    long long rank = s_run + wsum[warp] + __popc(b & ((1u << lane) - 1u));
    if (i < n) mask[i] = (valid && (key > T || (eq && rank < need))) ? 1 : 0;
    __syncthreads();
    if (tid == blockDim.x - 1) s_run += wsum[warp] + __popc(b);
    __syncthreads();
  }
}

// Same selection with the keys resident in shared memory (n <= TOPK_SMEM_MAX):
// one global read, then radix passes over SMEM only from the first byte in
// which the keys differ (min/max common prefix skipped: Q values share sign,
// exponent and leading mantissa bits), per-warp histograms (no cross-warp
// atomic contention on the hot bins), a warp-parallel digit search.
constexpr int TOPK_SMEM_MAX = 24576;   // 192 KB of uint64 keys (+ 32 KB warp histograms)
constexpr size_t TOPK_SMEM_BYTES = (size_t)TOPK_SMEM_MAX * 8 + 32 * 256 * 4;

__global__ void __launch_bounds__(1024)
k_topk_select_smem(int n, int64_t k, const double* __restrict__ vals, const double* __restrict__ gidx,
                   uint8_t* __restrict__ mask, double* __restrict__ thr) {
  extern __shared__ uint64_t keys[];
  unsigned* whist = reinterpret_cast<unsigned*>(keys + TOPK_SMEM_MAX);   // [32][256]
  __shared__ unsigned hist[256];
  __shared__ uint64_t s_prefix, s_min[32], s_max[32];
  __shared__ long long s_krem;
  __shared__ int wsum[32];
  __shared__ int s_first;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t kmin = ~0ull, kmax = 0ull;
#pragma unroll 4
  for (int i = tid; i < n; i += blockDim.x) {
    const uint64_t key = (gidx && gidx[i] < 0.0) ? 0ull : dkey(vals[i]);   // padding: key 0, below every value
    keys[i] = key;
    kmin = min(kmin, key);
    kmax = max(kmax, key);
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) { s_min[warp] = kmin; s_max[warp] = kmax; }
  __syncthreads();
  if (tid == 0) {
    uint64_t a = ~0ull, b = 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = min(a, s_min[w]); b = max(b, s_max[w]); }
    const int cp = (a == b) ? 8 : __clzll((long long)(a ^ b)) / 8;      // common leading bytes
    s_first = cp;
    s_prefix = (cp == 0) ? 0ull : (cp >= 8 ? a : (a & (~0ull << (64 - 8 * cp))));
    s_krem = k;
  }
  __syncthreads();
  const int first = s_first;
  uint64_t himask = (first == 0) ? 0ull : (first >= 8 ? ~0ull : (~0ull << (64 - 8 * first)));
  for (int pass = first; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int d = tid; d < 32 * 256; d += blockDim.x) whist[d] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    unsigned* wh = whist + warp * 256;
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + tid;
      const uint64_t key = i < n ? keys[i] : 0ull;
      if (i < n && (key & himask) == prefix) atomicAdd(&wh[(unsigned)(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int d = tid; d < 256; d += blockDim.x) {
      unsigned c = 0;
#pragma unroll 8
      for (int w = 0; w < 32; ++w) c += whist[w * 256 + d];
      hist[d] = c;
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns digits 255-8l .. 248-8l (descending)
      unsigned c[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { c[i] = hist[255 - 8 * lane - i]; tot += c[i]; }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const long long krem = s_krem;
      const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl >= krem);
      const int L = hit ? __ffs(hit) - 1 : 31;
      if (lane == L) {
        long long cum = (long long)(incl - tot);
        int d = 255 - 8 * lane;
        for (int i = 0; i < 8; ++i) {
          d = 255 - 8 * lane - i;
          if (cum + (long long)c[i] >= krem || i == 7) break;
          cum += c[i];
        }
        s_krem = krem - cum;
        s_prefix = prefix | ((uint64_t)d << shift);
      }
    }
    himask |= (0xFFull << shift);
    __syncthreads();
  }
  const uint64_t T = s_prefix;
  const long long need = s_krem;       // how many threshold-equal keys to take
  if (thr && tid == 0) *thr = dkey_inv(T);
  // tie resolution in index order: each thread owns a contiguous run of
  // keys; one block-wide exclusive scan of the threshold-equal counts
  const int per = (n + (int)blockDim.x - 1) / (int)blockDim.x;
  const int i0 = tid * per, i1 = min(i0 + per, n);
  int cnt = 0;
  for (int i = i0; i < i1; ++i) cnt += (keys[i] != 0ull && keys[i] == T) ? 1 : 0;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0, x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    wsum[lane] = x - v;               // exclusive warp offsets
  }
  __syncthreads();
  long long rank = wsum[warp] + (incl - cnt);
  for (int i = i0; i < i1; ++i) {
    const uint64_t key = keys[i];
    const bool valid = key != 0ull;
    const bool eq = valid && key == T;
    mask[i] = (valid && (key > T || (eq && rank < need))) ? 1 : 0;
    rank += eq ? 1 : 0;
  }
}

// candidate export: the selected local rows as (value, global index) pairs,
// index-ordered, padded with (0, -1) up to k.  cand layout: [k values][k idx]
__global__ void k_export_candidates(int64_t k, const int* __restrict__ n_act_dev,
                                    const int* __restrict__ rowidx, const double* __restrict__ Q,
                                    int64_t goff, double* __restrict__ cand) {
  int na = *n_act_dev;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < k;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (r < na) { cand[r] = Q[rowidx[r]]; cand[k + r] = (double)(goff + rowidx[r]); }
    else { cand[r] = 0.0; cand[k + r] = -1.0; }
  }
}

// gathered candidates [rank][2k] -> contiguous values / indices (rank order)
__global__ void k_unpack_candidates(int n_ranks, int64_t k, const double* __restrict__ all,
                                    double* __restrict__ vals, double* __restrict__ gidx) {
  int64_t tot = (int64_t)n_ranks * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / k, j = e % k;
    vals[e] = all[r * 2 * k + j];
    gidx[e] = all[r * 2 * k + k + j];
  }
}

// global selection over the gathered candidates -> its global indices in
// ascending order.  Candidates arrive rank-major and, within a rank, in
// ascending local row order (ordered compaction), so an ordered compaction of
// the mask is already sorted.  One block of 1024 threads.
__global__ void __launch_bounds__(1024)
k_selection_gidx(int64_t ncand, const uint8_t* __restrict__ cmask, const double* __restrict__ gidx,
                 int64_t k, int64_t* __restrict__ out) {
  __shared__ int s_w[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t base_out = 0;
  for (int64_t base = 0; base < ncand; base += 1024) {
    const int64_t e = base + tid;
    const bool f = e < ncand && cmask[e] && gidx[e] >= 0.0;
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_w[warp] = __popc(b);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < 32; ++w) { const int c = s_w[w]; before += (w < warp) ? c : 0; tot += c; }
    const int64_t pos = base_out + before + __popc(b & ((1u << lane) - 1u));
    if (f && pos < k) out[pos] = (int64_t)gidx[e];
    base_out += tot;
    __syncthreads();
  }
  for (int64_t p = base_out + tid; p < k; p += 1024) out[p] = -1;   // (never: the merge selects k)
}

// global selection mask over candidates -> local selection mask
__global__ void k_scatter_selection(int64_t ncand, const uint8_t* __restrict__ cmask,
                                    const double* __restrict__ gidx, int64_t goff, int64_t n,
                                    uint8_t* __restrict__ sel) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncand;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!cmask[e]) continue;
    int64_t g = (int64_t)gidx[e] - goff;
    if (g >= 0 && g < n) sel[g] = 1;
  }
}

// strided copy of G (n x ldg) -> dense (n x d_z) fp64
__global__ void k_copy_g(int64_t n, int d_z, int ldg, const float* __restrict__ G, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * d_z;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / d_z; int k = (int)(e % d_z);
    out[e] = G[i * ldg + k];
  }
}

// forward-mode layer-1 tangent: T[(i,k), c] = D0[i, c] * Pz[c, k]  (the
// tangent of x_z = V_z^T z through W1_z is the constant W1_z V_z^T)
__global__ void k_tangent_seed(int64_t rows, int d_z, int h1, const float* __restrict__ D0,
                               const float* __restrict__ Pz32t /* d_z x h1 */, float* __restrict__ T) {
  int64_t r = blockIdx.x;
  if (r >= rows) return;
  int64_t i = r / d_z; int k = (int)(r % d_z);
  for (int c = threadIdx.x; c < h1; c += blockDim.x)
    T[r * h1 + c] = (D0 ? D0[i * h1 + c] : 1.0f) * Pz32t[(int64_t)k * h1 + c];
}

// the same seed written as the first tangent GEMM's bf16x3 split operand
// (rows x ld, columns [h1, ld) zero): T[(i,k), c] = D0[i, c] Pz[k, c]
__global__ void __launch_bounds__(256)
k_tangent_seed_split(int64_t rows, int d_z, int h1, int ld, const float* __restrict__ D0,
                     const float* __restrict__ Pz32t, __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  // one warp per tangent row (8 rows per block, grid-strided), lanes over column pairs
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * 8) {
    const unsigned i = (unsigned)(r / d_z), k = (unsigned)(r - (int64_t)i * d_z);
    const float* dr = D0 ? D0 + (int64_t)i * h1 : nullptr;
    const float* pr = Pz32t + (int64_t)k * h1;
    __nv_bfloat162* ph = reinterpret_cast<__nv_bfloat162*>(hi + r * ld);
    __nv_bfloat162* pl = reinterpret_cast<__nv_bfloat162*>(lo + r * ld);
    for (int c = 2 * lane; c < ld; c += 64) {
      float x0 = 0.0f, x1 = 0.0f;
      if (c < h1) x0 = (dr ? __ldg(dr + c) : 1.0f) * __ldg(pr + c);
      if (c + 1 < h1) x1 = (dr ? __ldg(dr + c + 1) : 1.0f) * __ldg(pr + c + 1);
      const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1b = __float2bfloat16_rn(x1);
      ph[c / 2] = __halves2bfloat162(h0, h1b);
      pl[c / 2] = __halves2bfloat162(__float2bfloat16_rn(x0 - __bfloat162float(h0)),
                                     __float2bfloat16_rn(x1 - __bfloat162float(h1b)));
    }
  }
}

// linear model Jacobian (one layer): dy/dz rows are the seed; scale by the
// output std into Jt (rows x r_u, decoded next) or scatter into J[i, u, k]
__global__ void k_scale_cols(int64_t rows, int r_u, const float* __restrict__ scale, const float* __restrict__ T,
                             float* __restrict__ Jt, float* __restrict__ J, int d_z) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * r_u;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / r_u;
    const int u = (int)(e % r_u);
    const float v = scale[u] * T[e];
    if (Jt) Jt[e] = v;
    else J[((r / d_z) * r_u + u) * d_z + r % d_z] = v;
  }
}

// decoder set-up on the device (pod.py:104-110): Um = diag(M) U (fp32 of the
// fp64 product, the Gram GEMM's A), and per block j < r_u the fixed-order fp64
// c_j = sum_d U[d, j] (M s)[d] with s = b - u_t; block r_u: q0 = s.(M s)
__global__ void k_dec_scale(int64_t d_u, int r_u, const float* __restrict__ U, const float* __restrict__ Mdiag,
                            float* __restrict__ Um) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d_u * r_u;
       e += (int64_t)gridDim.x * blockDim.x)
    Um[e] = (float)((double)Mdiag[e / r_u] * (double)U[e]);
}
// ms = M (b - u_t) in fp64: lumped mass (Mdiag) or a general sparse mass in
// CSR (riskopt.py:103-108 takes any scipy sparse M; one warp per row, the
// row's entries in stored order, fixed butterfly)
__global__ void __launch_bounds__(256)
k_dec_ms(int64_t d_u, const float* __restrict__ ub, const float* __restrict__ ut, const float* __restrict__ Mdiag,
         const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, const float* __restrict__ data,
         double* __restrict__ ms) {
  if (Mdiag) {
    for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < d_u; d += (int64_t)gridDim.x * blockDim.x)
      ms[d] = (double)Mdiag[d] * ((double)ub[d] - (double)ut[d]);
    return;
  }
  const int lane = threadIdx.x & 31;
  for (int64_t d = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); d < d_u;
       d += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    double acc = 0.0;
    for (int64_t e = indptr[d] + lane; e < indptr[d + 1]; e += 32) {
      const int32_t q = indices[e];
      acc += (double)data[e] * ((double)ub[q] - (double)ut[q]);
    }
    acc = warp_sum(acc);
    if (lane == 0) ms[d] = acc;
  }
}
// Um = M U for a CSR mass (fp32 of the fp64 row sums): one warp per row, lanes
// over the r_u columns, the row's entries in stored order
__global__ void __launch_bounds__(256)
k_dec_spmm(int64_t d_u, int r_u, const float* __restrict__ U, const int64_t* __restrict__ indptr,
           const int32_t* __restrict__ indices, const float* __restrict__ data, float* __restrict__ Um) {
  const int lane = threadIdx.x & 31;
  for (int64_t d = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); d < d_u;
       d += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t e0 = indptr[d], e1 = indptr[d + 1];
    for (int j = lane; j < r_u; j += 32) {
      double acc = 0.0;
      for (int64_t e = e0; e < e1; ++e) acc += (double)data[e] * (double)U[(int64_t)indices[e] * r_u + j];
      Um[d * r_u + j] = (float)acc;
    }
  }
}
__global__ void __launch_bounds__(256)
k_dec_c(int64_t d_u, int r_u, const float* __restrict__ U, const float* __restrict__ ub,
        const double* __restrict__ msv, const float* __restrict__ ut, double* __restrict__ c, double* __restrict__ q0) {
  __shared__ double sw[8];
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int64_t d = threadIdx.x; d < d_u; d += blockDim.x) {
    const double sd = (double)ub[d] - (double)ut[d], ms = msv[d];
    acc += j < r_u ? (double)U[d * r_u + j] * ms : sd * ms;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sw[w];
    if (j < r_u) c[j] = t;
    else *q0 = t;
  }
}
// ---- tensor-core encoder operands: a three-way bf16 split x = p0 + p1 + p2
// (p0 = bf16(x), p1 = bf16(x - p0), p2 = bf16(x - p0 - p1): 24 mantissa bits,
// every subtraction exact).  With both operands split three ways, the products
// p_i q_j with i + j <= 2 carry the fp32 product to ~2^-24.  Layout, per K chunk
// of kc columns and per row: segments [p0 | p1 | p2 | p0] of kc values each
// (chunk-major, row length 4 kc), so that
//   pass A = ONE bf16x3 GEMM over K' = 2 kc with hi = the row at +0 (p0, p1) and
//            lo = the same row at +kc (p1, p2): (p0;p1)x(q0;q1) + (p1;p2)x(q1;q2),
//   pass B = ONE hi-only GEMM over K' = 2 kc with A hi at +2 kc (p2, p0) and B
//            from a second buffer [q0 | q2]: p2 q0 + p0 q2
// (engine.cu, sdn_encode_fields).  Columns >= cols are zero.
SDN_DEV void split3(float x, __nv_bfloat16& a, __nv_bfloat16& b, __nv_bfloat16& c) {
  a = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(a);
  b = __float2bfloat16_rn(r1);
  c = __float2bfloat16_rn(r1 - __bfloat162float(b));
}
// (chunk-major: chunk ch of every row first -- P[ch][row][4 kc] -- so a GEMM tile's
// rows are 8 KB apart instead of a whole plane row: DRAM pages are reused across
// the tile's k-blocks; rows_alloc = rows of the buffer per chunk)
__global__ void k_split3(int64_t rows, int cols, int64_t ld_src, const float* __restrict__ src, int nch, int kc,
                         int64_t rows_alloc, __nv_bfloat16* __restrict__ P) {
  // eight consecutive columns per thread: four 16-byte stores (kc % 8 == 0)
  const int64_t per_row = (int64_t)nch * kc, groups = per_row / 8, total = rows * groups;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / groups;
    const int64_t k = (e - r * groups) * 8;
    const int64_t ch = k / kc, kk = k - ch * kc;
    union { __nv_bfloat16 v[8]; uint4 u; } pa, pb, pc;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float x = k + j < cols ? __ldg(src + r * ld_src + k + j) : 0.0f;
      split3(x, pa.v[j], pb.v[j], pc.v[j]);
    }
    __nv_bfloat16* q = P + (ch * rows_alloc + r) * 4 * kc + kk;
    *reinterpret_cast<uint4*>(q) = pa.u;
    *reinterpret_cast<uint4*>(q + kc) = pb.u;
    *reinterpret_cast<uint4*>(q + 2 * kc) = pc.u;
    *reinterpret_cast<uint4*>(q + 3 * (int64_t)kc) = pa.u;
  }
}
// the same for V (d x r, row-major) transposed: rows of V^T in P ([q0 | q1 | q2 | q0]
// per chunk, chunk-major) and the pass-B operand [q0 | q2] per chunk in P2 (row length 2 kc)
__global__ void k_split3_transpose(int64_t d, int r, const float* __restrict__ V, int nch, int kc,
                                   __nv_bfloat16* __restrict__ P, __nv_bfloat16* __restrict__ P2) {
  __shared__ float tile[32][33];
  const int64_t d0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  const int64_t per_row = (int64_t)nch * kc;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t dd = d0 + i;
    const int j = j0 + threadIdx.x;
    tile[i][threadIdx.x] = (dd < d && j < r) ? V[dd * r + j] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int j = j0 + i;
    const int64_t k = d0 + threadIdx.x;
    if (j < r && k < per_row) {
      __nv_bfloat16 a, b, c;
      split3(tile[threadIdx.x][i], a, b, c);
      const int64_t ch = k / kc, kk = k - ch * kc;
      __nv_bfloat16* q = P + (ch * r + j) * 4 * kc + kk;
      q[0] = a; q[kc] = b; q[2 * kc] = c; q[3 * (int64_t)kc] = a;
      __nv_bfloat16* q2 = P2 + (ch * r + j) * 2 * kc + kk;
      q2[0] = a; q2[kc] = c;
    }
  }
}
// encoder: bias_j = -m_mean sum_d Vmm[d, j] (fixed-order fp64, one block per j)
__global__ void __launch_bounds__(256)
k_enc_bias(int64_t d_m, int r_m, const float* __restrict__ Vmm, double m_mean, double* __restrict__ bias) {
  __shared__ double sw[8];
  const int j = blockIdx.x;
  double acc = 0.0;
  for (int64_t d = threadIdx.x; d < d_m; d += blockDim.x) acc += (double)Vmm[d * r_m + j];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sw[w];
    bias[j] = -m_mean * t;
  }
}
// MR = float(acc + bias)
__global__ void k_enc_finish(int64_t n, int r_m, const double* __restrict__ acc, const double* __restrict__ bias,
                             float* __restrict__ MR) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r_m; e += (int64_t)gridDim.x * blockDim.x)
    MR[e] = (float)(acc[e] + bias[e % r_m]);
}
__global__ void k_f64_to_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[e] = (float)a[e];
}

// ---- per-layer vector softmax (surrogate.py:175-177, 214-217), SIMT chains
// One warp per row, fp64 row reductions (fixed lane order), widths <= any.
// forward: a = softmax(S) over the row; H = [prev +] a; D = a (for the sweep)
__global__ void __launch_bounds__(256)
k_softmax_rows(int64_t n, int w, float* __restrict__ H, float* __restrict__ D, const float* __restrict__ prev) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  float* h = H + r * w;
  float mx = -INFINITY;
  for (int c = lane; c < w; c += 32) mx = fmaxf(mx, h[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double sum = 0.0;
  for (int c = lane; c < w; c += 32) sum += exp((double)h[c] - (double)mx);
  sum = warp_sum(sum);
  for (int c = lane; c < w; c += 32) {
    const float a = (float)(exp((double)h[c] - (double)mx) / sum);
    if (D) D[r * w + c] = a;
    h[c] = prev ? prev[r * w + c] + a : a;
  }
}

// reverse: u = a (g - a.g) in place on U (rows r < *n_dev; a = D[rowidx[r]])
__global__ void __launch_bounds__(256)
k_softmax_bwd(int64_t n, const int* __restrict__ n_dev, const int* __restrict__ rowidx, int w,
              const float* __restrict__ D, float* __restrict__ U) {
  const int64_t nr = n_dev ? (int64_t)*n_dev : n;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= nr) return;
  const float* a = D + (rowidx ? (int64_t)rowidx[r] : r) * w;
  float* u = U + r * w;
  double dot = 0.0;
  for (int c = lane; c < w; c += 32) dot += (double)a[c] * (double)u[c];
  dot = warp_sum(dot);
  for (int c = lane; c < w; c += 32) u[c] = (float)((double)a[c] * ((double)u[c] - dot));
}

// tangent rows (sample i = r / rowdiv): T = a (U - a.U) [+ Tin]
__global__ void __launch_bounds__(256)
k_softmax_tangent(int64_t rows, int rowdiv, int w, const float* __restrict__ D, float* __restrict__ U,
                  const float* __restrict__ tin) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* a = D + (r / rowdiv) * w;
  float* u = U + r * w;
  double dot = 0.0;
  for (int c = lane; c < w; c += 32) dot += (double)a[c] * (double)u[c];
  dot = warp_sum(dot);
  for (int c = lane; c < w; c += 32) {
    const float t = (float)((double)a[c] * ((double)u[c] - dot));
    u[c] = tin ? tin[r * w + c] + t : t;
  }
}

}  // namespace sdn
