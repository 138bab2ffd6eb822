// refine.cuh -- fused fp64 Q refinement.
//
// Q from the bf16x3 (or fp32) chain carries ~1e-5 relative error (the
// tensor-core accumulation also biases it slightly low).  Where the risk is
// discontinuous or steep in Q -- the exact-CVaR selection boundary, the
// smoothed-CVaR window [t, t + eps] -- the rows within that error of the
// boundary are re-evaluated by an fp64 chain over the same fp32 weights (the
// oracle's arithmetic) and their Q replaced in place.
//
// One cooperative launch does the whole refinement: ordered band compaction,
// the L layers, the QoI, and (exact CVaR) the reselection among band rows,
// separated by grid barriers.  The work is tiny (a handful of rows) and
// latency-bound, so the point of the fusion is one launch and one barrier per
// layer instead of a dependent kernel chain, with every layer's W rows
// prefetched into L2 up front.
#pragma once
#include "kernels.cuh"

namespace sdn {

constexpr int REF_RB = 8;             // rows per pass (= warps per block: warp j stages row j)
constexpr int REF_KC = 1024;          // max layer input width on the fused path
constexpr int REF_THREADS = 256;
constexpr int REF_MAX_LAYERS = 16;

struct RefineLayer {
  const float* W;     // N x K (layer 0: W1[:, :r_m] unscaled)
  const float* b;     // N (layer 0: unused, b64 = zb64)
  int K, N, resid;
};

struct RefineArgs {
  // band selection
  int64_t n;
  int kind;                     // RISK_BAND (t, eps) or RISK_BAND_EXACT (*tdev)
  double t, eps;
  const double* tdev;
  int* rowidx;
  int* count;                   // band row count (read back by the host)
  int* blockcnt;                // gridDim.x scratch
  unsigned* bar;                // grid barrier {arrivals, generation}
  // chain
  int L;
  RefineLayer layer[REF_MAX_LAYERS];
  const float* MR;
  const float* iscale;
  const double* zb64;
  int act;
  const float* omean;
  const float* ostd;
  double* buf[2];               // cap_rows x maxw ping-pong
  int cap_rows;
  // QoI
  int r_u;
  const float* c32;
  const double* K64;            // decoded frame (null = reduced)
  const double* c64;
  double q0;
  double* Q;
  // exact CVaR: reselect among the band rows (null = no reselection)
  uint8_t* mask;
};

// Data written inside this kernel by other blocks (rowidx, the layer
// ping-pong, Q) is read with ld.global.cg (L2): L1 is not coherent across SMs.

SDN_DEV int warp_sum_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// grid-wide barrier (all blocks co-resident: cooperative launch)
SDN_DEV void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned arrived = atomicAdd(&bar[0], 1u);
    if (arrived == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicExch(&bar[1], gen + 1u);
    } else {
      while (*(volatile unsigned*)&bar[1] == gen) __nanosleep(20);
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

// block-wide exclusive scan helper over per-warp counts (REF_THREADS / 32 warps)
SDN_DEV int block_excl(int* s_w, int warp, int lane, int v, int& total) {
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < REF_THREADS / 32; ++w) {
    const int c = s_w[w];
    if (w < warp) base += c;
    tot += c;
  }
  __syncthreads();
  total = tot;
  return base;
}

__global__ void __launch_bounds__(REF_THREADS, 1) k_refine(RefineArgs a) {
  extern __shared__ double xs[];                  // REF_RB x REF_KC
  __shared__ int s_w[REF_THREADS / 32], s_m[REF_THREADS / 32];
  __shared__ unsigned s_gen;
  __shared__ int s_need;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x;
  if (tid == 0) s_gen = *(volatile unsigned*)&a.bar[1];
  __syncthreads();
  unsigned gen = s_gen;

  // ---- 1. band flags and ordered compaction (contiguous slice per block)
  const int64_t per = (a.n + G - 1) / G;
  const int64_t lo = min((int64_t)blockIdx.x * per, a.n), hi = min(lo + per, a.n);
  int mine = 0;
  for (int64_t base = lo; base < hi; base += REF_THREADS) {
    const int64_t i = base + tid;
    const bool f = i < hi && row_flag(a.kind, a.Q, nullptr, i, a.t, a.eps, a.tdev);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    mine += (lane == 0) ? __popc(b) : 0;
  }
  int tot;
  (void)block_excl(s_w, warp, lane, mine, tot);
  if (tid == 0) a.blockcnt[blockIdx.x] = tot;
  grid_barrier(a.bar, gen);
  int off = 0, m = 0;
  {                                              // block offsets: parallel loads, warp sums
    int po = 0, pm = 0;
    for (unsigned b = tid; b < G; b += REF_THREADS) {
      const int c = __ldcg(a.blockcnt + b);
      po += (b < blockIdx.x) ? c : 0;
      pm += c;
    }
    po = warp_sum_i(po);
    pm = warp_sum_i(pm);
    __syncthreads();
    if (lane == 0) { s_w[warp] = po; s_m[warp] = pm; }
    __syncthreads();
    for (int w = 0; w < REF_THREADS / 32; ++w) { off += s_w[w]; m += s_m[w]; }
    __syncthreads();
  }
  for (int64_t base = lo; base < hi; base += REF_THREADS) {
    const int64_t i = base + tid;
    const bool f = i < hi && row_flag(a.kind, a.Q, nullptr, i, a.t, a.eps, a.tdev);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    int t2;
    const int wb = block_excl(s_w, warp, lane, __popc(b), t2);
    if (f) a.rowidx[off + wb + __popc(b & ((1u << lane) - 1u))] = (int)i;
    off += t2;
  }
  if (blockIdx.x == 0 && tid == 0) *a.count = m;
  if (m == 0 || m > a.cap_rows) return;          // uniform: every block computed the same m
  grid_barrier(a.bar, gen);

  // ---- 2. fp64 chain over the m band rows
  const int gw = blockIdx.x * (REF_THREADS / 32) + warp, nw = G * (REF_THREADS / 32);
  for (int l = 0; l < a.L; ++l) {                // W rows of every layer -> L2 now
    const RefineLayer& ly = a.layer[l];
    for (int c = gw; c < ly.N; c += nw) {
      const char* row = reinterpret_cast<const char*>(ly.W + (int64_t)c * ly.K);
      for (int o = lane * 128; o < ly.K * 4; o += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
    }
  }
  for (int l = 0; l < a.L; ++l) {
    const RefineLayer& ly = a.layer[l];
    const int K = ly.K, N = ly.N;
    const bool first = l == 0, last = l == a.L - 1;
    const double* in64 = first ? nullptr : a.buf[(l - 1) & 1];
    double* out = a.buf[l & 1];
    for (int r0 = 0; r0 < m; r0 += REF_RB) {
      const int rb = min(REF_RB, m - r0);
      {                                          // warp j stages row r0 + j (clamped)
        const int rj = r0 + min(warp, rb - 1);
        if (first) {
          const float* src = a.MR + (int64_t)__ldcg(a.rowidx + rj) * K;
          float v[REF_KC / 32];
#pragma unroll
          for (int u = 0; u < REF_KC / 32; ++u) v[u] = __ldg(src + min(lane + 32 * u, K - 1));
#pragma unroll
          for (int u = 0; u < REF_KC / 32; ++u)
            if (lane + 32 * u < K) xs[warp * REF_KC + lane + 32 * u] = (double)v[u];
        } else {
          const double* src = in64 + (int64_t)rj * K;
          double v[REF_KC / 32];
#pragma unroll
          for (int u = 0; u < REF_KC / 32; ++u) v[u] = __ldcg(src + min(lane + 32 * u, K - 1));
#pragma unroll
          for (int u = 0; u < REF_KC / 32; ++u)
            if (lane + 32 * u < K) xs[warp * REF_KC + lane + 32 * u] = v[u];
        }
      }
      __syncthreads();
      for (int c = gw; c < N; c += nw) {
        const float* w = ly.W + (int64_t)c * K;
        float wf[REF_KC / 32], sf[REF_KC / 32];   // unconditional clamped loads: all in flight
#pragma unroll
        for (int u = 0; u < REF_KC / 32; ++u) {
          const int k = min(lane + 32 * u, K - 1);
          wf[u] = __ldg(w + k);
          sf[u] = first ? __ldg(a.iscale + k) : 1.0f;
        }
        double acc[REF_RB];
#pragma unroll
        for (int j = 0; j < REF_RB; ++j) acc[j] = 0.0;
#pragma unroll
        for (int u = 0; u < REF_KC / 32; ++u) {
          if (lane + 32 * u < K) {
            const double wk = (double)wf[u] * (double)sf[u];
#pragma unroll
            for (int j = 0; j < REF_RB; ++j) acc[j] = fma(xs[j * REF_KC + lane + 32 * u], wk, acc[j]);
          }
        }
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < REF_RB; ++j) {
          const double s = warp_sum(acc[j]);
          if (lane == j) v = s;
        }
        if (lane < rb) {
          const double S = v + (first ? a.zb64[c] : (double)ly.b[c]);
          double o;
          if (last) {
            o = (double)a.omean[c] + (double)a.ostd[c] * S;
          } else {
            o = act64(a.act, S);
            if (ly.resid) o += xs[lane * REF_KC + c];     // resid: K == N
          }
          out[(int64_t)(r0 + lane) * N + c] = o;
        }
      }
      __syncthreads();
    }
    grid_barrier(a.bar, gen);
  }

  // ---- 3. QoI of the band rows -> Q (reduced: phi.(phi + 2c); decoded: phi.(K phi + 2c))
  const double* phi = a.buf[(a.L - 1) & 1];
  for (int r = gw; r < m; r += nw) {
    const double* p = phi + (int64_t)r * a.r_u;
    double s = 0.0;
    for (int j = lane; j < a.r_u; j += 32) {
      double kp;
      if (a.K64) {
        kp = 2.0 * a.c64[j];
        for (int q = 0; q < a.r_u; ++q) kp = fma(a.K64[(int64_t)j * a.r_u + q], __ldcg(p + q), kp);
      } else {
        kp = __ldcg(p + j) + 2.0 * (double)a.c32[j];
      }
      s = fma(__ldcg(p + j), kp, s);
    }
    s = warp_sum(s);
    if (lane == 0) a.Q[__ldcg(a.rowidx + r)] = s + a.q0;
  }
  if (!a.mask) return;
  grid_barrier(a.bar, gen);

  // ---- 4. exact CVaR: the band holds `need` selected rows (rows outside keep
  // their side of the threshold); take the top `need` band rows by
  // (Q desc, position asc).  One block; m <= cap_rows <= 16 * REF_THREADS.
  if (blockIdx.x != 0) return;
  if (tid == 0) s_need = 0;
  __syncthreads();
  int cnt = 0;
  for (int r = tid; r < m; r += REF_THREADS) cnt += a.mask[__ldcg(a.rowidx + r)] ? 1 : 0;
  atomicAdd(&s_need, cnt);
  __syncthreads();
  const int need = s_need;
  bool selr[16];
  int t = 0;
  for (int r = tid; r < m && t < 16; r += REF_THREADS, ++t) {
    const int ri = __ldcg(a.rowidx + r);
    const uint64_t ki = dkey(__ldcg(a.Q + ri));
    int rank = 0;
    for (int u = 0; u < m; ++u) {
      const int rj = __ldcg(a.rowidx + u);
      const uint64_t kj = dkey(__ldcg(a.Q + rj));
      rank += (kj > ki || (kj == ki && rj < ri)) ? 1 : 0;
    }
    selr[t] = rank < need;
  }
  __syncthreads();                               // every rank computed from the pre-update mask
  t = 0;
  for (int r = tid; r < m && t < 16; r += REF_THREADS, ++t) a.mask[__ldcg(a.rowidx + r)] = selr[t] ? 1 : 0;
}

}  // namespace sdn
