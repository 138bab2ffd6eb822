// small.cuh -- the whole SAA evaluation of a SMALL sample set in ONE launch
// (BASELINE config 1: 256 samples, MLP 89 -> 256 x 3 -> 64, mean + beta var).
//
// At c1 the layer-by-layer path is ~20 dependent kernels of a few microseconds
// each: 0.16 GFLOP of work paced by launch latency (0.09 ms per evaluation).
// Samples are independent until the risk reduction, so here every CTA owns RB
// sample rows and runs the whole path for them out of shared memory:
//   zb = b1 + Pz z; forward chain (fp32 FFMA, activations and act' kept in
//   shared memory -- surrogate.py:161-191); Q in fp64 (riskopt.py:187-189);
//   unit-seed reverse sweep to u0 = dQ/dS1 (the reverse-mode equivalent of
//   surrogate.py:195-224); fp64 per-CTA sums.
// The mean / mean + beta var weights are affine in Q_i:
//   sum_i w_i u0_i = [(1 - 2 beta m1) A1 + 2 beta A2] / n,
//   A1 = sum_i u0_i, A2 = sum_i (Q_i - shift) u0_i, m1 = sum_i (Q_i - shift) / n
// so no grid-wide step separates the forward from the sweep: each CTA writes
// its partial (A1, A2, moments), and the last CTA to finish (atomic ticket)
// adds them in CTA order, applies each risk's coefficients, projects through
// PzT and writes the results to host-mapped memory.  Deterministic: fixed
// per-CTA row order, fixed CTA order in the final sums.
//
// The weights (1.3 MB per CTA and evaluation at c1) stream from L2 through a
// shared-memory ring of 32-row chunks filled by 1-D bulk copies
// (cp.async.bulk + mbarrier) that run ahead across layer boundaries: the
// chunk list of the whole evaluation (forward: rows of W^T; sweep: rows of W)
// is fixed, so the ring never drains; each CTA starts a matrix at its own
// chunk so the CTAs do not hammer the same L2 lines in step.  (Loading each
// weight straight into registers, 8 loads in flight per thread, was
// latency-bound: 0.14 ms; all CTAs in step through the ring: 0.054 ms.)
#pragma once
#include "kernels.cuh"

namespace sdn {

constexpr int SM_MAXW = 256;         // widest layer (one output column per thread)
constexpr int SM_MAXL = 8;           // weight matrices
constexpr int SM_THREADS = 256;
constexpr int SM_CH = 32;            // matrix rows per chunk
constexpr int SM_STAGES = 5;         // ring depth (<= 32 KB per stage; 3 stages: 0.83 us per chunk, latency-bound)

struct SmallArgs {
  unsigned long long* trace;         // optional %globaltimer stamps (SDN_SMALL_TRACE=1): CTA 0 phases, then the last CTA's
  int L, n, r_m, d_z, r_u, h1, act, R, plen;
  int w[SM_MAXL + 1];
  int res[SM_MAXL];
  const float* W[SM_MAXL];           // w[l+1] x w[l]  (W[0]: h1 x r_m, whitening folded in)
  const float* WT[SM_MAXL];          // w[l] x w[l+1]  (transposed copies: the forward streams rows of W^T)
  const float* b[SM_MAXL];
  const float* MR;
  const double* Pz;                  // h1 x d_z
  const double* z;                   // d_z (device)
  const float* omean;
  const float* ostd;
  const float* c;                    // r_u
  double q0, shift;
  int kind[SDN_RMAX];
  double beta[SDN_RMAX];
  double* Q;                         // n
  double* part;                      // gridDim.x x (2 h1 + 4)
  const double* PzT;                 // d_z x h1
  double* stats;                     // STATS_LEN (device copy)
  double* out;                       // R x plen (device copy)
  int* counter;
  double* hstats;                    // host-mapped results
  double* hpart;
  int* hband;
  int nband;
};

SDN_DEV void sm_stamp(const SmallArgs& a, int k, bool who) {
  if (a.trace && who && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[k] = t;
  }
}
SDN_DEV uint32_t sm_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// one chunk = one mbarrier phase, moved by SM_SPLIT bulk copies (1: splitting a
// chunk into 8 copies was slower, 0.072 vs 0.054 ms -- the issuing thread is
// on the CTA's critical path)
#ifndef SM_SPLIT
#define SM_SPLIT 1
#endif
SDN_DEV void sm_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(bar)), "r"(bytes) : "memory");
  const uint32_t piece = ((bytes / SM_SPLIT) + 15u) & ~15u;
  for (uint32_t o = 0; o < bytes; o += piece) {
    const uint32_t nb = min(piece, bytes - o);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sm_u32(dst) + o),
                 "l"(reinterpret_cast<const char*>(src) + o), "r"(nb), "r"(sm_u32(bar))
                 : "memory");
  }
}
SDN_DEV void sm_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SM_WAIT_%=;\n}" ::"r"(sm_u32(bar)),
      "r"(parity)
      : "memory");
}

// the evaluation's chunk list, in consumption order: forward l = 0..L-1 rows of
// WT[l] (K_l rows of N_l floats), then the sweep l = L-1..1 rows of W[l]
// (N_l rows of K_l floats); chunk i -> (source, bytes)
// Every CTA streams the same matrices; walking them in the same order at the
// same time makes all CTAs hit the same few L2 lines at once (measured: 2400
// cycles per 32-KB chunk with 64 CTAs in step).  So CTA b starts each matrix at
// chunk b mod nch and wraps around: at any time the CTAs read different
// chunks.  (The K order of a dot product then depends on the CTA -- still
// fixed for a given sample row.)
SDN_DEV int small_chunk(int i, int nch) { return (int)((blockIdx.x + (unsigned)i) % (unsigned)nch); }
struct SmallWalk {
  int l, row, phase;                 // phase 0 forward, 1 sweep, 2 done; row: chunks of this matrix handed out
  SDN_DEV void init() { l = 0; row = 0; phase = 0; }
  SDN_DEV bool next(const SmallArgs& a, const float*& src, uint32_t& bytes) {
    while (phase < 2) {
      const int rows = phase == 0 ? a.w[l] : a.w[l + 1], ld = phase == 0 ? a.w[l + 1] : a.w[l];
      const int nch = (rows + SM_CH - 1) / SM_CH;
      if (row < nch) {
        const int r0 = small_chunk(row, nch) * SM_CH, nr = min(SM_CH, rows - r0);
        src = (phase == 0 ? a.WT[l] : a.W[l]) + (int64_t)r0 * ld;
        bytes = (uint32_t)(nr * ld) * 4u;
        ++row;
        return true;
      }
      row = 0;
      if (phase == 0) {
        if (++l == a.L) { phase = 1; l = a.L - 1; if (l < 1) phase = 2; }
      } else {
        if (--l < 1) phase = 2;
      }
    }
    return false;
  }
};

// the shared-memory ring, consumed by every thread in lock step
struct SmallRing {
  float* buf;                        // SM_STAGES x SM_CH x SM_MAXW
  uint64_t* bar;                     // SM_STAGES
  SmallWalk prod;                    // thread 0: next chunk to request
  int ci;                            // chunks consumed so far
  SDN_DEV void fill(const SmallArgs& a, int stage) {             // thread 0 only
    const float* src;
    uint32_t bytes;
    if (prod.next(a, src, bytes)) sm_bulk_load(buf + (size_t)stage * SM_CH * SM_MAXW, src, bytes, &bar[stage]);
  }
  SDN_DEV const float* acquire() {                                // all threads: chunk ci is in shared memory
    const int s = ci % SM_STAGES;
    sm_wait(&bar[s], (uint32_t)(ci / SM_STAGES) & 1u);
    return buf + (size_t)s * SM_CH * SM_MAXW;
  }
  SDN_DEV void release(const SmallArgs& a) {                      // all threads are done with chunk ci
    __syncthreads();
    if (threadIdx.x == 0) fill(a, ci % SM_STAGES);
    ++ci;
  }
};

// acc[r] += sum_k x[k][r] * Mrows[k][col] over the `rows` matrix rows streamed
// through the ring (x k-major in shared memory: the RB rows of one input
// feature are contiguous)
template <int RB>
SDN_DEV void small_dot(const SmallArgs& a, SmallRing& ring, const float* __restrict__ x, int rows, int ld, int col,
                       bool active, float (&acc)[RB]) {
  const int nch = (rows + SM_CH - 1) / SM_CH;
  for (int i = 0; i < nch; ++i) {
    const float* wc = ring.acquire();
    const int k0 = small_chunk(i, nch) * SM_CH, nk = min(SM_CH, rows - k0);
    if (active) {
#pragma unroll 8
      for (int k = 0; k < nk; ++k) {
        const float wv = wc[k * ld + col];
        const float* xr = x + (k0 + k) * RB;
#pragma unroll
        for (int r = 0; r < RB; r += 4) {
          const float4 v = *reinterpret_cast<const float4*>(xr + r);
          acc[r] = fmaf(wv, v.x, acc[r]); acc[r + 1] = fmaf(wv, v.y, acc[r + 1]);
          acc[r + 2] = fmaf(wv, v.z, acc[r + 2]); acc[r + 3] = fmaf(wv, v.w, acc[r + 3]);
        }
      }
    }
    ring.release(a);
  }
}

template <int RB>
__global__ void __launch_bounds__(SM_THREADS, 1) k_small_eval(const SmallArgs a) {
  static_assert(RB == 4 || RB == 8, "rows per CTA");
  extern __shared__ __align__(128) float sm[];
  __shared__ double sred[RB][4];
  __shared__ __align__(8) uint64_t bars[SM_STAGES];
  __shared__ bool s_last;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int L = a.L, NH = L - 1;
  // layout: ring | two activation buffers [SM_MAXW][RB] | act' per hidden layer | zb
  SmallRing ring;
  ring.buf = sm;
  ring.bar = bars;
  ring.ci = 0;
  float* hb0 = sm + (size_t)SM_STAGES * SM_CH * SM_MAXW;
  float* hb1 = hb0 + SM_MAXW * RB;
  float* Ds = hb1 + SM_MAXW * RB;                  // [NH][SM_MAXW][RB]
  float* zb = Ds + (size_t)NH * SM_MAXW * RB;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nr = (int)min((int64_t)RB, (int64_t)a.n - r0);        // valid rows of this CTA

  const bool c0 = blockIdx.x == 0;
  sm_stamp(a, 0, c0);
  if (t == 0) {
    for (int s = 0; s < SM_STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm_u32(&bars[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ring.prod.init();
    for (int s = 0; s < SM_STAGES; ++s) ring.fill(a, s);          // the weights start streaming at once
  }
  // every weight line -> L2 now, the CTAs sharing the work: the bench (and an
  // optimizer between evaluations) leaves the weights cold, and a ring that is
  // two chunks ahead cannot hide a DRAM miss per chunk
  for (int l = 0; l < L; ++l) {
    const size_t lines = ((size_t)a.w[l] * a.w[l + 1] * 4 + 127) / 128;
    for (size_t i = (size_t)blockIdx.x * SM_THREADS + t; i < lines; i += (size_t)gridDim.x * SM_THREADS) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.WT[l]) + i * 128));
      if (l >= 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.W[l]) + i * 128));
    }
  }
  {                                                // ... and PzT for the last CTA's projection
    const size_t lines = ((size_t)a.d_z * a.h1 * 8 + 127) / 128;
    for (size_t i = (size_t)blockIdx.x * SM_THREADS + t; i < lines; i += (size_t)gridDim.x * SM_THREADS)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(a.PzT) + i * 128));
  }
  // zb = b1 + Pz z (fp64 sum, rounded once), and the CTA's input rows (k-major)
  // (one global round trip: every thread's Pz row and the staged z are in
  // flight together -- the inputs are DRAM-cold after an optimizer step)
  double* zs = reinterpret_cast<double*>(hb1);     // z staged in shared memory (hb1 is free until layer 0 writes it)
  double zacc = t < a.h1 ? (double)__ldg(a.b[0] + t) : 0.0;
  for (int k0 = 0; k0 < a.d_z; k0 += 32) {
    const int nk = min(32, a.d_z - k0);
    double pv[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) pv[u] = (t < a.h1 && u < nk) ? __ldg(a.Pz + (int64_t)t * a.d_z + k0 + u) : 0.0;
    if (k0 > 0) __syncthreads();
    if (t < nk) zs[t] = __ldg(a.z + k0 + t);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 32; ++u)
      if (u < nk) zacc += pv[u] * zs[u];
  }
  if (t < a.h1) zb[t] = (float)zacc;               // fp64 sum, rounded once
  for (int i = t; i < a.r_m * RB; i += SM_THREADS) {
    const int r = i / a.r_m, k = i - r * a.r_m;
    hb0[k * RB + r] = r < nr ? __ldg(a.MR + (r0 + r) * a.r_m + k) : 0.0f;
  }
  __syncthreads();
  sm_stamp(a, 1, c0);

  // ---- forward
  float* x = hb0;
  float* y = hb1;
  for (int l = 0; l < L; ++l) {
    const int K = a.w[l], N = a.w[l + 1];
    float acc[RB];
    const float bias = t < N ? (l == 0 ? zb[t] : __ldg(a.b[l] + t)) : 0.0f;
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = bias;
    small_dot<RB>(a, ring, x, K, N, t, t < N, acc);
    if (t < N) {
      if (l < NH) {
        float* D = Ds + ((size_t)l * SM_MAXW + t) * RB;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          float av, dv;
          act_eval(a.act, acc[r], av, dv);
          y[t * RB + r] = (a.res[l] ? x[t * RB + r] : 0.0f) + av;
          D[r] = dv;
        }
      } else {                                     // phi = mu + sigma (W h + b)
        const float mu = __ldg(a.omean + t), sg = __ldg(a.ostd + t);
#pragma unroll
        for (int r = 0; r < RB; ++r) y[t * RB + r] = fmaf(sg, acc[r], mu);
      }
    }
    __syncthreads();
    float* tmp = x; x = y; y = tmp;
  }

  // ---- Q (fp64; warp r reduces row r) and the unit seeds e = 2 sigma (phi + c)
  sm_stamp(a, 2, c0);
  const float* phi = x;
  if (warp < RB) {
    double s = 0.0;
    for (int j = lane; j < a.r_u; j += 32) {
      const double p = phi[j * RB + warp];
      s += p * (p + 2.0 * (double)__ldg(a.c + j));
    }
    s = warp_sum(s);
    const double q = s + a.q0;
    if (lane == 0) {
      const bool ok = warp < nr;
      if (ok) a.Q[r0 + warp] = q;
      const double qs = ok ? q - a.shift : 0.0;
      sred[warp][0] = ok ? 1.0 : 0.0;
      sred[warp][1] = qs;
      sred[warp][2] = qs * qs;
      sred[warp][3] = qs;                          // the row's (Q - shift): the A2 weights below
    }
  }
  float* g = y;
  if (t < a.r_u) {
    const float sg2 = 2.0f * __ldg(a.ostd + t), cc = __ldg(a.c + t);
#pragma unroll
    for (int r = 0; r < RB; ++r) g[t * RB + r] = r < nr ? sg2 * (phi[t * RB + r] + cc) : 0.0f;
  }
  __syncthreads();
  float* gin = g;                                  // current gradient (k-major over its features)
  float* gout = const_cast<float*>(phi);           // (phi is dead once the seeds exist)

  // ---- reverse sweep: g <- (res ? g : 0) + (D_l g) W_l, down to u0 = D_0 g
  sm_stamp(a, 3, c0);
  for (int l = L - 1; l >= 1; --l) {
    const int K = a.w[l], N = a.w[l + 1];          // W_l: N x K; gradient in: N features, out: K features
    const bool hidden = l < L - 1, resid = hidden && a.res[l];
    float rterm[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) rterm[r] = 0.0f;
    if (hidden) {                                  // u = D_l g in place; the residual term stays in registers
      if (t < N) {
        const float* D = Ds + ((size_t)l * SM_MAXW + t) * RB;
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const float gv = gin[t * RB + r];
          if (resid) rterm[r] = gv;                // (N == K: thread t owns feature t on both sides)
          gin[t * RB + r] = D[r] * gv;
        }
      }
      __syncthreads();
    }
    small_dot<RB>(a, ring, gin, N, K, t, t < K, rterm);
    if (t < K) {
#pragma unroll
      for (int r = 0; r < RB; ++r) gout[t * RB + r] = rterm[r];
    }
    __syncthreads();
    float* tmp = gin; gin = gout; gout = tmp;
  }
  // u0 = D_0 g (L == 1: the seeds themselves, w[1] = r_u) and the CTA's fp64 partials
  sm_stamp(a, 4, c0);
  {
    const int N = a.w[1];
    double* part = a.part + (size_t)blockIdx.x * (2 * a.h1 + 4);
    if (t < N) {
      const float* D = Ds + (size_t)t * RB;
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double u = (double)(NH > 0 ? D[r] * gin[t * RB + r] : gin[t * RB + r]);
        a1 += u;
        a2 += sred[r][3] * u;
      }
      part[t] = a1;
      part[a.h1 + t] = a2;
    }
    if (t < 4) {
      double s = 0.0;
      if (t < 3)
        for (int r = 0; r < RB; ++r) s += sred[r][t];
      part[2 * a.h1 + t] = s;
    }
  }

  // ---- the last CTA combines (fixed CTA order), projects and exports
  sm_stamp(a, 5, c0);
  __syncthreads();
  if (t == 0) {
    __threadfence();
    s_last = atomicAdd(a.counter, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  sm_stamp(a, 6, true);
  double* A1 = reinterpret_cast<double*>(hb0);     // h1, then A2 (h1), then per-risk V (h1): reuse the buffers
  double* A2 = A1 + a.h1;
  double* V = A2 + a.h1;
  double* st = V + a.h1;                           // 3 moments
  const int pw = 2 * a.h1 + 4;
  // column pairs (16-byte loads; pw is even), 16 loads in flight, added in CTA order
  for (int c = 2 * t; c < 2 * a.h1 + 4; c += 2 * SM_THREADS) {
    double s0 = 0.0, s1 = 0.0;
    unsigned b = 0;
    for (; b + 16 <= gridDim.x; b += 16) {
      double2 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(reinterpret_cast<const double2*>(a.part + (size_t)(b + u) * pw + c));
#pragma unroll
      for (int u = 0; u < 16; ++u) { s0 += v[u].x; s1 += v[u].y; }
    }
    for (; b < gridDim.x; ++b) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(a.part + (size_t)b * pw + c));
      s0 += v.x; s1 += v.y;
    }
    if (c < 2 * a.h1) { A1[c] = s0; A1[c + 1] = s1; }      // (A2 follows A1; h1 is even)
    else { st[c - 2 * a.h1] = s0; st[c + 1 - 2 * a.h1] = s1; }
  }
  __syncthreads();
  sm_stamp(a, 7, true);
  const double n = st[0], m1 = st[1] / n;
  if (t < STATS_LEN) {
    const double v = t < 3 ? st[t] : (t == 5 ? n : 0.0);
    a.stats[t] = v;
    a.hstats[t] = v;
  }
  for (int r = 0; r < a.R; ++r) {
    const bool mv = a.kind[r] == RISK_MEANVAR;
    const double c1 = (mv ? 1.0 - 2.0 * a.beta[r] * m1 : 1.0) / n, c2 = mv ? 2.0 * a.beta[r] / n : 0.0;
    for (int c = t; c < a.h1; c += SM_THREADS) V[c] = c1 * A1[c] + c2 * A2[c];
    __syncthreads();
    // out_r[k] = PzT[k] . V: thread (k = t / 8, slice j = t % 8) sums its eighth
    // of the columns with the loads in flight together, the eight slices of a
    // control are added in slice order by a fixed shuffle tree
    for (int k0 = 0; k0 < a.d_z; k0 += SM_THREADS / 8) {
      const int k = k0 + (t >> 3), j = t & 7;
      const int per = (a.h1 + 7) / 8, c0 = j * per, c1e = min(a.h1, c0 + per);
      double s = 0.0;
      if (k < a.d_z) {
        const double* prow = a.PzT + (int64_t)k * a.h1;
        int c = c0;
        for (; c + 8 <= c1e; c += 8) {
          double pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = __ldg(prow + c + u);
#pragma unroll
          for (int u = 0; u < 8; ++u) s += pv[u] * V[c + u];
        }
        for (; c < c1e; ++c) s += __ldg(prow + c) * V[c];
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (j == 0 && k < a.d_z) {
        a.out[(size_t)r * a.plen + k] = s;
        a.hpart[(size_t)r * a.plen + k] = s;
      }
    }
    if (t == 0) {                                  // value partials of a dense risk: sum Q, count
      const double sq = a.shift * n + st[1];
      a.out[(size_t)r * a.plen + a.d_z] = sq;
      a.out[(size_t)r * a.plen + a.d_z + 1] = n;
      a.hpart[(size_t)r * a.plen + a.d_z] = sq;
      a.hpart[(size_t)r * a.plen + a.d_z + 1] = n;
    }
    __syncthreads();
  }
  for (int i = t; i < a.nband; i += SM_THREADS) a.hband[i] = 0;
  if (t == 0) *a.counter = 0;
  sm_stamp(a, 8, true);
}

// dynamic shared memory of k_small_eval<RB> for a network with n_hidden hidden layers
inline size_t small_smem_bytes(int RB, int n_hidden) {
  return sizeof(float) * ((size_t)SM_STAGES * SM_CH * SM_MAXW + (size_t)(2 + n_hidden) * SM_MAXW * RB + SM_MAXW);
}

}  // namespace sdn
