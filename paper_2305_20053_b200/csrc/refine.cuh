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
constexpr int REF_KC = 1024;          // layer input width per K chunk (wider layers run in chunks)
constexpr int REF_THREADS = 256;
constexpr int REF_MAX_LAYERS = 16;
constexpr int REF_RESELECT_SMALL = 256;   // band rows up to which one block ranks them O(m^2)

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
  const double* tp;             // device-side t of the window (graph replay), else t
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
  // phase 0 (k > 0): the exact top-k selection itself (value desc, index
  // asc) over Q -> mask and the threshold (written to *tdev), cooperative
  int64_t k;
  unsigned* ghist;              // 2 x gridDim.x x 256 scratch
  unsigned long long* gmm;      // 2 x gridDim.x scratch (min / max keys)
  int refine;                   // 0: selection only
  int softmax;                  // hidden layers are per-row softmax (a row pass after each layer)
  unsigned long long* trace;    // optional phase timestamps (block 0, %globaltimer)
};

SDN_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define REF_STAMP(slot) do { if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[(slot)] = gtime(); } while (0)

// Data written inside this kernel by other blocks (rowidx, the layer
// ping-pong, Q) is read with ld.global.cg (L2): L1 is not coherent across SMs.

SDN_DEV int warp_sum_i(int v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// grid-wide barrier (all blocks co-resident: cooperative launch)
// (release on arrival, acquire on the generation flag: orders this block's
// prior writes before the release and everyone's after the acquire, without
// two full fences per block)
SDN_DEV void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned arrived;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    if (arrived == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1u) : "memory");
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      } while (g == gen);
    }
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

// one W row slice into registers: unconditional loads at clamped addresses so
// all are in flight at once (a branch per load would serialise the round trips)
// (KC: the layer's input width rounded up to 128/256/512/1024 -- no loads or
// registers for columns past it)
template <int KC>
SDN_DEV void ref_load_w(const float* w, int K, int lane, float (&wf)[KC / 32]) {
#pragma unroll
  for (int u = 0; u < KC / 32; ++u) wf[u] = __ldg(w + min(lane + 32 * u, K - 1));
}

// dot products of RB staged rows with one W row; transposed butterfly so that
// lanes 4j..4j+3 end with row j's total (9 double shuffles instead of 8 x 5)
template <int RB, int KC>
SDN_DEV double ref_column(const double* xs, const float (&wf)[KC / 32], int K, int lane) {
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
  for (int u = 0; u < KC / 32; ++u) {
    if (lane + 32 * u < K) {
      const double wk = (double)wf[u];
#pragma unroll
      for (int j = 0; j < RB; ++j) acc[j] = fma(xs[j * REF_KC + lane + 32 * u], wk, acc[j]);
    }
  }
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double b[4], c2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = h16 ? acc[i] : acc[i + 4], keep = h16 ? acc[i + 4] : acc[i];
    b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = h8 ? b[i] : b[i + 2], keep = h8 ? b[i + 2] : b[i];
    c2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double d = (h4 ? c2[1] : c2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? c2[0] : c2[1], 4);
  d += __shfl_xor_sync(0xffffffffu, d, 2);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  return d;                                      // total of row (lane >> 2)
}

// one pass of up to REF_RB band rows through layer ly (stage the rows in
// shared memory, then this warp's output columns)
// Layers wider than REF_KC run in K chunks [k0, k0 + Kc): each chunk's
// partial dot products are accumulated in `out` (fp64; the same lane owns the
// same (row, column) entry in every chunk), the epilogue runs on the last.
// ridx: the band rows of the current row chunk (ordered compaction).
template <int KC>
SDN_DEV void ref_rows(const RefineArgs& a, const RefineLayer& ly, double* xs, int warp, int lane, int gw, int nw,
                      const int* ridx, int r0, int rb, bool first, bool last, const double* in64, double* out,
                      int k0 = 0, int Kc = -1) {
  const int K = ly.K, N = ly.N;
  if (Kc < 0) Kc = K;
  const bool kfirst = k0 == 0, klast = k0 + Kc >= K;
  {                                          // warp j stages row r0 + j (clamped)
    const int rj = r0 + min(warp, rb - 1);
    if (first) {                              // x = m_r * in_scale (exact in fp64, as the oracle)
      const float* src = a.MR + (int64_t)__ldcg(ridx + rj) * K + k0;
      float v[KC / 32], sc[KC / 32];
#pragma unroll
      for (int u = 0; u < KC / 32; ++u) {
        v[u] = __ldg(src + min(lane + 32 * u, Kc - 1));
        sc[u] = __ldg(a.iscale + k0 + min(lane + 32 * u, Kc - 1));
      }
#pragma unroll
      for (int u = 0; u < KC / 32; ++u)
        if (lane + 32 * u < Kc) xs[warp * REF_KC + lane + 32 * u] = (double)v[u] * (double)sc[u];
    } else {
      const double* src = in64 + (int64_t)rj * K + k0;
      double v[KC / 32];
#pragma unroll
      for (int u = 0; u < KC / 32; ++u) v[u] = __ldcg(src + min(lane + 32 * u, Kc - 1));
#pragma unroll
      for (int u = 0; u < KC / 32; ++u)
        if (lane + 32 * u < Kc) xs[warp * REF_KC + lane + 32 * u] = v[u];
    }
  }
  __syncthreads();
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && r0 == 0) a.trace[first ? 30 : (last ? 31 : 32)] = gtime();
  // columns of this warp: c = gw, gw + nw, ...; the next column's W row is
  // loaded while the current one is reduced (software pipeline).  The fp64
  // epilogues (bias, activation with its exp, residual, store) of up to four
  // columns run together: after the butterfly the four lanes 4j..4j+3 all hold
  // row j's total, so lane 4j + i finishes column i instead of lane 4j doing
  // four activations one after another.
  float wf[KC / 32];
  int c = gw;
  if (c < N) ref_load_w<KC>(ly.W + (int64_t)c * K + k0, Kc, lane, wf);
  double vq[4] = {0.0, 0.0, 0.0, 0.0};
  int cq0 = gw, nq = 0;                       // queued columns: cq0 + i nw, i < nq
  for (; c < N; c += nw) {
    float wn[KC / 32];
    if (c + nw < N) ref_load_w<KC>(ly.W + (int64_t)(c + nw) * K + k0, Kc, lane, wn);
    double v;
    if (rb <= 2) v = ref_column<2, KC>(xs, wf, Kc, lane);
    else if (rb <= 4) v = ref_column<4, KC>(xs, wf, Kc, lane);
    else v = ref_column<8, KC>(xs, wf, Kc, lane);
    if (nq == 0) cq0 = c;
    if (nq == 0) vq[0] = v; else if (nq == 1) vq[1] = v; else if (nq == 2) vq[2] = v; else vq[3] = v;
    ++nq;
    if (nq == 4 || c + nw >= N) {
      const int i = lane & 3, j = lane >> 2;   // this lane's queued column and row
      const int ci = cq0 + i * nw;
      double vi = i == 0 ? vq[0] : i == 1 ? vq[1] : i == 2 ? vq[2] : vq[3];
      if (i < nq && j < rb) {
        double* dst = out + (int64_t)(r0 + j) * N + ci;
        if (!kfirst) vi += *dst;                 // earlier K chunks (written by this lane)
        if (!klast) {
          *dst = vi;
        } else {
          const double S = vi + (first ? a.zb64[ci] : (double)ly.b[ci]);
          double o;
          if (last) {
            o = (double)a.omean[ci] + (double)a.ostd[ci] * S;
          } else if (a.softmax) {
            o = S;                                        // normalised by the row pass below
          } else {
            o = act64(a.act, S);
            if (ly.resid)                                 // resid: K == N
              o += (kfirst && ci < Kc) ? xs[j * REF_KC + ci] : __ldcg(in64 + (int64_t)(r0 + j) * K + ci);
          }
          *dst = o;
        }
      }
      nq = 0;
    }
#pragma unroll
    for (int u = 0; u < KC / 32; ++u) wf[u] = wn[u];
  }
  __syncthreads();
}

struct RefShared {
  int w[REF_THREADS / 32], m[REF_THREADS / 32];
  unsigned gen;
  int need;
  unsigned hist[256];
  unsigned long long prefix;
  long long krem;
  unsigned long long mm[2][REF_THREADS / 32];
};

// Cooperative exact top-k over n items (value desc, position asc): MSD radix
// select on order-preserving keys, from the first byte in which the keys
// differ; per-block 256-bin histograms summed by every block (identical
// decisions), ties taken in position order via per-block counts of
// threshold-equal keys.  key(i) -> dkey, set(i, selected).  Returns the
// threshold value (the k-th largest), also written to *thr_out if given.
// With trailing = false the caller must barrier before reusing blockcnt.
// grid scratch of the cooperative select (a few pointers: passing the whole
// RefineArgs by reference to a non-inlined function would copy it to the stack)
struct SelScratch {
  unsigned* bar;
  unsigned* ghist;
  unsigned long long* gmm;
  int* blockcnt;
  unsigned long long* trace;
};

template <class KeyF, class SetF>
__device__ __noinline__ double coop_select(SelScratch a, RefShared& S, unsigned& gen, int64_t n, int64_t k, KeyF key,
                                           SetF set, double* thr_out, bool trailing) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x;
  const int64_t per = (n + G - 1) / G;            // contiguous slice per block (position order)
  const int64_t lo = min((int64_t)blockIdx.x * per, n), hi = min(lo + per, n);
  unsigned long long kmin = ~0ull, kmax = 0ull;
  for (int64_t i = lo + tid; i < hi; i += REF_THREADS) {
    const unsigned long long kk = key(i);
    kmin = min(kmin, kk);
    kmax = max(kmax, kk);
  }
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) { S.mm[0][warp] = kmin; S.mm[1][warp] = kmax; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < REF_THREADS / 32; ++w) { kmin = min(kmin, S.mm[0][w]); kmax = max(kmax, S.mm[1][w]); }
    a.gmm[blockIdx.x] = kmin;
    a.gmm[G + blockIdx.x] = kmax;
  }
  grid_barrier(a.bar, gen);
  REF_STAMP(1);
  {                                                // parallel loads, warp reductions
    unsigned long long x = ~0ull, y = 0ull;
    for (unsigned b = tid; b < G; b += REF_THREADS) { x = min(x, __ldcg(a.gmm + b)); y = max(y, __ldcg(a.gmm + G + b)); }
    for (int o = 16; o > 0; o >>= 1) {
      x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
      y = max(y, __shfl_xor_sync(0xffffffffu, y, o));
    }
    __syncthreads();
    if (lane == 0) { S.mm[0][warp] = x; S.mm[1][warp] = y; }
    __syncthreads();
  }
  if (tid == 0) {
    unsigned long long x = S.mm[0][0], y = S.mm[1][0];
    for (int w = 1; w < REF_THREADS / 32; ++w) { x = min(x, S.mm[0][w]); y = max(y, S.mm[1][w]); }
    const int cp = (x == y) ? 8 : __clzll((long long)(x ^ y)) / 8;
    S.w[0] = cp;
    S.prefix = (cp == 0) ? 0ull : (cp >= 8 ? x : (x & (~0ull << (64 - 8 * cp))));
    S.krem = k;
  }
  __syncthreads();
  const int first = S.w[0];
  unsigned long long himask = (first == 0) ? 0ull : (first >= 8 ? ~0ull : (~0ull << (64 - 8 * first)));
  bool early = false;
  unsigned long long tmin = 0ull;
  if (tid == 0) S.need = 0;
  __syncthreads();
  for (int pass = first; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    const unsigned long long prefix = S.prefix;
    for (int d = tid; d < 256; d += REF_THREADS) S.hist[d] = 0;
    __syncthreads();
    for (int64_t i = lo + tid; i < hi; i += REF_THREADS) {
      const unsigned long long kk = key(i);
      if ((kk & himask) == prefix) atomicAdd(&S.hist[(unsigned)(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    unsigned* gh = a.ghist + (size_t)(pass & 1) * G * 256;
    for (int d = tid; d < 256; d += REF_THREADS) gh[blockIdx.x * 256 + d] = S.hist[d];
    grid_barrier(a.bar, gen);
    for (int d = tid; d < 256; d += REF_THREADS) {
      unsigned c = 0;
#pragma unroll 16
      for (unsigned b = 0; b < G; ++b) c += __ldcg(gh + b * 256 + d);   // unrolled: loads in flight
      S.hist[d] = c;
    }
    __syncthreads();
    if (warp == 0) {                               // lane l owns digits 255-8l .. 248-8l
      unsigned c[8], t8 = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { c[q] = S.hist[255 - 8 * lane - q]; t8 += c[q]; }
      unsigned incl = t8;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const long long krem = S.krem;
      const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl >= krem);
      const int L = hit ? __ffs(hit) - 1 : 31;
      if (lane == L) {
        long long cum = (long long)(incl - t8);
        int d = 255 - 8 * lane;
        for (int q = 0; q < 8; ++q) {
          d = 255 - 8 * lane - q;
          if (cum + (long long)c[q] >= krem || q == 7) break;
          cum += c[q];
        }
        S.krem = krem - cum;
        S.prefix = prefix | ((unsigned long long)d << shift);
        S.need = (krem - cum == (long long)c[(255 - 8 * lane) - d]) ? 1 : 0;   // whole bucket taken
      }
    }
    himask |= (0xFFull << shift);
    __syncthreads();
    REF_STAMP(2 + pass);
    if (S.need && pass < 7) {
      // early exit: the k-th falls at the bottom of a bucket that is taken
      // whole, so the selection is {key >= Tlow}; the threshold value (the
      // band centre) is the smallest selected key
      const unsigned long long Tlow = S.prefix;
      unsigned long long mn = ~0ull;
      for (int64_t i = lo + tid; i < hi; i += REF_THREADS) {
        const unsigned long long kk = key(i);
        set(i, kk >= Tlow);
        if (kk >= Tlow) mn = min(mn, kk);
      }
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      __syncthreads();
      if (lane == 0) S.mm[0][warp] = mn;
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < REF_THREADS / 32; ++w) mn = min(mn, S.mm[0][w]);
        a.gmm[blockIdx.x] = mn;
      }
      grid_barrier(a.bar, gen);
      mn = ~0ull;
      for (unsigned b = tid; b < G; b += REF_THREADS) mn = min(mn, __ldcg(a.gmm + b));
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      __syncthreads();
      if (lane == 0) S.mm[0][warp] = mn;
      __syncthreads();
      for (int w = 0; w < REF_THREADS / 32; ++w) mn = min(mn, S.mm[0][w]);
      early = true;
      tmin = mn;
      break;
    }
  }
  double thr;
  if (early) {
    thr = dkey_inv(tmin);
    if (thr_out && blockIdx.x == 0 && tid == 0) *thr_out = thr;
    REF_STAMP(10);
    return thr;                                    // (blockcnt untouched on this path)
  }
  const unsigned long long T = S.prefix;
  const long long need = S.krem;                   // threshold-equal keys to take, lowest position first
  thr = dkey_inv(T);
  if (thr_out && blockIdx.x == 0 && tid == 0) *thr_out = thr;
  int eq = 0;
  for (int64_t i = lo + tid; i < hi; i += REF_THREADS) eq += (key(i) == T) ? 1 : 0;
  eq = warp_sum_i(eq);
  if (lane == 0) S.w[warp] = eq;
  __syncthreads();
  if (tid == 0) {
    int e = 0;
    for (int w = 0; w < REF_THREADS / 32; ++w) e += S.w[w];
    a.blockcnt[blockIdx.x] = e;
  }
  grid_barrier(a.bar, gen);
  long long run = 0;                               // threshold-equal keys in earlier blocks
  {
    int pr = 0;
    for (unsigned b = tid; b < blockIdx.x; b += REF_THREADS) pr += __ldcg(a.blockcnt + b);
    pr = warp_sum_i(pr);
    __syncthreads();
    if (lane == 0) S.w[warp] = pr;
    __syncthreads();
    for (int w = 0; w < REF_THREADS / 32; ++w) run += S.w[w];
    __syncthreads();
  }
  for (int64_t base = lo; base < hi; base += REF_THREADS) {
    const int64_t i = base + tid;
    const unsigned long long kk = i < hi ? key(i) : 0ull;
    const bool e = i < hi && kk == T;
    const unsigned bal = __ballot_sync(0xffffffffu, e);
    int t2;
    const int wb = block_excl(S.w, warp, lane, __popc(bal), t2);
    const long long rank = run + wb + __popc(bal & ((1u << lane) - 1u));
    if (i < hi) set(i, kk > T || (e && rank < need));
    run += t2;
  }
  REF_STAMP(10);
  if (trailing) grid_barrier(a.bar, gen);          // blockcnt is reused by the caller
  return thr;
}

__global__ void __launch_bounds__(REF_THREADS, 1) k_refine(RefineArgs a) {
  extern __shared__ double xs[];                  // REF_RB x REF_KC
  __shared__ RefShared S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x;
  REF_STAMP(0);
  if (tid == 0) S.gen = *(volatile unsigned*)&a.bar[1];
  __syncthreads();
  unsigned gen = S.gen;
  const int64_t per = (a.n + G - 1) / G;          // contiguous slice per block (index order)
  const int64_t lo = min((int64_t)blockIdx.x * per, a.n), hi = min(lo + per, a.n);
  const int gw = blockIdx.x * (REF_THREADS / 32) + warp, nw = G * (REF_THREADS / 32);
  const SelScratch sc{a.bar, a.ghist, a.gmm, a.blockcnt, a.trace};
  if (a.refine) {                                 // W rows of every layer -> L2 now (overlaps phases 0-1)
    for (int l = 0; l < a.L; ++l) {
      const RefineLayer& ly = a.layer[l];
      for (int c = gw; c < ly.N; c += nw) {
        const char* row = reinterpret_cast<const char*>(ly.W + (int64_t)c * ly.K);
        for (int o = lane * 128; o < ly.K * 4; o += 32 * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
      }
    }
  }

  // ---- 0. exact top-k (k > 0) over Q -> mask and the threshold (*tdev)
  double thr = 0.0;
  if (a.k > 0) {
    const double* Qp = a.Q;
    uint8_t* mk = a.mask;
    thr = coop_select(sc, S, gen, a.n, a.k, [&](int64_t i) { return (unsigned long long)dkey(Qp[i]); },
                      [&](int64_t i, bool v) { mk[i] = v ? 1 : 0; }, const_cast<double*>(a.tdev), a.refine != 0);
    if (!a.refine) return;
  }

  // ---- 1. band flags and ordered compaction
  const double tw = a.tp ? *a.tp : a.t;
  auto band = [&](int64_t i) -> bool {
    return a.kind == RISK_BAND_EXACT ? in_band_exact(a.Q[i], a.k > 0 ? thr : *a.tdev)
                                     : row_flag(a.kind, a.Q, nullptr, i, tw, a.eps, a.tdev);
  };
  int mine = 0;
  for (int64_t base = lo; base < hi; base += REF_THREADS) {
    const int64_t i = base + tid;
    const bool f = i < hi && band(i);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    mine += (lane == 0) ? __popc(b) : 0;
  }
  int tot;
  (void)block_excl(S.w, warp, lane, mine, tot);
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
    if (lane == 0) { S.w[warp] = po; S.m[warp] = pm; }
    __syncthreads();
    for (int w = 0; w < REF_THREADS / 32; ++w) { off += S.w[w]; m += S.m[w]; }
    __syncthreads();
  }
  for (int64_t base = lo; base < hi; base += REF_THREADS) {
    const int64_t i = base + tid;
    const bool f = i < hi && band(i);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    int t2;
    const int wb = block_excl(S.w, warp, lane, __popc(b), t2);
    if (f) a.rowidx[off + wb + __popc(b & ((1u << lane) - 1u))] = (int)i;
    off += t2;
  }
  if (blockIdx.x == 0 && tid == 0) *a.count = m;
  REF_STAMP(11);
  if (m == 0) return;                            // uniform: every block computed the same m
  grid_barrier(a.bar, gen);
  REF_STAMP(12);

  // ---- 2./3. fp64 chain + QoI over the m band rows, in row chunks of
  // cap_rows (the ping-pong buffers' size); layers wider than REF_KC in K chunks
  for (int c0 = 0; c0 < m; c0 += a.cap_rows) {
    const int mc = min(a.cap_rows, m - c0);
    const int* ridx = a.rowidx + c0;
    if (c0 > 0) grid_barrier(a.bar, gen);          // the previous chunk's QoI has read buf
    for (int l = 0; l < a.L; ++l) {
      const RefineLayer& ly = a.layer[l];
      const int K = ly.K, N = ly.N;
      const bool first = l == 0, last = l == a.L - 1;
      const double* in64 = first ? nullptr : a.buf[(l - 1) & 1];
      double* out = a.buf[l & 1];
      for (int r0 = 0; r0 < mc; r0 += REF_RB) {
        const int rb = min(REF_RB, mc - r0);
        if (K <= 128) ref_rows<128>(a, ly, xs, warp, lane, gw, nw, ridx, r0, rb, first, last, in64, out);
        else if (K <= 256) ref_rows<256>(a, ly, xs, warp, lane, gw, nw, ridx, r0, rb, first, last, in64, out);
        else if (K <= 512) ref_rows<512>(a, ly, xs, warp, lane, gw, nw, ridx, r0, rb, first, last, in64, out);
        else                                     // (one call site: K <= REF_KC is one chunk)
          for (int k0 = 0; k0 < K; k0 += REF_KC)
            ref_rows<REF_KC>(a, ly, xs, warp, lane, gw, nw, ridx, r0, rb, first, last, in64, out, k0,
                             min(REF_KC, K - k0));
      }
      REF_STAMP(13 + 2 * l);
      grid_barrier(a.bar, gen);
      REF_STAMP(14 + 2 * l);
      if (a.softmax && !last) {                    // per-row softmax (+ residual), one warp per row
        for (int r = gw; r < mc; r += nw) {
          double* o = out + (int64_t)r * N;
          double mx = -INFINITY;
          for (int c = lane; c < N; c += 32) mx = fmax(mx, __ldcg(o + c));
          for (int q = 16; q > 0; q >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, q));
          double sum = 0.0;
          for (int c = lane; c < N; c += 32) sum += exp(__ldcg(o + c) - mx);
          sum = warp_sum(sum);
          for (int c = lane; c < N; c += 32) {
            const double v = exp(__ldcg(o + c) - mx) / sum;
            o[c] = ly.resid ? __ldcg(in64 + (int64_t)r * K + c) + v : v;
          }
        }
        grid_barrier(a.bar, gen);
      }
    }
    // QoI of the chunk's rows -> Q (reduced: phi.(phi + 2c); decoded: phi.(K phi + 2c))
    const double* phi = a.buf[(a.L - 1) & 1];
    for (int r = gw; r < mc; r += nw) {
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
      if (lane == 0) a.Q[__ldcg(ridx + r)] = s + a.q0;
    }
  }
  REF_STAMP(40);
  if (!a.mask) return;
  grid_barrier(a.bar, gen);
  REF_STAMP(41);

  // ---- 4. exact CVaR: the band holds `need` selected rows (rows outside keep
  // their side of the threshold); take the top `need` band rows by
  // (refined Q desc, position asc -- positions are in index order).
  if (m > REF_RESELECT_SMALL) {                  // large band: cooperative radix select over the band
    int cnt = 0;
    for (int64_t r = (int64_t)blockIdx.x * REF_THREADS + tid; r < m; r += (int64_t)G * REF_THREADS)
      cnt += __ldcg(a.mask + __ldcg(a.rowidx + r)) ? 1 : 0;
    cnt = warp_sum_i(cnt);
    if (lane == 0) S.w[warp] = cnt;
    __syncthreads();
    if (tid == 0) {
      int e = 0;
      for (int w = 0; w < REF_THREADS / 32; ++w) e += S.w[w];
      a.blockcnt[blockIdx.x] = e;
    }
    grid_barrier(a.bar, gen);
    long long need = 0;
    {
      int pr = 0;
      for (unsigned b = tid; b < G; b += REF_THREADS) pr += __ldcg(a.blockcnt + b);
      pr = warp_sum_i(pr);
      __syncthreads();
      if (lane == 0) S.w[warp] = pr;
      __syncthreads();
      for (int w = 0; w < REF_THREADS / 32; ++w) need += S.w[w];
      __syncthreads();
    }
    grid_barrier(a.bar, gen);                      // blockcnt is reused by the select
    if (need == 0) {
      for (int64_t r = (int64_t)blockIdx.x * REF_THREADS + tid; r < m; r += (int64_t)G * REF_THREADS)
        a.mask[__ldcg(a.rowidx + r)] = 0;
    } else {
      const int* ri = a.rowidx;
      const double* Qp = a.Q;
      uint8_t* mk = a.mask;
      (void)coop_select(sc, S, gen, (int64_t)m, need,
                        [&](int64_t r) { return (unsigned long long)dkey(__ldcg(Qp + __ldcg(ri + r))); },
                        [&](int64_t r, bool v) { mk[__ldcg(ri + r)] = v ? 1 : 0; }, nullptr, false);
    }
    REF_STAMP(42);
    return;
  }
  // small band: one block ranks every band row against the others.  The band's
  // rows, keys and old mask bits are read into shared memory once (two global
  // round trips instead of two per pair of rows: this phase is on the c2
  // evaluation's critical path)
  if (blockIdx.x != 0) return;
  __shared__ unsigned long long s_key[REF_RESELECT_SMALL];
  __shared__ int s_row[REF_RESELECT_SMALL];
  if (tid == 0) S.need = 0;
  __syncthreads();
  int cnt = 0;
  for (int r = tid; r < m; r += REF_THREADS) {
    const int ri = __ldcg(a.rowidx + r);
    s_row[r] = ri;
    s_key[r] = (unsigned long long)dkey(__ldcg(a.Q + ri));
    cnt += __ldcg(a.mask + ri) ? 1 : 0;
  }
  atomicAdd(&S.need, cnt);
  __syncthreads();
  const int need = S.need;
  for (int r = tid; r < m; r += REF_THREADS) {
    const int ri = s_row[r];
    const unsigned long long ki = s_key[r];
    int rank = 0;
    for (int u = 0; u < m; ++u) {
      const unsigned long long kj = s_key[u];
      rank += (kj > ki || (kj == ki && s_row[u] < ri)) ? 1 : 0;
    }
    a.mask[ri] = rank < need ? 1 : 0;            // (ranks use the shared copies only: no ordering needed)
  }
  REF_STAMP(42);
}

}  // namespace sdn
