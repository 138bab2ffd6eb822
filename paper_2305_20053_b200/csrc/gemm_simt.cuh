// gemm_simt.cuh -- fp32 FFMA tiled GEMM with fused epilogues.
//
// C[M x N] = opA(A) * opB(B), fp32 accumulate, epilogue applied per float4
// of output columns.  A is M x K row-major (or K x M when AT); B is N x K
// row-major when BT (C = A B^T, torch-Linear forward) else K x N row-major
// (C = A B, the backward sweep).  VEC = 16-byte vector loads (needs K, lda,
// ldb multiples of 4 and aligned bases); otherwise scalar loads.
//
// This is the exact-fp32 path (used for small latency-bound shapes and as
// the SDN_GEMM_SIMT back end); large shapes go through the tcgen05 kernel
// in gemm_tc.cuh with the same epilogue functors.
#pragma once
#include "common.cuh"

namespace sdn {

// output widths that are not a multiple of 4 (d_u, d_z): the last float4
// group is written column by column through Epi::col
template <class Epi>
SDN_DEV void epi_tail(const Epi& epi, int64_t r, int c, int nv, float a, float b, float d) {
  float v[3] = {a, b, d};
  for (int j = 0; j < nv; ++j) epi.col(r, c + j, v[j]);
}

template <int BM, int BN, int BK, int TM, int TN, bool AT, bool BT, bool VEC, class Epi>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
gemm_simt_kernel(int64_t M, const int* __restrict__ Mdev, int N, int K, const float* __restrict__ A,
                 int64_t lda, const float* __restrict__ B, int64_t ldb, Epi epi) {
  constexpr int NTX = BN / TN;
  constexpr int NT = (BM / TM) * NTX;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];

  if (Mdev) M = min(M, (int64_t)*Mdev);   // compacted sweeps: device row count
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  if (m0 >= M) return;
  const int tid = threadIdx.x;
  const int tx = tid % NTX, ty = tid / NTX;
  const int n0 = blockIdx.y * BN;

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  // split-K over gridDim.z (default 1): this block's K range [kb, K) in
  // BK-aligned slices; the epilogue writes one partial per z (EpiStoreZ)
  int kb = 0;
  if (gridDim.z > 1) {
    const int kz = ((K + (int)gridDim.z - 1) / (int)gridDim.z + BK - 1) / BK * BK;
    kb = (int)blockIdx.z * kz;
    K = min(K, kb + kz);
  }
  for (int k0 = kb; k0 < K; k0 += BK) {
    // ---- A tile -> As[k][m]
    if (!AT) {
      if (VEC) {
        for (int e = tid; e < BM * BK / 4; e += NT) {
          int row = e / (BK / 4), kq = (e % (BK / 4)) * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (m0 + row < M && k0 + kq < K)
            v = *reinterpret_cast<const float4*>(A + (m0 + row) * lda + k0 + kq);
          As[kq + 0][row] = v.x; As[kq + 1][row] = v.y;
          As[kq + 2][row] = v.z; As[kq + 3][row] = v.w;
        }
      } else {
        for (int e = tid; e < BM * BK; e += NT) {
          int row = e / BK, kk = e % BK;
          As[kk][row] = (m0 + row < M && k0 + kk < K) ? A[(m0 + row) * lda + k0 + kk] : 0.0f;
        }
      }
    } else {  // A stored K x M
      for (int e = tid; e < BM * BK; e += NT) {
        int kk = e / BM, row = e % BM;
        As[kk][row] = (m0 + row < M && k0 + kk < K) ? A[(int64_t)(k0 + kk) * lda + m0 + row] : 0.0f;
      }
    }
    // ---- B tile -> Bs[k][n]
    if (BT) {
      if (VEC) {
        for (int e = tid; e < BN * BK / 4; e += NT) {
          int col = e / (BK / 4), kq = (e % (BK / 4)) * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (n0 + col < N && k0 + kq < K)
            v = *reinterpret_cast<const float4*>(B + (int64_t)(n0 + col) * ldb + k0 + kq);
          Bs[kq + 0][col] = v.x; Bs[kq + 1][col] = v.y;
          Bs[kq + 2][col] = v.z; Bs[kq + 3][col] = v.w;
        }
      } else {
        for (int e = tid; e < BN * BK; e += NT) {
          int col = e / BK, kk = e % BK;
          Bs[kk][col] = (n0 + col < N && k0 + kk < K) ? B[(int64_t)(n0 + col) * ldb + k0 + kk] : 0.0f;
        }
      }
    } else {
      if (VEC) {
        for (int e = tid; e < BN * BK / 4; e += NT) {
          int kk = e / (BN / 4), nq = (e % (BN / 4)) * 4;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (k0 + kk < K && n0 + nq < N)
            v = *reinterpret_cast<const float4*>(B + (int64_t)(k0 + kk) * ldb + n0 + nq);
          *reinterpret_cast<float4*>(&Bs[kk][nq]) = v;
        }
      } else {
        for (int e = tid; e < BN * BK; e += NT) {
          int kk = e / BN, col = e % BN;
          Bs[kk][col] = (k0 + kk < K && n0 + col < N) ? B[(int64_t)(k0 + kk) * ldb + n0 + col] : 0.0f;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        float4 v = *reinterpret_cast<const float4*>(&As[kk][ty * TM + i]);
        a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[kk][tx * TN + j]);
        b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    int64_t r = m0 + ty * TM + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; j += 4) {
      int c = n0 + tx * TN + j;
      if (c + 4 <= N) epi(r, c, make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]));
      else if (c < N) epi_tail(epi, r, c, N - c, acc[i][j], acc[i][j + 1], acc[i][j + 2]);
    }
  }
}

// ---------------------------------------------------------------------------
// epilogues.  N (output width) is a multiple of 4 for every caller; a float4
// of columns [c, c+4) is always fully in range.

// plain store C[r, c] = acc
struct EpiStore {
  float* C; int64_t ldc;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float* p = C + r * ldc + c;
    if ((ldc & 3) == 0) *reinterpret_cast<float4*>(p) = v;
    else { p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w; }
  }
  SDN_DEV void col(int64_t r, int c, float v) const { C[r * ldc + c] = v; }
};

// split-K partial store: C + blockIdx.z * zstride (reduced by k_sum_z)
struct EpiStoreZ {
  float* C; int64_t ldc; int64_t zstride;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float* p = C + blockIdx.z * zstride + r * ldc + c;
    if ((ldc & 3) == 0) *reinterpret_cast<float4*>(p) = v;
    else { p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w; }
  }
  SDN_DEV void col(int64_t r, int c, float v) const { C[blockIdx.z * zstride + r * ldc + c] = v; }
};

// fp64 accumulate (split-K setup GEMMs): C64[r, c] += acc
struct EpiAccum64 {
  double* C; int64_t ldc;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    double* p = C + r * ldc + c;
    p[0] += v.x; p[1] += v.y; p[2] += v.z; p[3] += v.w;
  }
  SDN_DEV void col(int64_t r, int c, float v) const { C[r * ldc + c] += v; }
};

// C = acc + bias with a column bound (GEMMs whose N is padded past the real
// width, e.g. the decoder operand's rows padded to 16): columns >= nvalid dropped
struct EpiAffineN {
  const float* bias; float* C; int64_t ldc; int64_t nvalid;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c + j < nvalid) C[r * ldc + c + j] = x[j] + (bias ? bias[c + j] : 0.0f);
  }
  SDN_DEV void col(int64_t r, int c, float v) const {
    if (c < nvalid) C[r * ldc + c] = v + (bias ? bias[c] : 0.0f);
  }
};

// store with bias add and an optional per-column scale/shift:
// C = shift + scale * (acc + bias)   (scale/shift may be null)
struct EpiAffine {
  const float* bias; const float* scale; const float* shift; float* C; int64_t ldc;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y = x[j] + (bias ? bias[c + j] : 0.0f);
      if (scale) y *= scale[c + j];
      if (shift) y += shift[c + j];
      x[j] = y;
    }
    float* p = C + r * ldc + c;
    if ((ldc & 3) == 0) *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
    else { p[0] = x[0]; p[1] = x[1]; p[2] = x[2]; p[3] = x[3]; }
  }
  SDN_DEV void col(int64_t r, int c, float v) const {
    float y = v + (bias ? bias[c] : 0.0f);
    if (scale) y *= scale[c];
    if (shift) y += shift[c];
    C[r * ldc + c] = y;
  }
};

// hidden-layer forward: s = acc + bias; H = [prev +] act(s); D = act'(s)
// (reference surrogate.py:171-181; residual gap).  D may be null (value-only).
struct EpiFwdHidden {
  const float* bias; const float* prev; float* H; float* D; int64_t ld; int act;
  // returns the value that feeds the next GEMM (H)
  SDN_DEV float4 apply(int64_t r, int c, float4 v) const {
    float s[4] = {v.x, v.y, v.z, v.w}, a[4], d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) act_eval(act, s[j] + bias[c + j], a[j], d[j]);
    if (prev) {
      float4 p = *reinterpret_cast<const float4*>(prev + r * ld + c);
      a[0] += p.x; a[1] += p.y; a[2] += p.z; a[3] += p.w;
    }
    float4 h = make_float4(a[0], a[1], a[2], a[3]);
    if (H) *reinterpret_cast<float4*>(H + r * ld + c) = h;
    if (D) *reinterpret_cast<float4*>(D + r * ld + c) = make_float4(d[0], d[1], d[2], d[3]);
    return h;
  }
  SDN_DEV void operator()(int64_t r, int c, float4 v) const { (void)apply(r, c, v); }
  SDN_DEV void col(int64_t, int, float) const {}   // widths are multiples of 4 (sdn_create)
};

// backward step: g = acc [+ resid]; U = D[row] * g; G = g (optional).
// rowidx maps compacted rows to sample rows of D (null = identity);
// rowdiv > 1 maps tangent rows (i*d_z + k) to sample i (forward mode).
struct EpiBwd {
  const float* resid; float* G; const float* D; int64_t ldD; const int* rowidx;
  float* U; int64_t ld;
  // returns the value that feeds the next GEMM (U)
  SDN_DEV float4 apply(int64_t r, int c, float4 v) const {
    float g[4] = {v.x, v.y, v.z, v.w};
    if (resid) {
      float4 p = *reinterpret_cast<const float4*>(resid + r * ld + c);
      g[0] += p.x; g[1] += p.y; g[2] += p.z; g[3] += p.w;
    }
    if (G) *reinterpret_cast<float4*>(G + r * ld + c) = make_float4(g[0], g[1], g[2], g[3]);
    int64_t rd = rowidx ? (int64_t)rowidx[r] : r;
    // D null: the derivative is applied after the GEMM (softmax: a (g - a.g))
    float4 d = D ? *reinterpret_cast<const float4*>(D + rd * ldD + c) : make_float4(1.f, 1.f, 1.f, 1.f);
    float4 u = make_float4(d.x * g[0], d.y * g[1], d.z * g[2], d.w * g[3]);
    if (U) *reinterpret_cast<float4*>(U + r * ld + c) = u;
    return u;
  }
  SDN_DEV void operator()(int64_t r, int c, float4 v) const { (void)apply(r, c, v); }
  SDN_DEV void col(int64_t, int, float) const {}   // widths are multiples of 4 (sdn_create)
};

// forward-mode tangent step (surrogate.py:208-223 with residual):
// T_out = D[row / d_z] * acc [+ T_in]
struct EpiTangent {
  const float* D; int64_t ldD; int rowdiv; const float* tin; float* tout; int64_t ld;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float4 d = D ? *reinterpret_cast<const float4*>(D + (r / rowdiv) * ldD + c) : make_float4(1.f, 1.f, 1.f, 1.f);
    float4 o = make_float4(d.x * v.x, d.y * v.y, d.z * v.z, d.w * v.w);
    if (tin) {
      float4 p = *reinterpret_cast<const float4*>(tin + r * ld + c);
      o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
    }
    *reinterpret_cast<float4*>(tout + r * ld + c) = o;
  }
  SDN_DEV void col(int64_t, int, float) const {}   // widths are multiples of 4 (sdn_create)
};

// Jacobian scatter: tangent row (i*d_z + k), column u -> J[i, u, k] * scale[u]
// (surrogate.py:232-233: out_std * T^T).  ncol = r_u (or d_u when decoding).
// (nvalid: columns past it are GEMM padding and not written; 0 = ncol)
struct EpiJacScatter {
  const float* scale; float* J; int d_z; int64_t ncol; int64_t nvalid = 0;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    int64_t i = r / d_z; int k = (int)(r % d_z);
    float x[4] = {v.x, v.y, v.z, v.w};
    float* base = J + i * ncol * d_z + k;
    const int64_t nv = nvalid ? nvalid : ncol;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c + j < nv) base[(int64_t)(c + j) * d_z] = scale ? x[j] * scale[c + j] : x[j];
  }
  SDN_DEV void col(int64_t r, int c, float v) const {
    int64_t i = r / d_z; int k = (int)(r % d_z);
    if (c < (nvalid ? nvalid : ncol)) J[i * ncol * d_z + (int64_t)c * d_z + k] = scale ? v * scale[c] : v;
  }
};

}  // namespace sdn
