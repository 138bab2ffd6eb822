// train.cuh -- derivative-informed (H1) training step on the device
// (reference surrogate.py:263-405).
//
// One step over a batch of B records (indices into the device-resident
// dataset):
//   forward with tangents   S_l = A_l W_l^T + b_l, U_l = T_l W_l^T,
//                           A_{l+1} = f(S_l), T_{l+1} = f'(S_l) U_l (linear last layer)
//   loss                    (|A_L - Y|^2 + lambda |T_L - J^T/sigma|^2) / B   (output-scaled frame)
//   reverse (forward-over-reverse)
//                           GU = f' GT,  GS = f' GA + f'' sum_k U GT
//                           gW_l = GS^T A_l + GU^T T_l,  gb_l = sum_b GS
//                           GA = GS W_l,  GT = GU W_l
//   Adam                    (0.9, 0.999, 1e-8) on fp64 master parameters
// The GEMMs are the engine's SIMT fp32 kernels (gradients accumulated in
// fp64, fixed order); every elementwise / reduction stage is a kernel below.
#pragma once
#include "kernels.cuh"

namespace sdn {

SDN_DEV void act_d12(int act, double s, double& d1, double& d2) {
  switch (act) {
    case ACT_TANH: { const double t = tanh(s); d1 = 1.0 - t * t; d2 = -2.0 * t * d1; break; }
    case ACT_SOFTPLUS: { const double g = 0.5 * (1.0 + tanh(0.5 * s)); d1 = g; d2 = g * (1.0 - g); break; }
    case ACT_SIGMOID: {
      const double g = 0.5 * (1.0 + tanh(0.5 * s));
      d1 = g * (1.0 - g);
      d2 = d1 * (1.0 - 2.0 * g);
      break;
    }
    case ACT_ELU: { const double e = exp(fmin(s, 0.0)); d1 = s > 0.0 ? 1.0 : e; d2 = s > 0.0 ? 0.0 : e; break; }
    default: d1 = 1.0; d2 = 0.0;
  }
}

// batch gather: X = [m_r * s, z] (B x n0), Y = (u - mu) / sigma (B x r_u),
// Jt[b, k, :] = j[b, :, k] / sigma (B*d_z x r_u), T0[b, k, :] = e_{r_m + k}
__global__ void k_tr_gather(int B, const int* __restrict__ idx, const float* __restrict__ dm,
                            const float* __restrict__ dz, const float* __restrict__ du,
                            const float* __restrict__ dj, int r_m, int d_z, int r_u,
                            const float* __restrict__ in_scale, const float* __restrict__ mu,
                            const float* __restrict__ sig, float* __restrict__ X, float* __restrict__ Y,
                            float* __restrict__ Jt, float* __restrict__ T0) {
  const int b = blockIdx.x;
  if (b >= B) return;
  const int64_t i = idx[b];
  const int n0 = r_m + d_z;
  for (int c = threadIdx.x; c < n0; c += blockDim.x)
    X[(int64_t)b * n0 + c] = c < r_m ? (float)((double)dm[i * r_m + c] * (double)in_scale[c]) : dz[i * d_z + c - r_m];
  for (int c = threadIdx.x; c < r_u; c += blockDim.x)
    Y[(int64_t)b * r_u + c] = (float)(((double)du[i * r_u + c] - (double)mu[c]) / (double)sig[c]);
  if (T0) {
    for (int e = threadIdx.x; e < d_z * n0; e += blockDim.x) {
      const int k = e / n0, c = e - k * n0;
      T0[((int64_t)b * d_z + k) * n0 + c] = (c == r_m + k) ? 1.0f : 0.0f;
    }
  }
  if (Jt) {
    for (int e = threadIdx.x; e < d_z * r_u; e += blockDim.x) {
      const int k = e / r_u, c = e - k * r_u;
      Jt[((int64_t)b * d_z + k) * r_u + c] = (float)((double)dj[(i * r_u + c) * d_z + k] / (double)sig[c]);
    }
  }
}

// A_out = f(S), T_out[b, k, :] = f'(S[b]) U[b, k, :]   (hidden layers)
__global__ void k_tr_act(int B, int d_z, int n, int act, const float* __restrict__ S, const float* __restrict__ U,
                         float* __restrict__ A, float* __restrict__ T) {
  const int b = blockIdx.x;
  if (b >= B) return;
  for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < n; c += gridDim.y * blockDim.x) {
    float a, d;
    act_eval(act, S[(int64_t)b * n + c], a, d);
    A[(int64_t)b * n + c] = a;
    if (T)
      for (int k = 0; k < d_z; ++k) {
        const int64_t r = ((int64_t)b * d_z + k) * n + c;
        T[r] = d * U[r];
      }
  }
}

// loss terms and output seeds: GA = 2 (A - Y) / B, GT = 2 lambda (T - Jt) / B;
// per-block fp64 partials of |A - Y|^2 and |T - Jt|^2 (fixed order)
__global__ void __launch_bounds__(256)
k_tr_loss(int B, int d_z, int r_u, double lam, const float* __restrict__ A, const float* __restrict__ Y,
          const float* __restrict__ T, const float* __restrict__ Jt, float* __restrict__ GA, float* __restrict__ GT,
          double* __restrict__ part) {
  __shared__ double sp[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double e2 = 0.0, t2 = 0.0;
  const int64_t ne = (int64_t)B * r_u, nt = T ? (int64_t)B * d_z * r_u : 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)A[e] - (double)Y[e];
    e2 += d * d;
    GA[e] = (float)(2.0 * d / B);
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nt; e += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)T[e] - (double)Jt[e];
    t2 += d * d;
    GT[e] = (float)(2.0 * lam * d / B);
  }
  e2 = warp_sum(e2);
  t2 = warp_sum(t2);
  if (lane == 0) { sp[warp][0] = e2; sp[warp][1] = t2; }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sp[w][threadIdx.x];
    part[(int64_t)blockIdx.x * 2 + threadIdx.x] = s;
  }
}

// hidden-layer reverse step: GU = f' GT ; GS = f' GA + f'' sum_k U GT
__global__ void k_tr_bwd(int B, int d_z, int n, int act, const float* __restrict__ S, const float* __restrict__ U,
                         const float* __restrict__ GA, const float* __restrict__ GT, float* __restrict__ GS,
                         float* __restrict__ GU) {
  const int b = blockIdx.x;
  if (b >= B) return;
  for (int c = blockIdx.y * blockDim.x + threadIdx.x; c < n; c += gridDim.y * blockDim.x) {
    double d1, d2;
    act_d12(act, (double)S[(int64_t)b * n + c], d1, d2);
    double ut = 0.0;
    if (GT)
      for (int k = 0; k < d_z; ++k) {
        const int64_t r = ((int64_t)b * d_z + k) * n + c;
        ut += (double)U[r] * (double)GT[r];
        GU[r] = (float)(d1 * (double)GT[r]);
      }
    GS[(int64_t)b * n + c] = (float)(d1 * (double)GA[(int64_t)b * n + c] + d2 * ut);
  }
}

// gb = sum_b GS[b, :]  (fp64, fixed order)
__global__ void k_tr_colsum(int B, int n, const float* __restrict__ GS, double* __restrict__ gb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += (double)GS[(int64_t)b * n + c];
  gb[c] = s;
}

// Adam (surrogate.py:393-403) on fp64 master parameters; refreshes the fp32 copy
// (mask: 0 on the zero-padded entries of a padded network, which stay zero)
__global__ void k_tr_adam(int64_t count, double* __restrict__ P, const double* __restrict__ G,
                          double* __restrict__ M, double* __restrict__ V, float* __restrict__ P32, double lr,
                          double b1, double b2, double eps, double c1, double c2, const double* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double g = mask ? G[i] * mask[i] : G[i];
    const double m = b1 * M[i] + (1.0 - b1) * g;
    const double v = b2 * V[i] + (1.0 - b2) * g * g;
    M[i] = m;
    V[i] = v;
    const double p = P[i] - lr * (m / c1) / (sqrt(v / c2) + eps);
    P[i] = p;
    P32[i] = (float)p;
  }
}

// out (cols x rows) = in (rows x cols)^T, 32 x 32 smem tiles
__global__ void k_tr_transpose(int64_t rows, int cols, const float* __restrict__ in, float* __restrict__ out) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32;
  const int c0 = blockIdx.x * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y;
    const int c = c0 + threadIdx.x;
    t[y][threadIdx.x] = (r < rows && c < cols) ? in[r * cols + c] : 0.0f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y;
    const int64_t r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[(int64_t)c * rows + r] = t[threadIdx.x][y];
  }
}

// G64 += sum_z part[z] (fixed z order)
__global__ void k_tr_sum_z(int64_t count, int Z, const float* __restrict__ part, double* __restrict__ G) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < Z; ++z) s += (double)part[(int64_t)z * count + i];
    G[i] += s;
  }
}

__global__ void k_tr_f64_to_f32(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

}  // namespace sdn
