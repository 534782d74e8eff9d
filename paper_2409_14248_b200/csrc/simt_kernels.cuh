// simt_kernels.cuh -- FP32 FFMA (CUDA-core) kernels of the HRKAN jet hot path.
//
// These are the band-limited kernels: at any x only k+1 of the B = G+k bases are non-zero
// (compact support), so each (point, input) touches k+1 weights.  They
// serve the layers where K = I(G+k) is tiny (first layer, last layer, the [2,5,...] nets of
// C1/C2) and are the reference engine every tensor-core kernel is checked against.
//
// Jet layout in HBM (point-major):  X[p][c][i],  c = 0 value, 1..NF first derivatives
// d/dxi_a (a = c-1), 1+NF..NF+NS diagonal second derivatives d^2/dxi_a^2 (a = c-1-NF).
// NS <= NF; Poisson runs NF = NS = D, Burgers NF = 2 (x,t), NS = 1 (xx), boundary NF = NS = 0.
#pragma once
#include "hr_basis.cuh"

namespace {   // internal linkage: every translation unit owns its kernels
using namespace hrkan;

template <int NF, int NS>
struct Ch {
  static constexpr int C = 1 + NF + NS;
};

// Layer-input jet of one (point, input): x, dx[NF], ddx[NS].  Layer 0 synthesises the jet of the
// raw coordinates: x_i = xi_i, dx_{i,a} = delta_ia, ddx = 0.
template <int NF, int NS, bool FIRST>
__device__ __forceinline__ void load_jet(const float* __restrict__ X, int64_t p, int i, int I,
                                         float& x, float (&dx)[NF > 0 ? NF : 1],
                                         float (&ddx)[NS > 0 ? NS : 1]) {
  constexpr int C = 1 + NF + NS;
  if (FIRST) {
    x = __ldg(X + p * I + i);
#pragma unroll
    for (int a = 0; a < NF; ++a) dx[a] = (a == i) ? 1.f : 0.f;
#pragma unroll
    for (int a = 0; a < NS; ++a) ddx[a] = 0.f;
  } else {
    const float* base = X + p * (int64_t)(C * I) + i;
    x = __ldg(base);
#pragma unroll
    for (int a = 0; a < NF; ++a) dx[a] = __ldg(base + (1 + a) * I);
#pragma unroll
    for (int a = 0; a < NS; ++a) ddx[a] = __ldg(base + (1 + NF + a) * I);
  }
}

// ---------------------------------------------------------------------------------------------
// Forward layer:  Y[p][c][j] = [c==0] b_j + sum_{i,n} W[j,i,n] A^c[p,i,n]
//   A^0 = v_n(x_i), A^{1,a} = v'_n(x_i) dx_{i,a}, A^{2,a} = v''_n(x_i) dx_{i,a}^2 + v'_n(x_i) ddx_{i,a}
// One thread per (p, j); Wt = W transposed to [i][n][j] so a warp's weight loads coalesce.
// ---------------------------------------------------------------------------------------------
template <int NF, int NS, int M, bool FIRST>
__global__ void __launch_bounds__(256) k_fwd_simt(const float* __restrict__ X, const float* __restrict__ Wt,
                                                  const float* __restrict__ bias, float* __restrict__ Y,
                                                  int64_t P, int I, int O, BasisCfg bc) {
  constexpr int C = 1 + NF + NS;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * O) return;
  const int64_t p = idx / O;
  const int j = (int)(idx - p * O);
  float acc[C];
  acc[0] = __ldg(bias + j);
#pragma unroll
  for (int c = 1; c < C; ++c) acc[c] = 0.f;
  for (int i = 0; i < I; ++i) {
    float x, dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
    load_jet<NF, NS, FIRST>(X, p, i, I, x, dx, ddx);
    if (x != x) acc[0] += x;   // propagate NaN inputs (the basis test t > 0 would drop them)
    const int n0 = first_basis(x, bc);
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
      if (r > bc.k) break;
      const int n = n0 + r;
      if (n < 0 || n >= bc.B) continue;
      float v0, v1, v2, v3;
      hr_eval<M, (NS > 0 ? 2 : (NF > 0 ? 1 : 0))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
      const float w = __ldg(Wt + ((int64_t)i * bc.B + n) * O + j);
      acc[0] = fmaf(w, v0, acc[0]);
#pragma unroll
      for (int a = 0; a < NF; ++a) acc[1 + a] = fmaf(w * v1, dx[a], acc[1 + a]);
#pragma unroll
      for (int a = 0; a < NS; ++a) acc[1 + NF + a] = fmaf(w, fmaf(v2 * dx[a], dx[a], v1 * ddx[a]), acc[1 + NF + a]);
    }
  }
  float* out = Y + p * (int64_t)(C * O) + j;
#pragma unroll
  for (int c = 0; c < C; ++c) out[c * O] = acc[c];
}

// ---------------------------------------------------------------------------------------------
// Reverse, input adjoint ("dgrad" + jet-chain epilogue):
//   Abar^c[p,i,n] = sum_j Ybar[p][c][j] W[j,i,n]
//   xbar      = sum_n [Abar^0 v' + sum_a Abar^{1,a} v'' dx_a + sum_a Abar^{2,a} (v''' dx_a^2 + v'' ddx_a)]
//   dxbar_a   = sum_n [Abar^{1,a} v' + 2 Abar^{2,a} v'' dx_a]
//   ddxbar_a  = sum_n  Abar^{2,a} v'
// One thread per (p, i); only the k+1 non-zero bases of x_i are visited.
// ---------------------------------------------------------------------------------------------
template <int NF, int NS, int M>
__global__ void __launch_bounds__(256) k_dgrad_simt(const float* __restrict__ X, const float* __restrict__ W,
                                                    const float* __restrict__ Ybar, float* __restrict__ Xbar,
                                                    int64_t P, int I, int O, BasisCfg bc) {
  constexpr int C = 1 + NF + NS;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * I) return;
  const int64_t p = idx / I;
  const int i = (int)(idx - p * I);
  float x, dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
  load_jet<NF, NS, false>(X, p, i, I, x, dx, ddx);
  const int n0 = first_basis(x, bc);
  float v1[KMAX], v2[KMAX], v3[KMAX];
  bool ok[KMAX];
  float ab[C][KMAX];
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {
    const int n = n0 + r;
    ok[r] = (r <= bc.k) && n >= 0 && n < bc.B;
    float v0;
    v1[r] = v2[r] = v3[r] = 0.f;
    if (ok[r]) hr_eval<M, (NS > 0 ? 3 : 2)>(basis_q(x, n, bc), bc.sc, v0, v1[r], v2[r], v3[r]);
    ok[r] = ok[r] && (v1[r] != 0.f || v2[r] != 0.f || v3[r] != 0.f);
#pragma unroll
    for (int c = 0; c < C; ++c) ab[c][r] = 0.f;
  }
  const float* yb = Ybar + p * (int64_t)(C * O);
  const float* wrow = W + (int64_t)i * bc.B + n0;
  for (int j = 0; j < O; ++j) {
    float y[C];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = __ldg(yb + c * O + j);
    const float* wj = wrow + (int64_t)j * I * bc.B;
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
      if (!ok[r]) continue;
      const float w = __ldg(wj + r);
#pragma unroll
      for (int c = 0; c < C; ++c) ab[c][r] = fmaf(y[c], w, ab[c][r]);
    }
  }
  float xb = 0.f, dxb[NF > 0 ? NF : 1], ddxb[NS > 0 ? NS : 1];
#pragma unroll
  for (int a = 0; a < NF; ++a) dxb[a] = 0.f;
#pragma unroll
  for (int a = 0; a < NS; ++a) ddxb[a] = 0.f;
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {
    if (!ok[r]) continue;
    xb = fmaf(ab[0][r], v1[r], xb);
#pragma unroll
    for (int a = 0; a < NF; ++a) {
      xb = fmaf(ab[1 + a][r] * v2[r], dx[a], xb);
      dxb[a] = fmaf(ab[1 + a][r], v1[r], dxb[a]);
    }
#pragma unroll
    for (int a = 0; a < NS; ++a) {
      const float g = ab[1 + NF + a][r];
      xb = fmaf(g, fmaf(v3[r] * dx[a], dx[a], v2[r] * ddx[a]), xb);
      dxb[a] = fmaf(2.f * g * v2[r], dx[a], dxb[a]);
      ddxb[a] = fmaf(g, v1[r], ddxb[a]);
    }
  }
  float* out = Xbar + p * (int64_t)(C * I) + i;
  out[0] = xb;
#pragma unroll
  for (int a = 0; a < NF; ++a) out[(1 + a) * I] = dxb[a];
#pragma unroll
  for (int a = 0; a < NS; ++a) out[(1 + NF + a) * I] = ddxb[a];
}

// ---------------------------------------------------------------------------------------------
// Reverse, weight gradient ("wgrad"):
//   dW[j,i,n] += sum_p sum_c Ybar[p][c][j] A^c[p,i,n],   db_j += sum_p Ybar[p][0][j]
// Block = (32 outputs j) x (8 inputs i); the block walks a contiguous slice of the points
// (grid.z splits the points) and accumulates band-limited contributions in shared memory
// acc[i][n][j].  Each block writes its partial tile to part[z][O][I][B] (+ part_b[z][O]);
// k_reduce_parts sums the z-slices in a fixed order (deterministic, no float atomics).
// ---------------------------------------------------------------------------------------------
constexpr int WG_J = 32, WG_I = 8;

template <int NF, int NS, int M, bool FIRST>
__global__ void __launch_bounds__(WG_J* WG_I) k_wgrad_simt(const float* __restrict__ X, const float* __restrict__ Ybar,
                                                           float* __restrict__ part, float* __restrict__ part_b,
                                                           int64_t P, int I, int O, BasisCfg bc) {
  constexpr int C = 1 + NF + NS;
  extern __shared__ float acc[];   // [WG_I][B][WG_J]
  const int jl = threadIdx.x, il = threadIdx.y;
  const int j = blockIdx.x * WG_J + jl;
  const int i = blockIdx.y * WG_I + il;
  const int B = bc.B;
  for (int t = il * WG_J + jl; t < WG_I * B * WG_J; t += WG_J * WG_I) acc[t] = 0.f;
  __syncthreads();
  const int64_t nz = gridDim.z;
  const int64_t p_lo = (P * blockIdx.z) / nz, p_hi = (P * (blockIdx.z + 1)) / nz;
  const bool active = (j < O) && (i < I);
  float db = 0.f;
  float* my = acc + il * B * WG_J + jl;
  if (active) {
    for (int64_t p = p_lo; p < p_hi; ++p) {
      float y[C];
      const float* yb = Ybar + p * (int64_t)(C * O) + j;
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = __ldg(yb + c * O);
      db += y[0];
      float x, dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
      load_jet<NF, NS, FIRST>(X, p, i, I, x, dx, ddx);
      // fold the seeds with the jet: sum_c y_c A^c = y0 v + v' (sum_a y1_a dx_a + sum_a y2_a ddx_a)
      //                                              + v'' sum_a y2_a dx_a^2
      float g1 = 0.f, g2 = 0.f;
#pragma unroll
      for (int a = 0; a < NF; ++a) g1 = fmaf(y[1 + a], dx[a], g1);
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        g1 = fmaf(y[1 + NF + a], ddx[a], g1);
        g2 = fmaf(y[1 + NF + a] * dx[a], dx[a], g2);
      }
      const int n0 = first_basis(x, bc);
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        if (r > bc.k) break;
        const int n = n0 + r;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 2 : (NF > 0 ? 1 : 0))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        const float contrib = fmaf(y[0], v0, fmaf(g1, v1, g2 * v2));
        my[n * WG_J] += contrib;
      }
    }
  }
  __syncthreads();
  const int64_t nparam = (int64_t)O * I * B;
  float* dst = part + blockIdx.z * nparam;
  if (active) {
    for (int n = 0; n < B; ++n) dst[((int64_t)j * I + i) * B + n] = my[n * WG_J];
    if (blockIdx.y == 0 && il == 0) part_b[blockIdx.z * (int64_t)O + j] = db;
  }
}

// dW[t] += sum_z part[z][t] in a fixed z order (t over O*I*B weights then O biases).
__global__ void k_reduce_parts(const float* __restrict__ part, const float* __restrict__ part_b, int nz,
                               int64_t nW, int O, float* __restrict__ dW, float* __restrict__ db) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nW) {
    float s0 = 0.f, s1 = 0.f;                      // 2 independent chains, combined in a fixed order
    int z = 0;
    for (; z + 2 <= nz; z += 2) {
      s0 += part[z * nW + t];
      s1 += part[(z + 1) * nW + t];
    }
    if (z < nz) s0 += part[z * nW + t];
    dW[t] += s0 + s1;
  } else if (t < nW + O) {
    const int j = (int)(t - nW);
    float s = 0.f;
    for (int z = 0; z < nz; ++z) s += part_b[z * (int64_t)O + j];
    db[j] += s;
  }
}

// W[j][i][n] -> Wt[i][n][j]
__global__ void k_transpose_w(const float* __restrict__ W, float* __restrict__ Wt, int O, int IB) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)O * IB) return;
  const int j = (int)(t / IB), q = (int)(t - (int64_t)j * IB);
  Wt[(int64_t)q * O + j] = W[t];
}

// Bias-corrected Adam.  bc1 = 1 - beta1^t, bc2 = 1 - beta2^t.
// Bias-corrected Adam.  The step count lives on the device (t_cnt[0] = t before this
// step, t_cnt[1] = finished-block counter): every block computes the corrections for t + 1 and the
// last block to finish advances t and resets the counter, so a CUDA-graph replay of this launch
// keeps advancing the bias correction.
__global__ void k_adam(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, int64_t n, float lr, float b1, float b2, float eps,
                       int* __restrict__ t_cnt) {
  __shared__ float s_bc[2];
  if (threadIdx.x == 0) {
    const double t = (double)(*(volatile int*)t_cnt + 1);
    s_bc[0] = (float)(1.0 / (1.0 - pow((double)b1, t)));
    s_bc[1] = (float)(1.0 / (1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) {
    const float gi = g[t];
    const float mi = fmaf(b1, m[t], (1.f - b1) * gi);
    const float vi = fmaf(b2, v[t], (1.f - b2) * gi * gi);
    m[t] = mi;
    v[t] = vi;
    theta[t] -= lr * (mi * s_bc[0]) / (sqrtf(vi * s_bc[1]) + eps);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(reinterpret_cast<unsigned*>(t_cnt + 1), 1u) == gridDim.x - 1) {
      t_cnt[0] += 1;
      t_cnt[1] = 0;
      __threadfence();
    }
  }
}

// Counter-based Philox4x32-10 (Salmon et al., SC'11) + Box-Muller: W ~ N(0, std^2), b = 0.
__device__ __forceinline__ void philox4x32_10(uint32_t (&ctr)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * ctr[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * ctr[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ ctr[1] ^ k0, n2 = hi0 ^ ctr[3] ^ k1;
    ctr[0] = n0; ctr[1] = lo1; ctr[2] = n2; ctr[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__global__ void k_init_layer(float* __restrict__ W, float* __restrict__ b, int64_t nW, int O, float stdv,
                             uint64_t seed, uint32_t layer) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nW) {
    uint32_t c[4] = {(uint32_t)t, (uint32_t)(t >> 32), layer, 0x48524b41u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const float u1 = ((float)(c[0] >> 8) + 0.5f) * (1.f / 16777216.f);   // (0,1)
    const float u2 = ((float)(c[1] >> 8)) * (1.f / 16777216.f);
    W[t] = stdv * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
  if (t < O) b[t] = 0.f;
}

}  // namespace
