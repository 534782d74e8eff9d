// jet_kernels.cuh -- higher-order and mixed jets: the HRKAN layer stack evaluated on
// jets beyond the diagonal second-order one, for PDEs with a fifth x-derivative ("If a PDE
// equation possesses derivative terms of order higher than 4, for example, u_xxxxx, we can pick m to be
// larger, like 6") or with mixed second derivatives (full Hessian).
//
// A jet spec S fixes the channels c = 0..C-1 of a layer's input/output jet and how a univariate basis
// function phi composes with them.  For an input jet x[c] of one (point, input i) and the basis
// derivatives f_k = phi^{(k)}(x_0), the layer operand is linear in the f_k:
//     A_c = sum_k f_k M_{c,k}(x)                                    (S::gen)
// so a layer is Y[p][c][j] = [c==0] b_j + sum_{i,n} W[j,i,n] A_c(p,i,n) (the KAN matrix product, P:45/P:87
// applied per channel).  The reverse pass uses two more forms of the same polynomials:
//     sum_c y_c A_c = sum_k g_k(y, x) f_k                            (S::fold, weight gradient)
//     xbar_0 = sum_k g_k(S_{k+1}, x),  xbar_s = sum_k dg_k/dx_s (S_k, x)   (S::dfold, input adjoint)
// with S_k[c] = sum_n phi_n^{(k)} Abar_c(n) accumulated over the k+1 non-zero bases.
//
//   JsTaylor5   D = 2 (x, t): channels [z, z_x, z_xx, z_xxx, z_xxxx, z_xxxxx, z_t]; the x-orders compose by
//               Faa di Bruno's formula d^r phi(h) = sum_k phi^{(k)}(h) B_{r,k}(h', ..., h^{(r-k+1)}) with the
//               partial Bell polynomials B_{r,k} written out for r <= 5; z_t = phi'(h) h_t.
//   JsHess<D>   D = 2, 3: channels [z, z_a (a < D), z_ab (a <= b, row-major upper triangle)];
//               z_ab = phi''(h) h_a h_b + phi'(h) h_ab (second-order chain rule).
// The CPU oracle (oracle/hrkan_oracle_jets.py) derives the same jets differently (truncated power-series
// composition; exact polynomial basis derivatives), shares no code with this file.
//
// Kernels (FP32 FFMA, band-limited: only the k+1 non-zero bases of each input are visited):
//   k_js_seed        layer-0 input jet from the points;
//   k_js_fwd         hidden / first layer: a block = PT points x all outputs j (one thread per j); the
//                    (point, input) operands of the non-zero bases are generated once into shared memory
//                    and every output thread contracts them with coalesced weight rows Wt[i][n][j];
//   k_js_fwd_o1      output layer (O = 1): a warp per point, lanes over inputs, butterfly reduction;
//   k_js_loss        residual, loss partials and seeds of the output jet (Kawahara / anisotropic);
//   k_js_wgrad       dW[j,i,n] = sum_p sum_k g_k(Ybar[p,.,j], X[p,.,i]) phi_n^{(k)}(X[p,0,i]) per point slice,
//                    summed over slices by k_reduce_parts (fixed order);
//   k_js_dgrad       input adjoint per (point, input).
#pragma once
#include "hr_basis.cuh"

namespace {
using namespace hrkan;

// ---------------------------------------------------------------------------------------------
// Basis derivatives of any order (Eq. 2 in the normalised coordinate q, t = 1 - q^2, v = t^m):
//   d^d v/dq^d = sum_{k = ceil(d/2)}^{min(d, m)} m!/(m-k)! d!/((2k-d)!(d-k)!) (-1)^{d-k} (-2q)^{2k-d} t^{m-k}
// (Faa di Bruno for g(t) = t^m, t(q) = 1 - q^2 with t' = -2q, t'' = -2), d^d v/dx^d = sc^d d^d v/dq^d.
// Zero outside the support (t <= 0), NaN kept.
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr double js_fact(int n) { return n <= 1 ? 1.0 : n * js_fact(n - 1); }
__host__ __device__ constexpr float js_coef(int m, int d, int k) {
  return (float)(js_fact(m) / js_fact(m - k) * js_fact(d) / (js_fact(2 * k - d) * js_fact(d - k)) *
                 (((d - k) & 1) ? -1.0 : 1.0));
}

// sum over k of the d-th derivative's terms; every coefficient is a compile-time constant
template <int M, int D, int K, int ND>
__device__ __forceinline__ float js_terms(const float (&qp)[ND + 1], const float (&tp)[M + 1]) {
  if constexpr (K > (D < M ? D : M)) {
    return 0.f;
  } else {
    constexpr float c = js_coef(M, D, K);
    return fmaf(c * qp[2 * K - D], tp[M - K], js_terms<M, D, K + 1, ND>(qp, tp));
  }
}
template <int M, int D, int ND>
__device__ __forceinline__ void js_fill(float (&f)[ND + 1], const float (&qp)[ND + 1], const float (&tp)[M + 1],
                                        float scd, float sc) {
  if constexpr (D <= ND) {
    f[D] = js_terms<M, D, (D + 1) / 2, ND>(qp, tp) * scd;
    js_fill<M, D + 1, ND>(f, qp, tp, scd * sc, sc);
  }
}

template <int M, int ND>
__device__ __forceinline__ void hr_eval_n(float q, float sc, float (&f)[ND + 1]) {
  const float t = 1.f - q * q;
  if (!(t > 0.f)) {
    const float z = (t != t) ? t : 0.f;
#pragma unroll
    for (int d = 0; d <= ND; ++d) f[d] = z;
    return;
  }
  float tp[M + 1];                       // t^0 .. t^M
  tp[0] = 1.f;
#pragma unroll
  for (int e = 1; e <= M; ++e) tp[e] = tp[e - 1] * t;
  const float m2q = -2.f * q;
  float qp[ND + 1];                      // (-2q)^0 .. (-2q)^ND
  qp[0] = 1.f;
#pragma unroll
  for (int e = 1; e <= ND; ++e) qp[e] = qp[e - 1] * m2q;
  js_fill<M, 0, ND>(f, qp, tp, 1.f, sc);
}

// ---------------------------------------------------------------------------------------------
// Jet specs
// ---------------------------------------------------------------------------------------------
struct JsTaylor5 {
  static constexpr int C = 7, D = 2, R = 5;
  static constexpr int TDIR = 1;          // t = input coordinate 1, x = coordinate 0
  __device__ static float seed(int c, int i) { return ((c == 1 && i == 0) || (c == 6 && i == TDIR)) ? 1.f : 0.f; }
  __device__ static void gen(const float (&f)[R + 1], const float (&x)[C], float (&A)[C]) {
    const float x1 = x[1], x2 = x[2], x3 = x[3], x4 = x[4], x5 = x[5];
    const float x11 = x1 * x1, x111 = x11 * x1;
    A[0] = f[0];
    A[1] = f[1] * x1;
    A[2] = fmaf(f[1], x2, f[2] * x11);
    A[3] = fmaf(f[1], x3, fmaf(3.f * f[2], x1 * x2, f[3] * x111));
    A[4] = fmaf(f[1], x4, fmaf(f[2], fmaf(4.f * x1, x3, 3.f * x2 * x2), fmaf(6.f * f[3], x11 * x2, f[4] * x11 * x11)));
    A[5] = fmaf(f[1], x5,
                fmaf(f[2], fmaf(5.f * x1, x4, 10.f * x2 * x3),
                     fmaf(f[3], fmaf(15.f * x1, x2 * x2, 10.f * x11 * x3), fmaf(10.f * f[4], x111 * x2, f[5] * x111 * x11))));
    A[6] = f[1] * x[6];
  }
  // sum_c y_c A_c = sum_k g_k f_k
  __device__ static void fold(const float (&y)[C], const float (&x)[C], float (&g)[R + 1]) {
    const float x1 = x[1], x2 = x[2], x3 = x[3], x4 = x[4], x5 = x[5];
    const float x11 = x1 * x1, x111 = x11 * x1;
    g[0] = y[0];
    g[1] = fmaf(y[1], x1, fmaf(y[2], x2, fmaf(y[3], x3, fmaf(y[4], x4, fmaf(y[5], x5, y[6] * x[6])))));
    g[2] = fmaf(y[2], x11, fmaf(3.f * y[3], x1 * x2, fmaf(y[4], fmaf(4.f * x1, x3, 3.f * x2 * x2), y[5] * fmaf(5.f * x1, x4, 10.f * x2 * x3))));
    g[3] = fmaf(y[3], x111, fmaf(6.f * y[4], x11 * x2, y[5] * fmaf(15.f * x1, x2 * x2, 10.f * x11 * x3)));
    g[4] = fmaf(y[4], x11 * x11, 10.f * y[5] * x111 * x2);
    g[5] = y[5] * x111 * x11;
  }
  // S[k][c] = sum_n phi_n^{(k)} Abar_c(n), k = 0..R+1:  xbar_0 = sum_k g_k(S_{k+1}), xbar_s = sum_k dg_k/dx_s(S_k)
  __device__ static void dfold(const float (&S)[R + 2][C], const float (&x)[C], float (&xb)[C]) {
    xb[0] = 0.f;
#pragma unroll
    for (int k = 0; k <= R; ++k) {
      float g[R + 1];
      fold(S[k + 1], x, g);
      xb[0] += g[k];
    }
    const float x1 = x[1], x2 = x[2], x3 = x[3], x4 = x[4];
    const float x11 = x1 * x1;
    xb[1] = S[1][1] + (2.f * S[2][2] * x1 + 3.f * S[2][3] * x2 + 4.f * S[2][4] * x3 + 5.f * S[2][5] * x4) +
            (3.f * S[3][3] * x11 + 12.f * S[3][4] * x1 * x2 + S[3][5] * (15.f * x2 * x2 + 20.f * x1 * x3)) +
            (4.f * S[4][4] * x11 * x1 + 30.f * S[4][5] * x11 * x2) + 5.f * S[5][5] * x11 * x11;
    xb[2] = S[1][2] + (3.f * S[2][3] * x1 + 6.f * S[2][4] * x2 + 10.f * S[2][5] * x3) +
            (6.f * S[3][4] * x11 + 30.f * S[3][5] * x1 * x2) + 10.f * S[4][5] * x11 * x1;
    xb[3] = S[1][3] + (4.f * S[2][4] * x1 + 10.f * S[2][5] * x2) + 10.f * S[3][5] * x11;
    xb[4] = S[1][4] + 5.f * S[2][5] * x1;
    xb[5] = S[1][5];
    xb[6] = S[1][6];
  }
};

template <int DD>
struct JsHess {
  static constexpr int D = DD, NPAIR = DD * (DD + 1) / 2, C = 1 + DD + NPAIR, R = 2;
  __device__ static constexpr int pa(int q) { return DD == 2 ? (q < 2 ? 0 : 1) : (q < 3 ? 0 : q < 5 ? 1 : 2); }
  __device__ static constexpr int pb(int q) { return DD == 2 ? (q == 0 ? 0 : 1) : (q == 0 ? 0 : q == 1 ? 1 : q == 2 ? 2 : q == 3 ? 1 : 2); }
  __device__ static float seed(int c, int i) { return (c == 1 + i && i < DD) ? 1.f : 0.f; }
  __device__ static void gen(const float (&f)[R + 1], const float (&x)[C], float (&A)[C]) {
    A[0] = f[0];
#pragma unroll
    for (int a = 0; a < DD; ++a) A[1 + a] = f[1] * x[1 + a];
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) A[1 + DD + q] = fmaf(f[2] * x[1 + pa(q)], x[1 + pb(q)], f[1] * x[1 + DD + q]);
  }
  __device__ static void fold(const float (&y)[C], const float (&x)[C], float (&g)[R + 1]) {
    g[0] = y[0];
    float g1 = 0.f, g2 = 0.f;
#pragma unroll
    for (int a = 0; a < DD; ++a) g1 = fmaf(y[1 + a], x[1 + a], g1);
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) {
      g1 = fmaf(y[1 + DD + q], x[1 + DD + q], g1);
      g2 = fmaf(y[1 + DD + q] * x[1 + pa(q)], x[1 + pb(q)], g2);
    }
    g[1] = g1;
    g[2] = g2;
  }
  __device__ static void dfold(const float (&S)[R + 2][C], const float (&x)[C], float (&xb)[C]) {
    xb[0] = 0.f;
#pragma unroll
    for (int k = 0; k <= R; ++k) {
      float g[R + 1];
      fold(S[k + 1], x, g);
      xb[0] += g[k];
    }
#pragma unroll
    for (int a = 0; a < DD; ++a) {
      float s = S[1][1 + a];
#pragma unroll
      for (int q = 0; q < NPAIR; ++q) {
        if (pa(q) == a) s = fmaf(S[2][1 + DD + q], x[1 + pb(q)], s);
        if (pb(q) == a) s = fmaf(S[2][1 + DD + q], x[1 + pa(q)], s);
      }
      xb[1 + a] = s;
    }
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) xb[1 + DD + q] = S[1][1 + DD + q];
  }
};

// layer-input jet of one (point, input): FIRST synthesises the jet of the raw coordinates
template <class S, bool FIRST>
__device__ __forceinline__ void js_load(const float* __restrict__ X, int64_t p, int i, int I, float (&x)[S::C]) {
  if (FIRST) {
    x[0] = __ldg(X + p * I + i);
#pragma unroll
    for (int c = 1; c < S::C; ++c) x[c] = S::seed(c, i);
  } else {
    const float* b = X + p * (int64_t)(S::C * I) + i;
#pragma unroll
    for (int c = 0; c < S::C; ++c) x[c] = __ldg(b + c * I);
  }
}

// ---------------------------------------------------------------------------------------------
// Forward layer, O >= 2 outputs.  Block: PT points, blockDim = O rounded up to 32 (one thread per
// output j); per chunk of JS_ICH inputs the (point, input) operands of the non-zero bases are generated
// once into shared memory tab[(ii, pl)][r][c] and contracted by every output thread.
// ---------------------------------------------------------------------------------------------
constexpr int JS_PT = 8, JS_ICH = 8;

template <class S, int M, bool FIRST>
__global__ void __launch_bounds__(256) k_js_fwd(const float* __restrict__ X, const float* __restrict__ Wt,
                                                const float* __restrict__ bias, float* __restrict__ Y, int64_t P,
                                                int I, int O, BasisCfg bc) {
  constexpr int C = S::C;
  __shared__ float tab[JS_ICH * JS_PT][KMAX][C];
  __shared__ int nb0[JS_ICH * JS_PT];
  const int64_t p0 = (int64_t)blockIdx.x * JS_PT;
  const int j = threadIdx.x;
  const int B = bc.B, kk = bc.k;
  float acc[JS_PT][C];
#pragma unroll
  for (int pl = 0; pl < JS_PT; ++pl)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[pl][c] = 0.f;
  for (int i0 = 0; i0 < I; i0 += JS_ICH) {
    __syncthreads();
    for (int e = threadIdx.x; e < JS_ICH * JS_PT; e += blockDim.x) {
      const int ii = e / JS_PT, pl = e - ii * JS_PT;
      const int i = i0 + ii;
      const int64_t p = p0 + pl;
      int n0 = 0;
      if (i < I && p < P) {
        float x[C];
        js_load<S, FIRST>(X, p, i, I, x);
        const bool nan = x[0] != x[0];
        n0 = nan ? 0 : first_basis(x[0], bc);
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          const int n = n0 + r;
          float A[C];
          if (nan) {
#pragma unroll
            for (int c = 0; c < C; ++c) A[c] = (r == 0) ? x[0] : 0.f;      // NaN reaches every channel
          } else if (r <= kk && n >= 0 && n < B) {
            float f[S::R + 1];
            hr_eval_n<M, S::R>(basis_q(x[0], n, bc), bc.sc, f);
            S::gen(f, x, A);
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) A[c] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < C; ++c) tab[e][r][c] = A[c];
        }
      } else {
#pragma unroll
        for (int r = 0; r < KMAX; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c) tab[e][r][c] = 0.f;
      }
      nb0[e] = n0;
    }
    __syncthreads();
    if (j < O) {
      const int iend = min(JS_ICH, I - i0);
      for (int ii = 0; ii < iend; ++ii) {
        const float* wrow = Wt + (int64_t)(i0 + ii) * B * O + j;
#pragma unroll
        for (int pl = 0; pl < JS_PT; ++pl) {
          const int e = ii * JS_PT + pl;
          const int n0 = nb0[e];
#pragma unroll
          for (int r = 0; r < KMAX; ++r) {
            if (r > kk) break;
            const int n = n0 + r;
            if (n < 0 || n >= B) continue;
            const float w = __ldg(wrow + (int64_t)n * O);
#pragma unroll
            for (int c = 0; c < C; ++c) acc[pl][c] = fmaf(w, tab[e][r][c], acc[pl][c]);
          }
        }
      }
    }
  }
  if (j < O) {
    const float b = __ldg(bias + j);
#pragma unroll
    for (int pl = 0; pl < JS_PT; ++pl) {
      const int64_t p = p0 + pl;
      if (p >= P) break;
      float* out = Y + p * (int64_t)(C * O) + j;
#pragma unroll
      for (int c = 0; c < C; ++c) out[c * O] = acc[pl][c] + (c == 0 ? b : 0.f);
    }
  }
}

// Output layer (O = 1): a warp per point, lanes over inputs, fixed-order butterfly reduction.
// W is the layer's own row W[0][i][n]; U[p][c] is the network's output jet.
constexpr int JS_LW = 8;   // warps per block
template <class S, int M, bool FIRST>
__global__ void __launch_bounds__(32 * JS_LW) k_js_fwd_o1(const float* __restrict__ X, const float* __restrict__ W,
                                                          const float* __restrict__ bias, float* __restrict__ U,
                                                          int64_t P, int I, BasisCfg bc) {
  constexpr int C = S::C;
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * JS_LW + (threadIdx.x >> 5);
  if (p >= P) return;
  float acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.f;
  for (int i = lane; i < I; i += 32) {
    float x[C];
    js_load<S, FIRST>(X, p, i, I, x);
    if (x[0] != x[0]) {
      acc[0] += x[0];
      continue;
    }
    const int n0 = first_basis(x[0], bc);
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
      if (r > bc.k) break;
      const int n = n0 + r;
      if (n < 0 || n >= bc.B) continue;
      float f[S::R + 1], A[C];
      hr_eval_n<M, S::R>(basis_q(x[0], n, bc), bc.sc, f);
      S::gen(f, x, A);
      const float w = __ldg(W + (int64_t)i * bc.B + n);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = fmaf(w, A[c], acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < C; ++c) U[p * C + c] = acc[c] + (c == 0 ? __ldg(bias) : 0.f);
  }
}

// ---------------------------------------------------------------------------------------------
// Residual, loss partials and seeds (output jet U[p][C]).
//   JS_KAWAHARA: r = u_t + adv u u_x + disp3 u_xxx - disp5 u_xxxxx  (S = JsTaylor5)
//   JS_ANISO:    r = sum_{a<=b} K_ab u_ab - f                          (S = JsHess<D>)
// seeds Ybar[p][c] = d(alpha r^2 / N_int)/dU_c; per block: (sum r^2, non-finite count) -> part[2*block]
// ---------------------------------------------------------------------------------------------
enum JsPde { JS_KAWAHARA = 0, JS_ANISO = 1 };
struct JsPdeArgs {
  float alpha, adv, disp3, disp5;
  float K[6];
  float inv_n;
};

template <class S, int PDE>
__global__ void __launch_bounds__(256) k_js_loss(const float* __restrict__ U, const float* __restrict__ forcing,
                                                 float* __restrict__ Ybar, float* __restrict__ part, int64_t P,
                                                 JsPdeArgs pa) {
  constexpr int C = S::C;
  __shared__ float sh_r[8], sh_f[8];
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float r2 = 0.f, bad = 0.f;
  if (p < P) {
    float u[C], y[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      u[c] = U[p * C + c];
      y[c] = 0.f;
    }
    float r;
    const float g0 = 2.f * pa.alpha * pa.inv_n;
    if constexpr (PDE == JS_KAWAHARA) {
      r = u[6] + pa.adv * u[0] * u[1] + pa.disp3 * u[3] - pa.disp5 * u[5];
      const float g = g0 * r;
      y[0] = g * pa.adv * u[1];
      y[1] = g * pa.adv * u[0];
      y[3] = g * pa.disp3;
      y[5] = -g * pa.disp5;
      y[6] = g;
    } else {
      r = -__ldg(forcing + p);
#pragma unroll
      for (int q = 0; q < S::NPAIR; ++q) r = fmaf(pa.K[q], u[1 + S::D + q], r);
      const float g = g0 * r;
#pragma unroll
      for (int q = 0; q < S::NPAIR; ++q) y[1 + S::D + q] = g * pa.K[q];
    }
    r2 = r * r;
    bad = isfinite(r) ? 0.f : 1.f;
#pragma unroll
    for (int c = 0; c < C; ++c) Ybar[p * C + c] = y[c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sh_r[threadIdx.x >> 5] = r2;
    sh_f[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += sh_r[w];
      b += sh_f[w];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// out_loss += scale * sum_b part[2b], out_flag += sum_b part[2b+1]  (one block, fixed order, fp64 sums)
__global__ void __launch_bounds__(256) k_js_reduce_loss(const float* __restrict__ part, int nb, float scale,
                                                        float* __restrict__ out_loss, float* __restrict__ out_flag) {
  __shared__ double sa[256], sb[256];
  double a = 0.0, b = 0.0;
  for (int q = threadIdx.x; q < nb; q += blockDim.x) {
    a += (double)part[2 * q];
    b += (double)part[2 * q + 1];
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      ta += sa[t];
      tb += sb[t];
    }
    *out_loss += (float)(ta * (double)scale);
    *out_flag += (float)tb;
  }
}

// ---------------------------------------------------------------------------------------------
// Weight gradient: block (JW outputs j) x (blockDim.y inputs i) over a slice of the points (grid.z),
// shared accumulator acc[i][n][j]; part[z][O][I][B] (+ part_b[z][O]) summed by k_reduce_parts.
// ---------------------------------------------------------------------------------------------
template <class S, int M, bool FIRST, int JW>
__global__ void __launch_bounds__(256) k_js_wgrad(const float* __restrict__ X, const float* __restrict__ Ybar,
                                                  float* __restrict__ part, float* __restrict__ part_b, int64_t P,
                                                  int I, int O, BasisCfg bc) {
  constexpr int C = S::C;
  extern __shared__ float acc[];   // [blockDim.y][B][JW]
  const int jl = threadIdx.x, il = threadIdx.y, IW = blockDim.y;
  const int j = blockIdx.x * JW + jl;
  const int i = blockIdx.y * IW + il;
  const int B = bc.B;
  for (int t = il * JW + jl; t < IW * B * JW; t += JW * IW) acc[t] = 0.f;
  __syncthreads();
  const int64_t nz = gridDim.z;
  const int64_t p_lo = (P * blockIdx.z) / nz, p_hi = (P * (blockIdx.z + 1)) / nz;
  const bool active = (j < O) && (i < I);
  float db = 0.f;
  float* my = acc + il * B * JW + jl;
  if (active) {
    for (int64_t p = p_lo; p < p_hi; ++p) {
      float y[C], x[C], g[S::R + 1];
      const float* yb = Ybar + p * (int64_t)(C * O) + j;
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = __ldg(yb + c * O);
      db += y[0];
      js_load<S, FIRST>(X, p, i, I, x);
      S::fold(y, x, g);
      const int n0 = first_basis(x[0], bc);
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        if (r > bc.k) break;
        const int n = n0 + r;
        if (n < 0 || n >= B) continue;
        float f[S::R + 1];
        hr_eval_n<M, S::R>(basis_q(x[0], n, bc), bc.sc, f);
        float contrib = 0.f;
#pragma unroll
        for (int k = 0; k <= S::R; ++k) contrib = fmaf(g[k], f[k], contrib);
        my[n * JW] += contrib;
      }
    }
  }
  __syncthreads();
  const int64_t nparam = (int64_t)O * I * B;
  float* dst = part + blockIdx.z * nparam;
  if (active) {
    for (int n = 0; n < B; ++n) dst[((int64_t)j * I + i) * B + n] = my[n * JW];
    if (blockIdx.y == 0 && il == 0) part_b[blockIdx.z * (int64_t)O + j] = db;
  }
}

// ---------------------------------------------------------------------------------------------
// Input adjoint per (point, input): Abar_c(n) = sum_j Ybar[p][c][j] W[j,i,n] over the non-zero bases,
// S_k = sum_n phi_n^{(k)} Abar(n), then S::dfold.
// ---------------------------------------------------------------------------------------------
template <class S, int M>
__global__ void __launch_bounds__(256) k_js_dgrad(const float* __restrict__ X, const float* __restrict__ W,
                                                  const float* __restrict__ Ybar, float* __restrict__ Xbar, int64_t P,
                                                  int I, int O, BasisCfg bc) {
  constexpr int C = S::C, R = S::R;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * I) return;
  const int64_t p = idx / I;
  const int i = (int)(idx - p * I);
  float x[C];
  js_load<S, false>(X, p, i, I, x);
  float* out = Xbar + p * (int64_t)(C * I) + i;
  if (x[0] != x[0]) {
#pragma unroll
    for (int c = 0; c < C; ++c) out[c * I] = x[0];
    return;
  }
  const int n0 = first_basis(x[0], bc);
  bool ok[KMAX];
  float ab[KMAX][C];
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {
    const int n = n0 + r;
    ok[r] = (r <= bc.k) && n >= 0 && n < bc.B;
#pragma unroll
    for (int c = 0; c < C; ++c) ab[r][c] = 0.f;
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
      for (int c = 0; c < C; ++c) ab[r][c] = fmaf(y[c], w, ab[r][c]);
    }
  }
  float Sk[R + 2][C];
#pragma unroll
  for (int k = 0; k < R + 2; ++k)
#pragma unroll
    for (int c = 0; c < C; ++c) Sk[k][c] = 0.f;
#pragma unroll
  for (int r = 0; r < KMAX; ++r) {
    if (!ok[r]) continue;
    float f[R + 2];
    hr_eval_n<M, R + 1>(basis_q(x[0], n0 + r, bc), bc.sc, f);
#pragma unroll
    for (int k = 1; k < R + 2; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) Sk[k][c] = fmaf(f[k], ab[r][c], Sk[k][c]);
  }
  float xb[C];
  S::dfold(Sk, x, xb);
#pragma unroll
  for (int c = 0; c < C; ++c) out[c * I] = xb[c];
}

}  // namespace
