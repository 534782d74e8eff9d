// hr_basis.cuh -- device evaluation of the Higher-order-ReLU basis and its x-derivatives.
//
// PAPER.md:90-94 (Sec. 3, Eq. 2):  v_{m,n}(x) = ReLU(e_n - x)^m ReLU(x - s_n)^m c_m,
// c_m = (2/(e_n - s_n))^{2m}.  The kernels use the normalised coordinate
// q = (x - mid_n) (2/w), w = e_n - s_n = (k+1)h, in which Eq. 2 reads v = (1 - q^2)^m:
//   dv/dq     = -2m q t^{m-1}                         (t = 1 - q^2)
//   d2v/dq2   = -2m t^{m-2} [1 - (2m-1) q^2]
//   d3v/dq3   =  4m(m-1) q t^{m-3} [3 - (2m-1) q^2]     (m = 2:  24 q)
//   d^d v/dx^d = (2/w)^d d^d v/dq^d.
// Strict interior (t > 0) only; every derivative is exactly 0 elsewhere (DESIGN.md reading:
// ReLU(0) = 0, one-sided limits are not taken at the knots).  A NaN input yields NaN values so that
// non-finite inputs reach the loss and its non-finite flag.
//
// Supports ("same support as the B-splines"; reading 1):
// s_n = lo + (n-k)h, e_n = s_n + (k+1)h, h = (hi-lo)/G, n = 0..G+k-1, so at any x the only
// non-zero bases are n = floor((x-lo)/h) + r, r = 0..k  (at most k+1 of them).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hrkan {

constexpr int KMAX = 8;   // k+1 <= KMAX bases can be non-zero at one x (k <= 7 supported)

struct BasisCfg {
  float lo;       // grid_lo
  float h;        // (hi - lo) / G
  float inv_h;    // 1 / h
  float sc;       // 2 / w,  w = (k+1) h
  float mid0;     // centre of support 0:  lo + (1 - k)/2 * h
  int k;          // B-spline order (k+1 non-zero bases per x)
  int B;          // G + k bases
};

template <int M>
__device__ __forceinline__ float ipow(float t) {
  float r = 1.f;
#pragma unroll
  for (int i = 0; i < M; ++i) r *= t;
  return r;
}

// Values and x-derivatives up to order ND (0..3) at normalised coordinate q; zero outside.
template <int M, int ND>
__device__ __forceinline__ void hr_eval(float q, float sc, float& v0, float& v1, float& v2, float& v3) {
  const float q2 = q * q;
  const float t = 1.f - q2;
  if (!(t > 0.f)) {                      // outside the support (or NaN: propagate it)
    v0 = v1 = v2 = v3 = (t != t) ? t : 0.f;
    return;
  }
  // t^{m-3} ... t^m by repeated products (M is a compile-time constant)
  const float tm2 = ipow<(M >= 2 ? M - 2 : 0)>(t);
  const float tm1 = tm2 * t;
  v0 = tm1 * t;
  v1 = (-2.f * M) * q * tm1 * sc;
  if (ND >= 2) v2 = (-2.f * M) * tm2 * (1.f - (2.f * M - 1.f) * q2) * (sc * sc); else v2 = 0.f;
  if (ND >= 3) {
    if (M == 2) {
      v3 = 24.f * q * (sc * sc * sc);
    } else {
      const float tm3 = ipow<(M >= 3 ? M - 3 : 0)>(t);
      v3 = (4.f * M * (M - 1)) * q * tm3 * (3.f - (2.f * M - 1.f) * q2) * (sc * sc * sc);
    }
  } else {
    v3 = 0.f;
  }
}

// First candidate basis index at x (may be negative / >= B: callers test 0 <= n < B).
__device__ __forceinline__ int first_basis(float x, const BasisCfg& bc) {
  float u = (x - bc.lo) * bc.inv_h;
  u = fminf(fmaxf(u, -1.0e6f), 1.0e6f);   // keeps the int conversion defined for inf
  return __float2int_rd(u);
}

__device__ __forceinline__ float basis_q(float x, int n, const BasisCfg& bc) {
  return (x - fmaf((float)n, bc.h, bc.mid0)) * bc.sc;
}

}  // namespace hrkan
