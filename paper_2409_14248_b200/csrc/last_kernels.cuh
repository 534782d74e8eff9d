// last_kernels.cuh -- the output layer (O = 1) fused with the residual, the loss and its own reverse
// pass, one warp per collocation point.
//
// The output layer contracts K = I(G+k) features into ONE neuron, so per point it is a reduction
// over (i, n), not a GEMM: lanes own inputs i = lane, lane+32, ... (coalesced loads of the saved
// jet X[p][c][i]), each visits only the k+1 bases that are non-zero at x_i (compact support,
// PAPER.md:90-94), and a butterfly reduction gives every lane the output jet.  Then, without
// leaving the kernel:
//   residual   Poisson r = sum_a u_aa - f, f = -D pi^2 prod sin(pi xi_a) (Eq. 3) or forcing;
//              Burgers r = u_t + adv u u_x - visc u_xx (Eq. 5); boundary e = u - g;
//   seeds      ybar_c = dL/d(output jet channel c), L = alpha/N_int sum r^2 + 1/N_bi sum e^2;
//   reverse    per (p, i), with w_n = W[0, i, n] and T_d = sum_n w_n v_n^(d)(x_i):
//                dW[0,i,n] += y0 v_n + g1 v'_n + g2 v''_n,   g1 = sum_a y1_a dx_a + sum_a y2_a ddx_a,
//                                                            g2 = sum_a y2_a dx_a^2
//                xbar      = y0 T1 + g1 T2 + g2 T3
//                dxbar_a   = y1_a T1 + 2 y2_a dx_a T2,        ddxbar_a = y2_a T1
//              (the jet chain rule of SURVEY §8(c) c5 with Abar^c = ybar_c W specialised to O = 1).
// dW is accumulated per warp in shared memory acc[warp][n][i] (lanes own distinct i: no atomics,
// conflict-free), reduced over the block's warps in a fixed order into part[block][I*B + 4]
// (+ db, sum r^2, non-finite count), and k_reduce_last sums the blocks in a fixed order: the
// result is bitwise reproducible for a fixed grid.
#pragma once
#include "tc_ptx.cuh"   // packed fp32 pair helpers (FFMA2 / FMUL2)

namespace {   // internal linkage: every translation unit owns its kernels
using namespace hrkan;

constexpr int LF_WARPS = 4;

// Output-layer basis arithmetic on packed fp32 pairs (two bases per FFMA2/FMUL2, m >= 4): v0..v3 of
// bases na, nb at x with t = 1 - q^2 clamped at 0 (NaN kept), zero where !ok (outside [0, B)).
#ifndef HRKAN_LAST_F32X2
#define HRKAN_LAST_F32X2 1
#endif
template <int M>
__device__ __forceinline__ void hr_eval_pair(float x, int na, int nb, bool oka, bool okb, const BasisCfg& bc,
                                             uint64_t& v0, uint64_t& v1, uint64_t& v2, uint64_t& v3) {
  using namespace tc;
  const float sc = bc.sc, k2 = -(2.f * M - 1.f);
  const uint64_t ONE2 = pk2(1.f, 1.f), NEG2 = pk2(-1.f, -1.f), K22 = pk2(k2, k2);
  const uint64_t qq = pk2(basis_q(x, na, bc), basis_q(x, nb, bc));
  const uint64_t q2 = mul2(qq, qq);
  float t0, t1;
  upk2(fma2(q2, NEG2, ONE2), t0, t1);
  t0 = oka ? max_nan(t0, 0.f) : 0.f;
  t1 = okb ? max_nan(t1, 0.f) : 0.f;
  const uint64_t t = pk2(t0, t1);
  uint64_t tm3 = ONE2;
#pragma unroll
  for (int e = 0; e < M - 3; ++e) tm3 = mul2(tm3, t);
  const uint64_t tm2 = mul2(tm3, t), tm1 = mul2(tm2, t);
  v0 = mul2(tm1, t);
  const float c1 = -2.f * M * sc, c2 = c1 * sc, c3 = 4.f * M * (M - 1) * sc * sc * sc;
  v1 = mul2(mul2(qq, tm1), pk2(c1, c1));
  v2 = mul2(mul2(tm2, fma2(q2, K22, ONE2)), pk2(c2, c2));
  v3 = mul2(mul2(mul2(qq, tm3), fma2(q2, K22, pk2(3.f, 3.f))), pk2(c3, c3));
}
enum LastMode { LAST_JET = 0, LAST_POISSON = 1, LAST_BURGERS = 2, LAST_BOUNDARY = 3 };

template <int NF, int NS, int M, int MODE, bool FIRST>
__global__ void __launch_bounds__(32 * LF_WARPS)
    k_last_fused(const float* __restrict__ X, const float* __restrict__ W, const float* __restrict__ bias,
                 int64_t P, int I, BasisCfg bc,
                 float* __restrict__ u_out, float* __restrict__ du_out, float* __restrict__ d2u_out,
                 const float* __restrict__ pts, const float* __restrict__ forcing, const float* __restrict__ gtar,
                 float alpha, float adv, float visc, float inv_n,
                 float* __restrict__ Xbar, float* __restrict__ part) {
  constexpr int C = 1 + NF + NS;
  constexpr int D = (MODE == LAST_POISSON || MODE == LAST_JET) ? NF : 2;
  extern __shared__ float acc_sh[];     // [LF_WARPS][B][I]   (not used by LAST_JET)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = bc.B;
  const int IB = I * B;
  float* acc = acc_sh + (size_t)warp * IB;
  if (MODE != LAST_JET) {
    for (int t = lane; t < IB; t += 32) acc[t] = 0.f;
    __syncwarp();
  }
  const int64_t lo = (P * blockIdx.x) / gridDim.x, hi = (P * (blockIdx.x + 1)) / gridDim.x;
  const float b0 = __ldg(bias);
  float db = 0.f, sq = 0.f, bad = 0.f;
  for (int64_t p = lo + warp; p < hi; p += LF_WARPS) {
    // ---------------- pass 1: output jet
    float s[C];
#pragma unroll
    for (int c = 0; c < C; ++c) s[c] = 0.f;
    for (int i = lane; i < I; i += 32) {
      float x, dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
      load_jet<NF, NS, FIRST>(X, p, i, I, x, dx, ddx);
      if (x != x) s[0] += x;            // propagate NaN inputs into the residual / flag
      const int n0 = first_basis(x, bc);
      float T0 = 0.f, T1 = 0.f, T2 = 0.f;
      if constexpr (HRKAN_LAST_F32X2 && M >= 4) {
        uint64_t P0 = tc::pk2(0.f, 0.f), P1 = P0, P2 = P0;
#pragma unroll
        for (int r = 0; r < KMAX; r += 2) {
          if (r > bc.k) break;
          const int na = n0 + r, nb = na + 1;
          const bool oka = na >= 0 && na < B, okb = r + 1 <= bc.k && nb >= 0 && nb < B;
          uint64_t v0, v1, v2, v3;
          hr_eval_pair<M>(x, na, nb, oka, okb, bc, v0, v1, v2, v3);
          const uint64_t w = tc::pk2(oka ? __ldg(W + i * B + na) : 0.f, okb ? __ldg(W + i * B + nb) : 0.f);
          P0 = tc::fma2(w, v0, P0);
          P1 = tc::fma2(w, v1, P1);
          P2 = tc::fma2(w, v2, P2);
        }
        float lo_, hi_;
        tc::upk2(P0, lo_, hi_); T0 = lo_ + hi_;
        tc::upk2(P1, lo_, hi_); T1 = lo_ + hi_;
        tc::upk2(P2, lo_, hi_); T2 = lo_ + hi_;
      } else {
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        if (r > bc.k) break;
        const int n = n0 + r;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 2 : (NF > 0 ? 1 : 0))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        const float w = __ldg(W + i * B + n);
        T0 = fmaf(w, v0, T0);
        T1 = fmaf(w, v1, T1);
        T2 = fmaf(w, v2, T2);
      }
      }
      s[0] += T0;
#pragma unroll
      for (int a = 0; a < NF; ++a) s[1 + a] = fmaf(T1, dx[a], s[1 + a]);
#pragma unroll
      for (int a = 0; a < NS; ++a) s[1 + NF + a] = fmaf(T2 * dx[a], dx[a], fmaf(T1, ddx[a], s[1 + NF + a]));
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s[c] += __shfl_xor_sync(0xffffffffu, s[c], o);
    }
    s[0] += b0;
    if (MODE == LAST_JET) {
      if (lane == 0) {
        if (u_out) u_out[p] = s[0];
#pragma unroll
        for (int a = 0; a < NF; ++a) {
          if (du_out) du_out[p * NF + a] = s[1 + a];
          if (d2u_out) d2u_out[p * NF + a] = s[1 + NF + a];
        }
      }
      continue;
    }
    // ---------------- residual, loss, seeds (identical in every lane)
    float y[C];
#pragma unroll
    for (int c = 0; c < C; ++c) y[c] = 0.f;
    float r;
    if (MODE == LAST_BOUNDARY) {
      r = s[0] - __ldg(gtar + p);
      y[0] = 2.f * r * inv_n;
    } else if (MODE == LAST_BURGERS) {
      r = s[2] + adv * s[0] * s[1] - visc * s[1 + NF];
      const float g = 2.f * alpha * r * inv_n;
      y[0] = g * adv * s[1];
      y[1] = g * adv * s[0];
      y[2] = g;
      y[1 + NF] = -g * visc;
    } else {
      float f;
      if (forcing) {
        f = __ldg(forcing + p);
      } else {
        float prod = 1.f;
#pragma unroll
        for (int a = 0; a < D; ++a) prod *= sinpif(__ldg(pts + p * D + a));
        f = -(float)D * 9.8696044010893586f * prod;   // -D pi^2 prod_a sin(pi xi_a)
      }
      float lap = 0.f;
#pragma unroll
      for (int a = 0; a < NS; ++a) lap += s[1 + NF + a];
      r = lap - f;
      const float g = 2.f * alpha * r * inv_n;
#pragma unroll
      for (int a = 0; a < NS; ++a) y[1 + NF + a] = g;
    }
    sq = fmaf(r, r, sq);
    bad += isfinite(r) ? 0.f : 1.f;
    db += y[0];
    // ---------------- pass 2: dW and the adjoint of the input jet
    for (int i = lane; i < I; i += 32) {
      float x, dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
      load_jet<NF, NS, FIRST>(X, p, i, I, x, dx, ddx);
      float g1 = 0.f, g2 = 0.f;
#pragma unroll
      for (int a = 0; a < NF; ++a) g1 = fmaf(y[1 + a], dx[a], g1);
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        g1 = fmaf(y[1 + NF + a], ddx[a], g1);
        g2 = fmaf(y[1 + NF + a] * dx[a], dx[a], g2);
      }
      const int n0 = first_basis(x, bc);
      float T1 = 0.f, T2 = 0.f, T3 = 0.f;
#pragma unroll
      for (int rr = 0; rr < KMAX; ++rr) {
        if (rr > bc.k) break;
        const int n = n0 + rr;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 3 : (NF > 0 ? 2 : 1))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        acc[n * I + i] += fmaf(y[0], v0, fmaf(g1, v1, g2 * v2));
        if (!FIRST) {
          const float w = __ldg(W + i * B + n);
          T1 = fmaf(w, v1, T1);
          T2 = fmaf(w, v2, T2);
          T3 = fmaf(w, v3, T3);
        }
      }
      if (!FIRST) {
        float* out = Xbar + p * (int64_t)(C * I) + i;
        out[0] = fmaf(y[0], T1, fmaf(g1, T2, g2 * T3));
#pragma unroll
        for (int a = 0; a < NF; ++a) {
          float v = y[1 + a] * T1;
          if (a < NS) v = fmaf(2.f * y[1 + NF + a] * dx[a], T2, v);
          out[(1 + a) * I] = v;
        }
#pragma unroll
        for (int a = 0; a < NS; ++a) out[(1 + NF + a) * I] = y[1 + NF + a] * T1;
      }
    }
  }
  if (MODE == LAST_JET) return;
  // ---------------- fixed-order block reduction -> part[block][IB + 4]
  __shared__ float red[3][LF_WARPS];
  if (lane == 0) {
    red[0][warp] = db;
    red[1][warp] = sq;
    red[2][warp] = bad;
  }
  __syncthreads();
  float* dst = part + (size_t)blockIdx.x * (IB + 4);
  for (int t = threadIdx.x; t < IB; t += 32 * LF_WARPS) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < LF_WARPS; ++w) v += acc_sh[(size_t)w * IB + t];
    const int n = t / I, i = t - n * I;
    dst[i * B + n] = v;                  // flat W layout [i][n]
  }
  if (threadIdx.x < 3) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < LF_WARPS; ++w) v += red[threadIdx.x][w];
    dst[IB + threadIdx.x] = v;
  }
}

// dW[t] += sum_b part[b][t] (t < IB), db += sum_b part[b][IB], out_loss += scale * sum_b part[b][IB+1],
// out_flag += sum_b part[b][IB+2].  A block of 256 threads takes 32 columns; its 8 warps sum the
// blocks b = g (mod 8) (8 independent chains, coalesced 128-B rows) in double, and warp 0 adds the 8
// chains in order: every sum is in a fixed order (bitwise reproducible for a fixed grid).
constexpr int RL_COLS = 32, RL_CHAINS = 8;
__global__ void __launch_bounds__(RL_COLS * RL_CHAINS)
    k_reduce_last(const float* __restrict__ part, int nb, int IB, float* __restrict__ dW, float* __restrict__ db,
                  float scale, float* __restrict__ out_loss, float* __restrict__ out_flag) {
  __shared__ double sh[RL_CHAINS][RL_COLS];
  const int lane = threadIdx.x & (RL_COLS - 1), g = threadIdx.x / RL_COLS;
  const int t = blockIdx.x * RL_COLS + lane;
  double s = 0.0;
  if (t < IB + 3)
    for (int b = g; b < nb; b += RL_CHAINS) s += (double)__ldg(part + (size_t)b * (IB + 4) + t);
  sh[g][lane] = s;
  __syncthreads();
  if (g == 0 && t < IB + 3) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < RL_CHAINS; ++k) v += sh[k][lane];
    if (t < IB) dW[t] += (float)v;
    else if (t == IB) *db += (float)v;
    else if (t == IB + 1) *out_loss += (float)(v * (double)scale);
    else *out_flag += (float)v;
  }
}

// ---------------------------------------------------------------------------------------------
// Output layer, input-parallel variant (I % 32 == 0, hidden-layer inputs): a block of I/32 warps
// takes a contiguous range of points in batches of LV_PB; warp w owns inputs [32w, 32w+32) (lane =
// input, coalesced 128-B rows of the saved jet), so its share of dW lives in the block's shared
// acc[n][i] columns it alone touches (no atomics; ~I*B*4 bytes per block instead of per warp, which
// keeps ~48-64 warps per SM in flight to hide the jet-load latency).  Per batch:
//   pass 1   per point, warp partial jets over its inputs (butterfly) -> smem part[q][w][c];
//   seeds    thread q < LV_PB sums the warps (fixed order) + bias -> residual, loss, seeds ybar;
//   pass 2   per point, dW contributions and the input-jet adjoint Xbar (same formulas as above).
// ---------------------------------------------------------------------------------------------
constexpr int LV_PB = 4;


// Transposing warp sum of NV values per lane (NV a power of two <= 32): at each step of width h the
// lanes with bit h set keep the upper half of their values and send the lower half (and vice versa),
// so NV - 1 shuffles replace 5*NV; the remaining butterflies (h >= NV) finish the sum.  Afterwards
// lane l holds the warp total of value l % NV.  Fixed order: deterministic.
template <int NV>
__device__ __forceinline__ float warp_sum_transpose(float (&V)[NV], int lane) {
#pragma unroll
  for (int h = NV / 2; h >= 1; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const float send = up ? V[k] : V[k + h];
      const float keep = up ? V[k + h] : V[k];
      V[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  float r = V[0];
#pragma unroll
  for (int h = NV; h < 32; h <<= 1) r += __shfl_xor_sync(0xffffffffu, r, h);
  return r;
}

template <int NF, int NS, int M, int MODE>
__global__ void __launch_bounds__(256, 3)
    k_last_v2(const float* __restrict__ X, const float* __restrict__ W, const float* __restrict__ bias,
              int64_t P, int I, BasisCfg bc,
              float* __restrict__ u_out, float* __restrict__ du_out, float* __restrict__ d2u_out,
              const float* __restrict__ pts, const float* __restrict__ forcing, const float* __restrict__ gtar,
              float alpha, float adv, float visc, float inv_n,
              float* __restrict__ Xbar, float* __restrict__ part, int pbm) {
  constexpr int C = 1 + NF + NS;
  constexpr int D = (MODE == LAST_POISSON || MODE == LAST_JET) ? NF : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;                 // = I / 32
  // pbm <= LV_PB points per batch (host-chosen so that the block's shared memory stays <= 48 KB)
  const int B = bc.B;
  const int IB = I * B;
  extern __shared__ float sm[];
  float* acc = sm;                                // [B][I]           (not used by LAST_JET)
  float* wpart = sm + (MODE == LAST_JET ? 0 : IB);   // [LV_PB][nw][C]
  float* ys = wpart + LV_PB * nw * C;             // [LV_PB][C]
  float* jsm = ys + LV_PB * C;                    // [nw][pbm][C][32]   this batch's jets
  __shared__ float red[3][LV_PB];
  if (MODE != LAST_JET)
    for (int t = threadIdx.x; t < IB; t += blockDim.x) acc[t] = 0.f;
  const int64_t lo = (P * blockIdx.x) / gridDim.x, hi = (P * (blockIdx.x + 1)) / gridDim.x;
  const int i = warp * 32 + lane;
  float* jw = jsm + warp * (pbm * C * 32) + lane;
  float db = 0.f, sq = 0.f, bad = 0.f;            // thread q < LV_PB accumulates its batch slot
  for (int64_t p0 = lo; p0 < hi; p0 += pbm) {
    const int npb = (int)((hi - p0) < pbm ? (hi - p0) : pbm);
    __syncthreads();                              // previous batch's seeds and jets consumed
    // ---------------- stage this batch's jets (all loads in flight together), then pass 1
    {
      float v[LV_PB][C];
#pragma unroll
      for (int q = 0; q < LV_PB; ++q) {
        const float* base = X + (p0 + q) * (int64_t)(C * I) + i;
#pragma unroll
        for (int c = 0; c < C; ++c) v[q][c] = (q < npb) ? __ldg(base + c * I) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < LV_PB; ++q)
        if (q < npb) {
#pragma unroll
          for (int c = 0; c < C; ++c) jw[(q * C + c) * 32] = v[q][c];
        }
    }
    // pass 1: the warp's partial jets of all batch points, then ONE transposing butterfly over the
    // LV_PB*C values (log2 NV exchange steps of halving width instead of 5 per value)
    constexpr int NVT = LV_PB * C;
    constexpr int NV = NVT <= 4 ? 4 : NVT <= 8 ? 8 : NVT <= 16 ? 16 : 32;
    static_assert(NVT <= 32, "batch x channels must fit one warp");
    float V[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) V[k] = 0.f;
#pragma unroll
    for (int q = 0; q < LV_PB; ++q) {
      if (q >= npb) break;
      const float* jq = jw + q * C * 32;
      const float x = jq[0];
      float s[C];
#pragma unroll
      for (int c = 0; c < C; ++c) s[c] = 0.f;
      if (x != x) s[0] = x;
      const int n0 = first_basis(x, bc);
      float T0 = 0.f, T1 = 0.f, T2 = 0.f;
      if constexpr (HRKAN_LAST_F32X2 && M >= 4) {
        uint64_t P0 = tc::pk2(0.f, 0.f), P1 = P0, P2 = P0;
#pragma unroll
        for (int r = 0; r < KMAX; r += 2) {
          if (r > bc.k) break;
          const int na = n0 + r, nb = na + 1;
          const bool oka = na >= 0 && na < B, okb = r + 1 <= bc.k && nb >= 0 && nb < B;
          uint64_t v0, v1, v2, v3;
          hr_eval_pair<M>(x, na, nb, oka, okb, bc, v0, v1, v2, v3);
          const uint64_t w = tc::pk2(oka ? __ldg(W + i * B + na) : 0.f, okb ? __ldg(W + i * B + nb) : 0.f);
          P0 = tc::fma2(w, v0, P0);
          P1 = tc::fma2(w, v1, P1);
          P2 = tc::fma2(w, v2, P2);
        }
        float lo_, hi_;
        tc::upk2(P0, lo_, hi_); T0 = lo_ + hi_;
        tc::upk2(P1, lo_, hi_); T1 = lo_ + hi_;
        tc::upk2(P2, lo_, hi_); T2 = lo_ + hi_;
      } else {
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        if (r > bc.k) break;
        const int n = n0 + r;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 2 : (NF > 0 ? 1 : 0))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        const float w = __ldg(W + i * B + n);
        T0 = fmaf(w, v0, T0);
        T1 = fmaf(w, v1, T1);
        T2 = fmaf(w, v2, T2);
      }
      }
      s[0] += T0;
#pragma unroll
      for (int a = 0; a < NF; ++a) s[1 + a] = T1 * jq[(1 + a) * 32];
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        const float d1 = jq[(1 + a) * 32], d2 = jq[(1 + NF + a) * 32];
        s[1 + NF + a] = fmaf(T2 * d1, d1, T1 * d2);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) V[q * C + c] = s[c];
    }
    {
      const float tot = warp_sum_transpose<NV>(V, lane);   // lane l: warp total of value l % NV
      if (lane < NVT && lane / C < npb) wpart[((lane / C) * nw + warp) * C + lane % C] = tot;
    }
    __syncthreads();
    // ---------------- totals, residual, loss, seeds (thread q per point)
    if (threadIdx.x < npb) {
      const int q = threadIdx.x;
      const int64_t p = p0 + q;
      float s[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float v = 0.f;
        for (int w = 0; w < nw; ++w) v += wpart[(q * nw + w) * C + c];
        s[c] = v;
      }
      s[0] += __ldg(bias);
      if (MODE == LAST_JET) {
        if (u_out) u_out[p] = s[0];
#pragma unroll
        for (int a = 0; a < NF; ++a) {
          if (du_out) du_out[p * NF + a] = s[1 + a];
          if (d2u_out) d2u_out[p * NF + a] = s[1 + NF + a];
        }
      } else {
        float y[C];
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = 0.f;
        float r;
        if (MODE == LAST_BOUNDARY) {
          r = s[0] - __ldg(gtar + p);
          y[0] = 2.f * r * inv_n;
        } else if (MODE == LAST_BURGERS) {
          r = s[2] + adv * s[0] * s[1] - visc * s[1 + NF];
          const float g = 2.f * alpha * r * inv_n;
          y[0] = g * adv * s[1];
          y[1] = g * adv * s[0];
          y[2] = g;
          y[1 + NF] = -g * visc;
        } else {
          float f;
          if (forcing) {
            f = __ldg(forcing + p);
          } else {
            float prod = 1.f;
#pragma unroll
            for (int a = 0; a < D; ++a) prod *= sinpif(__ldg(pts + p * D + a));
            f = -(float)D * 9.8696044010893586f * prod;   // -D pi^2 prod_a sin(pi xi_a)
          }
          float lap = 0.f;
#pragma unroll
          for (int a = 0; a < NS; ++a) lap += s[1 + NF + a];
          r = lap - f;
          const float g = 2.f * alpha * r * inv_n;
#pragma unroll
          for (int a = 0; a < NS; ++a) y[1 + NF + a] = g;
        }
        sq = fmaf(r, r, sq);
        bad += isfinite(r) ? 0.f : 1.f;
        db += y[0];
#pragma unroll
        for (int c = 0; c < C; ++c) ys[q * C + c] = y[c];
      }
    }
    if (MODE == LAST_JET) continue;
    __syncthreads();
    // ---------------- pass 2: dW and the adjoint of the input jet (jets from shared memory)
#pragma unroll 1
    for (int q = 0; q < npb; ++q) {
      const int64_t p = p0 + q;
      const float* jq = jw + q * C * 32;
      float y[C];
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = ys[q * C + c];
      const float x = jq[0];
      float dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
#pragma unroll
      for (int a = 0; a < NF; ++a) dx[a] = jq[(1 + a) * 32];
#pragma unroll
      for (int a = 0; a < NS; ++a) ddx[a] = jq[(1 + NF + a) * 32];
      float g1 = 0.f, g2 = 0.f;
#pragma unroll
      for (int a = 0; a < NF; ++a) g1 = fmaf(y[1 + a], dx[a], g1);
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        g1 = fmaf(y[1 + NF + a], ddx[a], g1);
        g2 = fmaf(y[1 + NF + a] * dx[a], dx[a], g2);
      }
      const int n0 = first_basis(x, bc);
      float T1 = 0.f, T2 = 0.f, T3 = 0.f;
      if constexpr (HRKAN_LAST_F32X2 && M >= 4) {
        const uint64_t Y0 = tc::pk2(y[0], y[0]), G1 = tc::pk2(g1, g1), G2 = tc::pk2(g2, g2);
        uint64_t P1 = tc::pk2(0.f, 0.f), P2 = P1, P3 = P1;
#pragma unroll
        for (int rr = 0; rr < KMAX; rr += 2) {
          if (rr > bc.k) break;
          const int na = n0 + rr, nb = na + 1;
          const bool oka = na >= 0 && na < B, okb = rr + 1 <= bc.k && nb >= 0 && nb < B;
          uint64_t v0, v1, v2, v3;
          hr_eval_pair<M>(x, na, nb, oka, okb, bc, v0, v1, v2, v3);
          float ca, cb;
          tc::upk2(tc::fma2(Y0, v0, tc::fma2(G1, v1, tc::mul2(G2, v2))), ca, cb);
          if (oka) acc[na * I + i] += ca;
          if (okb) acc[nb * I + i] += cb;
          const uint64_t w = tc::pk2(oka ? __ldg(W + i * B + na) : 0.f, okb ? __ldg(W + i * B + nb) : 0.f);
          P1 = tc::fma2(w, v1, P1);
          P2 = tc::fma2(w, v2, P2);
          P3 = tc::fma2(w, v3, P3);
        }
        float lo_, hi_;
        tc::upk2(P1, lo_, hi_); T1 = lo_ + hi_;
        tc::upk2(P2, lo_, hi_); T2 = lo_ + hi_;
        tc::upk2(P3, lo_, hi_); T3 = lo_ + hi_;
      } else {
#pragma unroll
      for (int rr = 0; rr < KMAX; ++rr) {
        if (rr > bc.k) break;
        const int n = n0 + rr;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 3 : (NF > 0 ? 2 : 1))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        acc[n * I + i] += fmaf(y[0], v0, fmaf(g1, v1, g2 * v2));
        const float w = __ldg(W + i * B + n);
        T1 = fmaf(w, v1, T1);
        T2 = fmaf(w, v2, T2);
        T3 = fmaf(w, v3, T3);
      }
      }
      float* out = Xbar + p * (int64_t)(C * I) + i;
      out[0] = fmaf(y[0], T1, fmaf(g1, T2, g2 * T3));
#pragma unroll
      for (int a = 0; a < NF; ++a) {
        float v = y[1 + a] * T1;
        if (a < NS) v = fmaf(2.f * y[1 + NF + a] * dx[a], T2, v);
        out[(1 + a) * I] = v;
      }
#pragma unroll
      for (int a = 0; a < NS; ++a) out[(1 + NF + a) * I] = y[1 + NF + a] * T1;
    }
  }
  if (MODE == LAST_JET) return;
  // ---------------- fixed-order block reduction -> part[block][IB + 4]
  if (threadIdx.x < LV_PB) {
    red[0][threadIdx.x] = db;
    red[1][threadIdx.x] = sq;
    red[2][threadIdx.x] = bad;
  }
  __syncthreads();
  float* dst = part + (size_t)blockIdx.x * (IB + 4);
  for (int t = threadIdx.x; t < IB; t += blockDim.x) {
    const int n = t / I, ii = t - n * I;
    dst[ii * B + n] = acc[t];                     // flat W layout [i][n]
  }
  if (threadIdx.x < 3) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < LV_PB; ++q) v += red[threadIdx.x][q];
    dst[IB + threadIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------------------------
// Output layer, input-parallel, loss modes only (k <= 3, I % 32 == 0): the v2 algorithm with
//   * the batch's jets [PB points][C][I] fetched by ONE 1-D bulk copy into a 2-stage shared-memory
//     ring (batch b+2 is in flight while b is processed: no per-thread load latency, no staging STS),
//   * the basis values v, v', v'' of the k+1 candidates and T1..T3 = sum_n w_n v_n^(1..3) computed
//     once in pass 1 and kept in registers for pass 2 (v2 re-evaluated the basis and reloaded W),
//   * W and the dW accumulator in shared memory with KT-1 zero rows on each side of the B bases, so
//     the KT candidate rows are read / updated without predicates.
// Same arithmetic and reduction order as k_last_v2 (fixed order: deterministic).
// ---------------------------------------------------------------------------------------------
constexpr int LV3_PB = 4;    // points per batch
constexpr int LV3_KT = 4;    // candidate bases per x (k + 1 <= 4)

__host__ __device__ constexpr int lv3_bp(int B) { return (B + 2 * (LV3_KT - 1)) | 1; }   // odd: conflict-free rows

// SPLIT: the adjoint of the input jet is not written in fp32; instead the block emits the bf16 hi/lo
// operand stages of the preceding tensor-core layer's reverse kernels (k_split_ybar's YW / YD layouts,
// see tc_kernels.cuh) and that layer's bias-gradient partials part_bias[block][I] -- the fp32 adjoint
// never goes to HBM and the separate split pass disappears.  Block point ranges are multiples of 8
// (YW's 8-point blocks: a batch of PB = 4 points is one half of one block).
template <int NF, int NS, int M, int MODE, bool SPLIT>
__global__ void __launch_bounds__(256, 2)
    k_last_v3(const float* __restrict__ X, const float* __restrict__ W, const float* __restrict__ bias, int64_t P,
              int I, BasisCfg bc, const float* __restrict__ pts, const float* __restrict__ forcing,
              const float* __restrict__ gtar, float alpha, float adv, float visc, float inv_n, float* __restrict__ Xbar,
              float* __restrict__ part, uint16_t* __restrict__ YW, uint16_t* __restrict__ YD,
              float* __restrict__ part_bias) {
  constexpr int C = 1 + NF + NS;
  constexpr int D = (MODE == LAST_POISSON) ? NF : 2;
  constexpr int PB = LV3_PB, KT = LV3_KT, KO = KT - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;                 // = I / 32
  const int i = threadIdx.x;
  const int B = bc.B, BP = lv3_bp(B);
  extern __shared__ __align__(16) float sm3[];
  const int STG = PB * C * (I + 4);               // stage floats: jets [PB][C][I], or (SPLIT) the adjoint [PB*C][I+4]
  float* jst = sm3;                               // [2][STG] jet stages (bulk copies)
  float* Ws = jst + 2 * STG;                      // [I][BP]   W[0][i][n] at column KO + n
  float* acc = Ws + I * BP;                       // [BP][I]   dW rows KO + n
  float* wpart = acc + BP * I;                    // [PB][nw][C]
  float* ys = wpart + PB * nw * C;                // [PB][C]
  __shared__ __align__(8) uint64_t full[2];
  __shared__ float red[3][PB];
  for (int t = threadIdx.x; t < I * BP; t += blockDim.x) {
    const int ii = t / BP, n = t - ii * BP - KO;
    Ws[t] = (n >= 0 && n < B) ? __ldg(W + ii * B + n) : 0.f;
    acc[t] = 0.f;
  }
  const int64_t nb8 = (P + 7) / 8;                // 8-point blocks (block ranges are whole blocks)
  const int64_t lo = 8 * ((nb8 * blockIdx.x) / gridDim.x);
  const int64_t hi = min(P, 8 * ((nb8 * (blockIdx.x + 1)) / gridDim.x));
  const int nbat = (int)((hi - lo + PB - 1) / PB);
  const uint32_t row_bytes = (uint32_t)(C * I * 4);
  auto issue = [&](int b) {                       // thread 0: batch b -> stage b & 1
    const int64_t p0 = lo + (int64_t)b * PB;
    const int npb = (int)((hi - p0) < PB ? (hi - p0) : PB);
    tc::mbar_arrive_expect_tx(&full[b & 1], row_bytes * npb);
    tc::bulk_g2s(jst + (b & 1) * STG, X + p0 * (int64_t)(C * I), row_bytes * npb, &full[b & 1]);
  };
  if (threadIdx.x == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_mbar_init();
    if (nbat > 0) issue(0);
    if (nbat > 1) issue(1);
  }
  __syncthreads();
  const float b0 = __ldg(bias);
  const float sc = bc.sc;
  float db = 0.f, sq = 0.f, bad = 0.f;            // thread q < PB accumulates its batch slot
  float dbi = 0.f;                                // SPLIT: bias gradient of the preceding layer, output i
  for (int b = 0; b < nbat; ++b) {
    const int64_t p0 = lo + (int64_t)b * PB;
    const int npb = (int)((hi - p0) < PB ? (hi - p0) : PB);
    const float* J = jst + (b & 1) * STG + i;
    tc::mbar_wait(&full[b & 1], (uint32_t)((b >> 1) & 1));
    // ---------------- pass 1: output-jet partials; cache the candidate basis values and T1..T3
    constexpr int NVT = PB * C;
    constexpr int NV = NVT <= 4 ? 4 : NVT <= 8 ? 8 : NVT <= 16 ? 16 : 32;
    static_assert(NVT <= 32, "batch x channels must fit one warp");
    float V[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) V[k] = 0.f;
    float cv[PB][3][KT], cT[PB][3];
    int cn[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      cn[q] = 0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        cT[q][d] = 0.f;
#pragma unroll
        for (int r = 0; r < KT; ++r) cv[q][d][r] = 0.f;
      }
      if (q >= npb) continue;
      const float* jq = J + q * C * I;
      const float x = jq[0];
      const int n0 = first_basis(x, bc);
      uint64_t P0 = 0ull, P1 = 0ull, P2 = 0ull, P3 = 0ull;
#pragma unroll
      for (int r = 0; r < KT; r += 2) {
        const int na = n0 + r, nb = na + 1;
        const bool oka = r <= bc.k && na >= 0 && na < B, okb = r + 1 <= bc.k && nb >= 0 && nb < B;
        uint64_t v0, v1, v2, v3;
        hr_eval_pair<M>(x, na, nb, oka, okb, bc, v0, v1, v2, v3);
        tc::upk2(v0, cv[q][0][r], cv[q][0][r + 1]);
        tc::upk2(v1, cv[q][1][r], cv[q][1][r + 1]);
        tc::upk2(v2, cv[q][2][r], cv[q][2][r + 1]);
        // W rows of the candidates (zero rows outside [0, B)); n0 clamped below keeps them in range
        const int nc = min(max(n0, -KO), B - 1);
        const float* wr = Ws + i * BP + KO + nc + r;
        const uint64_t w = tc::pk2((n0 == nc) ? wr[0] : 0.f, (n0 == nc) ? wr[1] : 0.f);
        P0 = tc::fma2(w, v0, P0);
        P1 = tc::fma2(w, v1, P1);
        P2 = tc::fma2(w, v2, P2);
        P3 = tc::fma2(w, v3, P3);
      }
      cn[q] = min(max(n0, -KO), B - 1);           // all candidates zero when n0 was clamped
      float lo_, hi_, T0;
      tc::upk2(P0, lo_, hi_); T0 = lo_ + hi_;
      tc::upk2(P1, lo_, hi_); cT[q][0] = lo_ + hi_;
      tc::upk2(P2, lo_, hi_); cT[q][1] = lo_ + hi_;
      tc::upk2(P3, lo_, hi_); cT[q][2] = lo_ + hi_;
      float s[C];
      s[0] = (x != x) ? x : T0;                   // propagate NaN inputs into the residual / flag
#pragma unroll
      for (int a = 0; a < NF; ++a) s[1 + a] = cT[q][0] * jq[(1 + a) * I];
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        const float d1 = jq[(1 + a) * I], d2 = jq[(1 + NF + a) * I];
        s[1 + NF + a] = fmaf(cT[q][1] * d1, d1, cT[q][0] * d2);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) V[q * C + c] = s[c];
    }
    {
      const float tot = warp_sum_transpose<NV>(V, lane);   // lane l: warp total of value l % NV
      if (lane < NVT && lane / C < npb) wpart[((lane / C) * nw + warp) * C + lane % C] = tot;
    }
    __syncthreads();
    // ---------------- totals, residual, loss, seeds (thread q per point)
    if (threadIdx.x < npb) {
      const int q = threadIdx.x;
      const int64_t p = p0 + q;
      float s[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float v = 0.f;
        for (int w = 0; w < nw; ++w) v += wpart[(q * nw + w) * C + c];
        s[c] = v;
      }
      s[0] += b0;
      float y[C];
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = 0.f;
      float r;
      if (MODE == LAST_BOUNDARY) {
        r = s[0] - __ldg(gtar + p);
        y[0] = 2.f * r * inv_n;
      } else if (MODE == LAST_BURGERS) {
        r = s[2] + adv * s[0] * s[1] - visc * s[1 + NF];
        const float g = 2.f * alpha * r * inv_n;
        y[0] = g * adv * s[1];
        y[1] = g * adv * s[0];
        y[2] = g;
        y[1 + NF] = -g * visc;
      } else {
        float f;
        if (forcing) {
          f = __ldg(forcing + p);
        } else {
          float prod = 1.f;
#pragma unroll
          for (int a = 0; a < D; ++a) prod *= sinpif(__ldg(pts + p * D + a));
          f = -(float)D * 9.8696044010893586f * prod;   // -D pi^2 prod_a sin(pi xi_a)
        }
        float lap = 0.f;
#pragma unroll
        for (int a = 0; a < NS; ++a) lap += s[1 + NF + a];
        r = lap - f;
        const float g = 2.f * alpha * r * inv_n;
#pragma unroll
        for (int a = 0; a < NS; ++a) y[1 + NF + a] = g;
      }
      sq = fmaf(r, r, sq);
      bad += isfinite(r) ? 0.f : 1.f;
      db += y[0];
#pragma unroll
      for (int c = 0; c < C; ++c) ys[q * C + c] = y[c];
    }
    __syncthreads();
    // ---------------- pass 2: dW and the adjoint of the input jet, from the cached values
    float ov[PB][C];                              // (SPLIT) this thread's adjoint values of the batch
#pragma unroll
    for (int q = 0; q < PB; ++q)
#pragma unroll
      for (int c = 0; c < C; ++c) ov[q][c] = 0.f;
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      if (q >= npb) break;
      const int64_t p = p0 + q;
      const float* jq = J + q * C * I;
      float y[C];
#pragma unroll
      for (int c = 0; c < C; ++c) y[c] = ys[q * C + c];
      float dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
#pragma unroll
      for (int a = 0; a < NF; ++a) dx[a] = jq[(1 + a) * I];
#pragma unroll
      for (int a = 0; a < NS; ++a) ddx[a] = jq[(1 + NF + a) * I];
      float g1 = 0.f, g2 = 0.f;
#pragma unroll
      for (int a = 0; a < NF; ++a) g1 = fmaf(y[1 + a], dx[a], g1);
#pragma unroll
      for (int a = 0; a < NS; ++a) {
        g1 = fmaf(y[1 + NF + a], ddx[a], g1);
        g2 = fmaf(y[1 + NF + a] * dx[a], dx[a], g2);
      }
      float* ar = acc + (KO + cn[q]) * I + i;
#pragma unroll
      for (int r = 0; r < KT; ++r) ar[r * I] += fmaf(y[0], cv[q][0][r], fmaf(g1, cv[q][1][r], g2 * cv[q][2][r]));
      const float T1 = cT[q][0], T2 = cT[q][1], T3 = cT[q][2];
      ov[q][0] = fmaf(y[0], T1, fmaf(g1, T2, g2 * T3));
#pragma unroll
      for (int a = 0; a < NF; ++a) {
        float v = y[1 + a] * T1;
        if (a < NS) v = fmaf(2.f * y[1 + NF + a] * dx[a], T2, v);
        ov[q][1 + a] = v;
      }
#pragma unroll
      for (int a = 0; a < NS; ++a) ov[q][1 + NF + a] = y[1 + NF + a] * T1;
      if constexpr (!SPLIT) {
        float* out = Xbar + p * (int64_t)(C * I) + i;
#pragma unroll
        for (int c = 0; c < C; ++c) out[c * I] = ov[q][c];
      }
    }
    __syncthreads();                              // stage b & 1 fully read
    if constexpr (SPLIT) {
      // the adjoint of the batch -> stage (rows q*C + c, stride I + 4), then the bf16 hi/lo operand stages
      constexpr int NP = tc_np(C), N = NP * C;
      float* xs = jst + (b & 1) * STG;
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        dbi += ov[q][0];
#pragma unroll
        for (int c = 0; c < C; ++c) xs[(q * C + c) * (I + 4) + i] = ov[q][c];
      }
      __syncthreads();
      // YW (wgrad B operand): chunk z = block*C + c of 8 points; this batch is half (p0 / 4) & 1
      const int64_t b8 = p0 >> 3;
      const int half = (int)((p0 >> 2) & 1);
      for (int t = threadIdx.x; t < C * I; t += blockDim.x) {
        const int c = t / I, o = t - c * I;
        const float4 v = make_float4(xs[c * (I + 4) + o], xs[(C + c) * (I + 4) + o], xs[(2 * C + c) * (I + 4) + o],
                                     xs[(3 * C + c) * (I + 4) + o]);
        uint2 h, l;
        tc::split4_bf16(v, h, l);
        const int64_t z = b8 * C + c;
        uint16_t* dst = YW + (z >> 1) * (int64_t)(4 * I * 8) + ((z & 1) * I + o) * 8 + half * 4;
        *reinterpret_cast<uint2*>(dst) = h;
        *reinterpret_cast<uint2*>(dst + 2 * I * 8) = l;
      }
      // YD (dgrad B operand): row p*C + c of the point tile, 8 consecutive outputs per 16 B
      const int64_t tile = p0 / NP;
      const int row0 = (int)(p0 - tile * NP) * C;
      const int nkb = I / 16;
      for (int t = threadIdx.x; t < PB * C * (I / 8); t += blockDim.x) {
        const int rw = t % (PB * C), og = t / (PB * C);
        const float4* sp = reinterpret_cast<const float4*>(xs + rw * (I + 4) + og * 8);
        const float4 a0 = sp[0], a1 = sp[1];
        float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        uint4 h, l;
        tc::split8_bf16(v, h, l);
        uint16_t* dst = YD + (tile * nkb + og / 2) * (int64_t)(4 * N * 8) + ((og & 1) * N + row0 + rw) * 8;
        *reinterpret_cast<uint4*>(dst) = h;
        *reinterpret_cast<uint4*>(dst + 2 * N * 8) = l;
      }
      __syncthreads();                            // stage read by the emitters
    }
    if (threadIdx.x == 0 && b + 2 < nbat) {
      tc::fence_proxy_async_smem();               // generic reads of the stage before the async-proxy refill
      issue(b + 2);
    }
  }
  if constexpr (SPLIT) {
    part_bias[(int64_t)blockIdx.x * I + i] = dbi;
    if (hi == P && lo < P) {                      // the block holding the last point: YW tails
      const int rem = (int)(P & 7);
      if (rem >= 1 && rem <= 4) {                 // last 8-point block: its second half has no batch
        for (int t = threadIdx.x; t < C * I; t += blockDim.x) {
          const int c = t / I, o = t - c * I;
          const int64_t z = (nb8 - 1) * C + c;
          uint16_t* dst = YW + (z >> 1) * (int64_t)(4 * I * 8) + ((z & 1) * I + o) * 8 + 4;
          *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
          *reinterpret_cast<uint2*>(dst + 2 * I * 8) = make_uint2(0u, 0u);
        }
      }
      if ((nb8 * C) & 1) {                        // odd chunk total: zero the final half-stage
        const int64_t z = nb8 * C;
        for (int o = threadIdx.x; o < I; o += blockDim.x) {
          uint16_t* dst = YW + (z >> 1) * (int64_t)(4 * I * 8) + (I + o) * 8;
          *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(dst + 2 * I * 8) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
  }
  // ---------------- fixed-order block reduction -> part[block][IB + 4]
  if (threadIdx.x < PB) {
    red[0][threadIdx.x] = db;
    red[1][threadIdx.x] = sq;
    red[2][threadIdx.x] = bad;
  }
  __syncthreads();
  float* dst = part + (size_t)blockIdx.x * (I * B + 4);
  for (int t = threadIdx.x; t < I * B; t += blockDim.x) {
    const int ii = t / B, n = t - ii * B;
    dst[t] = acc[(KO + n) * I + ii];              // flat W layout [i][n]
  }
  if (threadIdx.x < 3) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < PB; ++q) v += red[threadIdx.x][q];
    dst[I * B + threadIdx.x] = v;
  }
}

}  // namespace
