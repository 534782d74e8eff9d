// tiny_kernels.cuh -- the whole PINN loss + gradient of a TINY HRKAN (every width <= TINY_W, at most
// TINY_L layers: the paper's own [2,2,1] / [2,3,3,3,1]-class nets and BASELINE's C1 [2,5,1], C2
// [2,5,5,1]) in ONE kernel launch, plus one fixed-order reduction launch.
//
// One thread per collocation point; the parameters live in shared memory; every layer's input jet
// stays in the thread (local memory); the forward jet, residual, seeds and the whole reverse pass are
// the formulas of the layered kernels (Eq. 2, Eq. 3-4, Eq. 5-8
// P:195-236), band-limited to the k+1 bases that are non-zero at each x.  Gradients are reduced
// deterministically: per parameter a warp butterfly (all lanes see the same parameter index; lanes
// whose band misses it add 0), per-warp slots in shared memory, a fixed-order block sum into
// part[block][np + 4], summed over the blocks in order by the last block to finish.  Blocks [0, nb_int) take interior points,
// the rest boundary then initial points (value-only, C = 1), so a block never mixes modes.
#pragma once

namespace {   // internal linkage: every translation unit owns its kernels
using namespace hrkan;

constexpr int TINY_W = 8;           // max layer width
constexpr int TINY_L = 4;           // max number of layers
constexpr int TINY_THREADS = 128;   // 4 warps per block
constexpr int TINY_MAXP = 2048;     // max parameters (shared memory slots per warp)

struct TinyNet {
  int L, B, np;
  int w[TINY_L + 1];
  int woff[TINY_L], boff[TINY_L];
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One point through the whole net: forward jet, residual/loss, seeds, reverse pass.  Gradient
// contributions are warp-reduced into gw[np] (this warp's shared slot); sq / bad accumulate in lane 0.
// MODE: LAST_POISSON / LAST_BURGERS (interior, NF/NS channels) or LAST_BOUNDARY (NF = NS = 0).
template <int NF, int NS, int M, int MODE>
__device__ __forceinline__ void tiny_point(const TinyNet& tn, const float* __restrict__ prm, const BasisCfg& bc,
                                           bool valid, const float* __restrict__ pt, int D, float aux,
                                           float alpha, float adv, float visc, float inv_n, float* __restrict__ gw,
                                           float& sq, float& bad) {
  constexpr int C = 1 + NF + NS;
  const int lane = threadIdx.x & 31;
  const int B = tn.B;
  float xs[TINY_L][TINY_W][C];          // layer-input jets (layer 0 holds the raw coordinates)
  float y[TINY_W][C];
  // ---------------- layer-0 input jet: x_a = xi_a, dx_{a,a'} = delta, ddx = 0
  for (int a = 0; a < D; ++a) {
    xs[0][a][0] = valid ? pt[a] : 0.f;
#pragma unroll
    for (int c = 1; c < C; ++c) xs[0][a][c] = (c >= 1 && c <= NF && c - 1 == a) ? 1.f : 0.f;
  }
  // ---------------- forward
  for (int l = 0; l < tn.L; ++l) {
    const int I = tn.w[l], O = tn.w[l + 1];
    const float* W = prm + tn.woff[l];
    for (int o = 0; o < O; ++o) {
      y[o][0] = prm[tn.boff[l] + o];
#pragma unroll
      for (int c = 1; c < C; ++c) y[o][c] = 0.f;
    }
    for (int i = 0; i < I; ++i) {
      const float x = xs[l][i][0];
      const int n0 = first_basis(x, bc);
#pragma unroll
      for (int r = 0; r < KMAX; ++r) {
        if (r > bc.k) break;
        const int n = n0 + r;
        if (n < 0 || n >= B) continue;
        float v0, v1, v2, v3;
        hr_eval<M, (NS > 0 ? 2 : (NF > 0 ? 1 : 0))>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        float A[C];
        A[0] = v0;
#pragma unroll
        for (int a = 0; a < NF; ++a) A[1 + a] = v1 * xs[l][i][1 + a];
#pragma unroll
        for (int a = 0; a < NS; ++a) A[1 + NF + a] = fmaf(v2 * xs[l][i][1 + a], xs[l][i][1 + a], v1 * xs[l][i][1 + NF + a]);
        for (int o = 0; o < O; ++o) {
          const float w = W[(o * I + i) * B + n];
#pragma unroll
          for (int c = 0; c < C; ++c) y[o][c] = fmaf(w, A[c], y[o][c]);
        }
      }
      if (x != x) y[0][0] += x;          // propagate NaN inputs into the residual / flag
    }
    if (l + 1 < tn.L)
      for (int o = 0; o < O; ++o)
#pragma unroll
        for (int c = 0; c < C; ++c) xs[l + 1][o][c] = y[o][c];
  }
  // ---------------- residual, loss, seeds (output layer has one neuron: y[0][.])
  float yb[TINY_W][C];
#pragma unroll
  for (int c = 0; c < C; ++c) yb[0][c] = 0.f;
  float r = 0.f;
  if (MODE == LAST_BOUNDARY) {
    r = y[0][0] - aux;
    yb[0][0] = 2.f * r * inv_n;
  } else if (MODE == LAST_BURGERS) {
    r = y[0][2] + adv * y[0][0] * y[0][1] - visc * y[0][1 + NF];
    const float g = 2.f * alpha * r * inv_n;
    yb[0][0] = g * adv * y[0][1];
    yb[0][1] = g * adv * y[0][0];
    yb[0][2] = g;
    yb[0][1 + NF] = -g * visc;
  } else {
    float lap = 0.f;
#pragma unroll
    for (int a = 0; a < NS; ++a) lap += y[0][1 + NF + a];
    r = lap - aux;                        // aux = f (forcing)
    const float g = 2.f * alpha * r * inv_n;
#pragma unroll
    for (int a = 0; a < NS; ++a) yb[0][1 + NF + a] = g;
  }
  if (!valid) {
    r = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) yb[0][c] = 0.f;
  }
  const float sqw = warp_sum(r * r), badw = warp_sum((valid && !isfinite(r)) ? 1.f : 0.f);
  if (lane == 0) {
    sq += sqw;
    bad += badw;
  }
  // ---------------- reverse, last layer to first
  for (int l = tn.L - 1; l >= 0; --l) {
    const int I = tn.w[l], O = tn.w[l + 1];
    const float* W = prm + tn.woff[l];
    for (int o = 0; o < O; ++o) {
      const float db = warp_sum(yb[o][0]);
      if (lane == 0) gw[tn.boff[l] + o] += db;
    }
    float xb[TINY_W][C];
    for (int i = 0; i < I; ++i) {
      const float x = xs[l][i][0];
      const int n0 = first_basis(x, bc);
      float vv[4][KMAX];
#pragma unroll
      for (int rr = 0; rr < KMAX; ++rr) {
        const int n = n0 + rr;
        vv[0][rr] = vv[1][rr] = vv[2][rr] = vv[3][rr] = 0.f;
        if (rr <= bc.k && n >= 0 && n < B)
          hr_eval<M, (NS > 0 ? 3 : (NF > 0 ? 2 : 1))>(basis_q(x, n, bc), bc.sc, vv[0][rr], vv[1][rr], vv[2][rr],
                                                    vv[3][rr]);
      }
      const float* dx = &xs[l][i][1];
      float S1 = 0.f, S2 = 0.f, S3 = 0.f;     // sum_{o,n} W yb-weighted derivative terms for xbar
      float dxb[NF > 0 ? NF : 1], ddxb[NS > 0 ? NS : 1];
#pragma unroll
      for (int a = 0; a < NF; ++a) dxb[a] = 0.f;
#pragma unroll
      for (int a = 0; a < NS; ++a) ddxb[a] = 0.f;
      for (int o = 0; o < O; ++o) {
        // fold the seeds with the jet: sum_c yb_c A^c = y0 v + g1 v' + g2 v''
        float g1 = 0.f, g2 = 0.f;
#pragma unroll
        for (int a = 0; a < NF; ++a) g1 = fmaf(yb[o][1 + a], dx[a], g1);
#pragma unroll
        for (int a = 0; a < NS; ++a) {
          g1 = fmaf(yb[o][1 + NF + a], dx[NF + a], g1);
          g2 = fmaf(yb[o][1 + NF + a] * dx[a], dx[a], g2);
        }
        float T1 = 0.f, T2 = 0.f, T3 = 0.f;
        // dW[o, i, n] for every n: the lane's k+1 band contributions placed at n0 + rr, then ONE
        // transposing butterfly over the B (<= 16) values -- lane n ends with the warp total of basis n
        float cr[KMAX];
#pragma unroll
        for (int rr = 0; rr < KMAX; ++rr) cr[rr] = fmaf(yb[o][0], vv[0][rr], fmaf(g1, vv[1][rr], g2 * vv[2][rr]));
        float* gdst = gw + tn.woff[l] + (o * I + i) * B;
        if (B <= 8) {
          float V[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float v = 0.f;
            if (bc.k == 3) {                     // the paper's / BASELINE's k: 4 candidates, not KMAX
#pragma unroll
              for (int rr = 0; rr < 4; ++rr) v = (q - rr == n0) ? cr[rr] : v;
            } else {
#pragma unroll
              for (int rr = 0; rr < KMAX; ++rr) v = (rr <= bc.k && q - rr == n0) ? cr[rr] : v;
            }
            V[q] = v;
          }
          const float tot = warp_sum_transpose<8>(V, lane);
          if (lane < B) gdst[lane] += tot;
        } else if (B <= 16) {
          float V[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float v = 0.f;
            if (bc.k == 3) {                     // the paper's / BASELINE's k: 4 candidates, not KMAX
#pragma unroll
              for (int rr = 0; rr < 4; ++rr) v = (q - rr == n0) ? cr[rr] : v;
            } else {
#pragma unroll
              for (int rr = 0; rr < KMAX; ++rr) v = (rr <= bc.k && q - rr == n0) ? cr[rr] : v;
            }
            V[q] = v;
          }
          const float tot = warp_sum_transpose<16>(V, lane);
          if (lane < B) gdst[lane] += tot;
        } else {
          for (int n = 0; n < B; ++n) {
            const int rr = n - n0;
            float c = 0.f;
#pragma unroll
            for (int q = 0; q < KMAX; ++q)
              if (q == rr) c = cr[q];
            const float sw = warp_sum(c);
            if (lane == 0) gdst[n] += sw;
          }
        }
        if (l > 0) {
#pragma unroll
          for (int rr = 0; rr < KMAX; ++rr) {
            const int n = n0 + rr;
            if (rr > bc.k || n < 0 || n >= B) continue;
            const float w = W[(o * I + i) * B + n];
            T1 = fmaf(w, vv[1][rr], T1);
            T2 = fmaf(w, vv[2][rr], T2);
            T3 = fmaf(w, vv[3][rr], T3);
          }
          S1 = fmaf(yb[o][0], T1, fmaf(g1, T2, fmaf(g2, T3, S1)));
#pragma unroll
          for (int a = 0; a < NF; ++a) {
            dxb[a] = fmaf(yb[o][1 + a], T1, dxb[a]);
            if (a < NS) dxb[a] = fmaf(2.f * yb[o][1 + NF + a] * dx[a], T2, dxb[a]);
          }
#pragma unroll
          for (int a = 0; a < NS; ++a) ddxb[a] = fmaf(yb[o][1 + NF + a], T1, ddxb[a]);
        }
      }
      if (l > 0) {
        xb[i][0] = S1;
#pragma unroll
        for (int a = 0; a < NF; ++a) xb[i][1 + a] = dxb[a];
#pragma unroll
        for (int a = 0; a < NS; ++a) xb[i][1 + NF + a] = ddxb[a];
      }
      (void)S2; (void)S3;
    }
    if (l > 0)
      for (int i = 0; i < I; ++i)
#pragma unroll
        for (int c = 0; c < C; ++c) yb[i][c] = xb[i][c];
  }
}

// Blocks [0, nb_int) interior, [nb_int, nb_int + nb_bnd) boundary, then initial points.
// part[block][np + 4]: gradient partials, sum r^2 interior, sum e^2 boundary/initial, non-finite count.
template <int NF, int NS, int M, bool BURGERS>
__global__ void __launch_bounds__(TINY_THREADS)
    k_tiny_step(TinyNet tn, const float* __restrict__ params, BasisCfg bc, int D,
                const float* __restrict__ interior, const float* __restrict__ forcing, int64_t Ni, int nb_int,
                const float* __restrict__ boundary, const float* __restrict__ gb, int64_t Nb, int nb_bnd,
                const float* __restrict__ initial, const float* __restrict__ gi, int64_t N0,
                float alpha, float adv, float visc, float inv_int, float inv_bi, float* __restrict__ part,
                unsigned* __restrict__ done, float s_int, float* __restrict__ out) {
  __shared__ float prm[TINY_MAXP];
  __shared__ float gws[TINY_THREADS / 32][TINY_MAXP];
  const int np = tn.np;
  const int warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < np; t += blockDim.x) prm[t] = params[t];
  for (int t = threadIdx.x; t < (TINY_THREADS / 32) * np; t += blockDim.x) gws[t / np][t % np] = 0.f;
  __syncthreads();
  float sq_int = 0.f, sq_bi = 0.f, bad = 0.f;
  const int b = blockIdx.x;
  if (b < nb_int) {
    const int64_t p = (int64_t)b * TINY_THREADS + threadIdx.x;
    const bool valid = p < Ni;
    const float* pt = interior + (valid ? p : 0) * D;
    float aux = 0.f;
    if (!BURGERS && valid) {
      if (forcing) {
        aux = forcing[p];
      } else {
        float prod = 1.f;
        for (int a = 0; a < D; ++a) prod *= sinpif(pt[a]);
        aux = -(float)D * 9.8696044010893586f * prod;   // -D pi^2 prod_a sin(pi xi_a)  (Eq. 3)
      }
    }
    tiny_point<NF, NS, M, (BURGERS ? LAST_BURGERS : LAST_POISSON)>(tn, prm, bc, valid, pt, D, aux, alpha, adv, visc,
                                                                  inv_int, gws[warp], sq_int, bad);
  } else {
    int64_t p = (int64_t)(b - nb_int) * TINY_THREADS + threadIdx.x;
    const float* set = boundary;
    const float* tg = gb;
    int64_t n = Nb;
    if (b >= nb_int + nb_bnd) {
      p = (int64_t)(b - nb_int - nb_bnd) * TINY_THREADS + threadIdx.x;
      set = initial;
      tg = gi;
      n = N0;
    }
    const bool valid = p < n;
    const float* pt = set + (valid ? p : 0) * D;
    const float aux = valid ? tg[p] : 0.f;
    tiny_point<0, 0, M, LAST_BOUNDARY>(tn, prm, bc, valid, pt, D, aux, alpha, adv, visc, inv_bi, gws[warp], sq_bi,
                                       bad);
  }
  __shared__ float red[3][TINY_THREADS / 32];
  if ((threadIdx.x & 31) == 0) {
    red[0][warp] = sq_int;
    red[1][warp] = sq_bi;
    red[2][warp] = bad;
  }
  __syncthreads();
  float* dst = part + (size_t)blockIdx.x * (np + 4);
  for (int t = threadIdx.x; t < np; t += blockDim.x) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < TINY_THREADS / 32; ++w) v += gws[w][t];
    dst[t] = v;
  }
  if (threadIdx.x < 3) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < TINY_THREADS / 32; ++w) v += red[threadIdx.x][w];
    dst[np + threadIdx.x] = v;
  }
  // the last block to finish sums every block's partials in block order (deterministic) -- the
  // whole loss + gradient is one launch
  __shared__ unsigned ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(done, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  const int nb = (int)gridDim.x;
  for (int t = threadIdx.x; t < np + 4; t += blockDim.x) {
    if (t < np) {
      float sv = 0.f;
      for (int bb = 0; bb < nb; ++bb) sv += __ldcg(part + (size_t)bb * (np + 4) + t);
      out[t] = sv;
    } else {
      double sv = 0.0;
      if (t < np + 3)
        for (int bb = 0; bb < nb; ++bb) sv += (double)__ldcg(part + (size_t)bb * (np + 4) + t);
      const double sc = (t == np) ? (double)s_int : (t == np + 1) ? (double)inv_bi : 1.0;
      out[t] = (t == np + 3) ? 0.f : (float)(sv * sc);
    }
  }
  if (threadIdx.x == 0) *done = 0u;                // ready for the next call (and graph replay)
}

}  // namespace
