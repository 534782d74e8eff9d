// first_kernels.cuh -- the first KAN layer (raw coordinates -> hidden jet) and its weight gradient
// (SURVEY §8(a) rows a1, a7).  The layer input is the point itself: x_a = xi_a, dx_{a,a'} = delta,
// ddx = 0, so its contraction is structured and tiny (K = D(G+k) <= 57):
//   y_o     = b_o + sum_{a,n} W[o,a,n] v_n(xi_a)        y'_{o,a} = sum_n W[o,a,n] v'_n(xi_a)
//   y''_{o,a} = sum_n W[o,a,n] v''_n(xi_a)                                  (Eq. 2)
//   dW[o,a,n] += ybar_o v_n(xi_a) + ybar'_{o,a} v'_n(xi_a) + ybar''_{o,a} v''_n(xi_a),  db_o += ybar_o
// Both kernels share one idea: a block takes a batch of points, evaluates the k+1 non-zero bases of
// each coordinate ONCE into a shared table, and then every thread (one per output neuron o) works
// on that batch with coalesced loads/stores of the [P][C][O] jets.  FP32 FFMA.
#pragma once

namespace {   // internal linkage: every translation unit owns its kernels
using namespace hrkan;

constexpr int FL_BATCH = 32;            // points per shared basis table
constexpr int FL_THREADS = 256;

// Shared basis table entry for (point, coordinate a): first basis n0 and v, v', v'' of the k+1
// candidates n0 .. n0+k (zero where n is outside [0, B) or x outside the support).
struct __align__(8) FlBasis {
  float v[3][KMAX];     // 8-byte aligned pairs v[c][2j], v[c][2j+1] (packed-pair loads)
  int n0;
  int pad;
};

template <int D, int M, int ND>
__device__ __forceinline__ void fl_table(const float* __restrict__ pts, int64_t p0, int64_t P, const BasisCfg& bc,
                                         FlBasis* tab) {
  for (int e = threadIdx.x; e < FL_BATCH * D; e += blockDim.x) {
    const int q = e / D, a = e - (e / D) * D;
    const int64_t p = p0 + q;
    FlBasis t;
    const float x = (p < P) ? __ldg(pts + p * D + a) : 0.f;
    t.n0 = first_basis(x, bc);
#pragma unroll
    for (int r = 0; r < KMAX; ++r) {
      const int n = t.n0 + r;
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3;
      if (r <= bc.k && n >= 0 && n < bc.B) hr_eval<M, ND>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
      t.v[0][r] = v0;
      t.v[1][r] = v1;
      t.v[2][r] = v2;
    }
    if (x != x) {                         // propagate NaN inputs (the support test would drop them)
      t.n0 = 0;
      t.v[0][0] = x;
    }
    tab[q * D + a] = t;
  }
}

// Forward:  Y[p][c][o], channels c = 0 value, 1..NF first, NF+1..NF+NS diagonal second derivatives.
// Wt = W transposed to [D][B][O] (coalesced across o).
template <int NF, int NS, int M>
__global__ void __launch_bounds__(FL_THREADS) k_fwd_first(const float* __restrict__ pts, const float* __restrict__ Wt,
                                                          const float* __restrict__ bias, float* __restrict__ Y,
                                                          int64_t P, int D_, int O, BasisCfg bc) {
  constexpr int D = (NF > 0) ? NF : 1;   // interior passes carry D = NF coordinates; value-only passes
  constexpr int C = 1 + NF + NS;         // get D from the argument below
  __shared__ FlBasis tab[FL_BATCH * 3];
  const int Dr = (NF > 0) ? D : D_;
  for (int64_t p0 = (int64_t)blockIdx.x * FL_BATCH; p0 < P; p0 += (int64_t)gridDim.x * FL_BATCH) {
    __syncthreads();
    if (NF > 0) fl_table<D, M, (NS > 0 ? 2 : 1)>(pts, p0, P, bc, tab);
    else {
      for (int e = threadIdx.x; e < FL_BATCH * Dr; e += blockDim.x) {   // value-only: v only
        const int q = e / Dr, a = e - (e / Dr) * Dr;
        const int64_t p = p0 + q;
        FlBasis t;
        const float x = (p < P) ? __ldg(pts + p * Dr + a) : 0.f;
        t.n0 = first_basis(x, bc);
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          const int n = t.n0 + r;
          float v0 = 0.f, v1, v2, v3;
          if (r <= bc.k && n >= 0 && n < bc.B) hr_eval<M, 0>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
          t.v[0][r] = v0;
          t.v[1][r] = 0.f;
          t.v[2][r] = 0.f;
        }
        if (x != x) {
          t.n0 = 0;
          t.v[0][0] = x;
        }
        tab[q * Dr + a] = t;
      }
    }
    __syncthreads();
    const int nq = (int)((P - p0) < FL_BATCH ? (P - p0) : FL_BATCH);
    // thread -> (output o, point group qg): narrow layers (O < blockDim) split the batch's points
    const int QG = O <= (int)blockDim.x ? (int)blockDim.x / O : 1;
    const int qg = O <= (int)blockDim.x ? (int)threadIdx.x / O : 0;
    const int o0 = (O <= (int)blockDim.x && qg >= QG) ? O : (O <= (int)blockDim.x ? (int)threadIdx.x % O : (int)threadIdx.x);
    const int ostep = O <= (int)blockDim.x ? O : (int)blockDim.x;
    for (int o = o0; o < O; o += ostep) {
      const float b = __ldg(bias + o);
      for (int q = qg; q < nq; q += QG) {
        float acc[C];
        acc[0] = b;
#pragma unroll
        for (int c = 1; c < C; ++c) acc[c] = 0.f;
        for (int a = 0; a < Dr; ++a) {
          const FlBasis& t = tab[q * Dr + a];
          // two bases per FFMA2 (table pairs are 8-byte aligned)
          uint64_t S0 = tc::pk2(0.f, 0.f), S1 = S0, S2 = S0;
#pragma unroll
          for (int r = 0; r < KMAX; r += 2) {
            if (r > bc.k) break;
            const int na = t.n0 + r, nb = na + 1;
            const bool oka = na >= 0 && na < bc.B, okb = r + 1 <= bc.k && nb >= 0 && nb < bc.B;
            const uint64_t w = tc::pk2(oka ? __ldg(Wt + ((int64_t)a * bc.B + na) * O + o) : 0.f,
                                       okb ? __ldg(Wt + ((int64_t)a * bc.B + nb) * O + o) : 0.f);
            S0 = tc::fma2(w, *reinterpret_cast<const uint64_t*>(&t.v[0][r]), S0);
            S1 = tc::fma2(w, *reinterpret_cast<const uint64_t*>(&t.v[1][r]), S1);
            S2 = tc::fma2(w, *reinterpret_cast<const uint64_t*>(&t.v[2][r]), S2);
          }
          float s0, s1, s2, hi_;
          tc::upk2(S0, s0, hi_); s0 += hi_;
          tc::upk2(S1, s1, hi_); s1 += hi_;
          tc::upk2(S2, s2, hi_); s2 += hi_;
          acc[0] += s0;
#pragma unroll
          for (int aa = 0; aa < NF; ++aa)
            if (aa == a) acc[1 + aa] = s1;
#pragma unroll
          for (int aa = 0; aa < NS; ++aa)
            if (aa == a) acc[1 + NF + aa] = s2;
        }
        float* out = Y + (p0 + q) * (int64_t)(C * O) + o;
#pragma unroll
        for (int c = 0; c < C; ++c) out[c * O] = acc[c];
      }
    }
  }
}

// Weight gradient of the first layer: a grid of blocks over contiguous point ranges; thread (o, point
// group qg) keeps its (a, n) accumulators in shared memory acc[qg][a][n][o] (private column, no
// atomics); the block sums its point groups in a fixed order into part[block][O][D][B] (+ part_b)
// and k_reduce_parts sums the blocks in a fixed order.  Narrow layers (O < blockDim) use several
// point groups so that every thread works.
template <int NF, int NS, int M>
__global__ void __launch_bounds__(FL_THREADS) k_wgrad_first(const float* __restrict__ pts,
                                                            const float* __restrict__ Ybar, float* __restrict__ part,
                                                            float* __restrict__ part_b, int64_t P, int D_, int O,
                                                            BasisCfg bc) {
  constexpr int D = (NF > 0) ? NF : 1;
  constexpr int C = 1 + NF + NS;
  __shared__ FlBasis tab[FL_BATCH * 3];
  __shared__ float dbs_sh[FL_THREADS * 2];
  extern __shared__ float acc[];          // [QG][Dr][B][O]
  const int Dr = (NF > 0) ? D : D_;
  const int B = bc.B;
  const int QG = O <= (int)blockDim.x ? (int)blockDim.x / O : 1;
  const int qg = O <= (int)blockDim.x ? (int)threadIdx.x / O : 0;
  const bool active = qg < QG;
  const int o0 = O <= (int)blockDim.x ? (int)threadIdx.x % O : (int)threadIdx.x;
  const int ostep = O <= (int)blockDim.x ? O : (int)blockDim.x;
  const int64_t nW = (int64_t)O * Dr * B;
  for (int64_t e = threadIdx.x; e < QG * nW; e += blockDim.x) acc[e] = 0.f;
  float* accq = acc + (active ? qg : 0) * nW;
  const int64_t lo = (P * blockIdx.x) / gridDim.x, hi = (P * (blockIdx.x + 1)) / gridDim.x;
  float dbs[2] = {0.f, 0.f};              // O <= 2 * FL_THREADS
  for (int64_t p0 = lo; p0 < hi; p0 += FL_BATCH) {
    __syncthreads();
    const int64_t pe = (hi < p0 + FL_BATCH) ? hi : p0 + FL_BATCH;
    if (NF > 0) fl_table<D, M, (NS > 0 ? 2 : 1)>(pts, p0, pe, bc, tab);
    else {
      for (int e = threadIdx.x; e < FL_BATCH * Dr; e += blockDim.x) {
        const int q = e / Dr, a = e - (e / Dr) * Dr;
        const int64_t p = p0 + q;
        FlBasis t;
        const float x = (p < pe) ? __ldg(pts + p * Dr + a) : 0.f;
        t.n0 = first_basis(x, bc);
#pragma unroll
        for (int r = 0; r < KMAX; ++r) {
          const int n = t.n0 + r;
          float v0 = 0.f, v1, v2, v3;
          if (r <= bc.k && n >= 0 && n < bc.B) hr_eval<M, 0>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
          t.v[0][r] = v0;
          t.v[1][r] = 0.f;
          t.v[2][r] = 0.f;
        }
        tab[q * Dr + a] = t;
      }
    }
    __syncthreads();
    if (!active) continue;
    const int nq = (int)(pe - p0);
    int oo = 0;
    for (int o = o0; o < O; o += ostep, ++oo) {
      // the next point's adjoint row is loaded while this one is accumulated (latency hiding)
      float yn[C];
#pragma unroll
      for (int c = 0; c < C; ++c) yn[c] = (qg < nq) ? __ldg(Ybar + (p0 + qg) * (int64_t)(C * O) + c * O + o) : 0.f;
      for (int q = qg; q < nq; q += QG) {
        float y[C];
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = yn[c];
        if (q + QG < nq) {
          const float* ybn = Ybar + (p0 + q + QG) * (int64_t)(C * O) + o;
#pragma unroll
          for (int c = 0; c < C; ++c) yn[c] = __ldg(ybn + c * O);
        }
        dbs[oo] += y[0];
        for (int a = 0; a < Dr; ++a) {
          const FlBasis& t = tab[q * Dr + a];
          float y1 = 0.f, y2 = 0.f;
#pragma unroll
          for (int aa = 0; aa < NF; ++aa)
            if (aa == a) y1 = y[1 + aa];
#pragma unroll
          for (int aa = 0; aa < NS; ++aa)
            if (aa == a) y2 = y[1 + NF + aa];
          // two bases per FFMA2/FMUL2 (table pairs are 8-byte aligned); the accumulations stay per basis
          const uint64_t Y0 = tc::pk2(y[0], y[0]), Y1 = tc::pk2(y1, y1), Y2 = tc::pk2(y2, y2);
#pragma unroll
          for (int r = 0; r < KMAX; r += 2) {
            if (r > bc.k) break;
            const int na = t.n0 + r, nb = na + 1;
            const bool oka = na >= 0 && na < B, okb = r + 1 <= bc.k && nb >= 0 && nb < B;
            const uint64_t c2 = tc::fma2(Y0, *reinterpret_cast<const uint64_t*>(&t.v[0][r]),
                                         tc::fma2(Y1, *reinterpret_cast<const uint64_t*>(&t.v[1][r]),
                                                  tc::mul2(Y2, *reinterpret_cast<const uint64_t*>(&t.v[2][r]))));
            float ca, cb;
            tc::upk2(c2, ca, cb);
            if (oka) accq[(a * B + na) * O + o] += ca;
            if (okb) accq[(a * B + nb) * O + o] += cb;
          }
        }
      }
    }
  }
  // fixed-order sum over the point groups
  dbs_sh[threadIdx.x] = active ? dbs[0] : 0.f;
  dbs_sh[FL_THREADS + threadIdx.x] = active ? dbs[1] : 0.f;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < nW; e += blockDim.x) {
    float v = 0.f;
    for (int g = 0; g < QG; ++g) v += acc[g * nW + e];
    const int o = (int)(e % O), an = (int)(e / O);          // acc index (a*B + n)*O + o
    part[blockIdx.x * nW + (int64_t)o * Dr * B + an] = v;
  }
  for (int o = threadIdx.x; o < O; o += blockDim.x) {
    float v = 0.f;
    if (O <= (int)blockDim.x) {
      for (int g = 0; g < QG; ++g) v += dbs_sh[g * O + o];
    } else {
      v = dbs_sh[(o / blockDim.x) * FL_THREADS + (o % blockDim.x)];
    }
    part_b[blockIdx.x * (int64_t)O + o] = v;
  }
}

}  // namespace
