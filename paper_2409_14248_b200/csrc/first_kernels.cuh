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

// Forward of the first layer for interior passes (NF > 0), W staged in shared memory.
// Ws[a][KT + n][o] (n in [-KT, B + KT)) holds W^T with KT zero rows on each side, and the per-batch table
// stores the clamped first basis n0 and the values of the KT candidate bases n0 .. n0+KT-1 (zero outside
// the support, beyond k and outside [0, B)), so the contraction is KT unpredicated shared loads of W and
// 3*KT FFMAs per (point, coordinate, output) -- no global loads and no branches in the inner loop.
// Persistent grid (blocks stride over the 32-point batches).  KT = 4 covers k <= 3, KT = 8 any k <= 7.
template <int KT>
struct __align__(16) FlTab {
  float v[3][KT];       // v, v', v'' of the candidate bases n0 .. n0+KT-1
  int n0;               // clamped to [-KT, B]
  int pad[3];
};

template <int NF, int NS, int M, int KT>
__global__ void __launch_bounds__(FL_THREADS) k_fwd_first_s(const float* __restrict__ pts, const float* __restrict__ Wt,
                                                            const float* __restrict__ bias, float* __restrict__ Y,
                                                            int64_t P, int O, BasisCfg bc) {
  constexpr int D = NF;
  constexpr int C = 1 + NF + NS;
  extern __shared__ __align__(16) float fsm[];
  FlTab<KT>* tab = reinterpret_cast<FlTab<KT>*>(fsm);          // [FL_BATCH][D]
  float* Ws = fsm + FL_BATCH * D * (int)(sizeof(FlTab<KT>) / 4);   // [D][B + 2 KT][O]
  const int B = bc.B, BP = B + 2 * KT;
  for (int e = threadIdx.x; e < D * BP * O; e += blockDim.x) {
    const int o = e % O, r = e / O, a = r / BP, n = r - a * BP - KT;
    Ws[e] = (n >= 0 && n < B) ? __ldg(Wt + ((int64_t)a * B + n) * O + o) : 0.f;
  }
  const int QG = (int)blockDim.x / O;                            // point groups (O <= blockDim)
  const int qg = (int)threadIdx.x / O, o = (int)threadIdx.x % O;
  const float b = (qg < QG) ? __ldg(bias + o) : 0.f;
  for (int64_t p0 = (int64_t)blockIdx.x * FL_BATCH; p0 < P; p0 += (int64_t)gridDim.x * FL_BATCH) {
    __syncthreads();                                             // Ws staged / previous batch consumed
    for (int e = threadIdx.x; e < FL_BATCH * D; e += blockDim.x) {
      const int q = e / D, a = e - (e / D) * D;
      const int64_t p = p0 + q;
      const float x = (p < P) ? __ldg(pts + p * D + a) : 0.f;
      const int n0 = first_basis(x, bc);
      FlTab<KT>& t = tab[q * D + a];
#pragma unroll
      for (int r = 0; r < KT; ++r) {
        const int n = n0 + r;
        float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3;
        if (r <= bc.k && n >= 0 && n < B) hr_eval<M, (NS > 0 ? 2 : 1)>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        t.v[0][r] = (r == 0 && x != x) ? x : v0;   // propagate NaN inputs (the support test would drop them)
        t.v[1][r] = v1;
        t.v[2][r] = v2;
      }
      t.n0 = (x != x) ? 0 : min(max(n0, -KT), B);
    }
    __syncthreads();
    if (qg >= QG) continue;
    const int nq = (int)((P - p0) < FL_BATCH ? (P - p0) : FL_BATCH);
#pragma unroll 2
    for (int q = qg; q < nq; q += QG) {
      float acc[C];
      acc[0] = b;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const FlTab<KT>& t = tab[q * D + a];
        const float* wp = Ws + (a * BP + KT + t.n0) * O + o;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int r = 0; r < KT; ++r) {
          const float w = wp[r * O];
          s0 = fmaf(w, t.v[0][r], s0);
          s1 = fmaf(w, t.v[1][r], s1);
          s2 = fmaf(w, t.v[2][r], s2);
        }
        acc[0] += s0;
        acc[1 + a] = s1;
        if (a < NS) acc[1 + NF + a] = s2;
      }
      float* out = Y + (p0 + q) * (int64_t)(C * O) + o;
#pragma unroll
      for (int c = 0; c < C; ++c) out[c * O] = acc[c];
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

// Weight gradient of the first layer for interior passes, accumulated in REGISTERS: thread (o, point
// group qg) owns dW[o][a][n] for every coordinate a and every basis n < BMAX (BMAX >= B, packed pairs), and
// each point's contribution is applied densely over n from a per-batch shared table that holds
// v, v', v'' of every basis (zero outside the k+1 active ones):
//   acc[a][n] += ybar_o v_n(xi_a) + ybar'_{o,a} v'_n(xi_a) + ybar''_{o,a} v''_n(xi_a)
// -- (BMAX/(k+1))x more FMAs than the band-limited update, but no shared-memory read-modify-write
// chain (the previous kernel serialised on it) and no branches.  Block partials part[block][O][D][B]
// (+ part_b) are summed in a fixed order by k_reduce_parts.
// points per batch of k_wgrad_first_r (one bulk copy of their adjoint rows): 8, or 4 when two 8-point stages
// would exceed 72 KB (C5's 7 x 256 rows: 4 keeps two blocks per SM)
__host__ __device__ constexpr int wf_pb(int C, int O) { return 2 * 8 * C * O * 4 <= 72 * 1024 ? 8 : 4; }

template <int NF, int NS, int M, int BMAX>
__global__ void __launch_bounds__(FL_THREADS) k_wgrad_first_r(const float* __restrict__ pts,
                                                              const float* __restrict__ Ybar, float* __restrict__ part,
                                                              float* __restrict__ part_b, int64_t P, int O,
                                                              BasisCfg bc) {
  constexpr int D = NF;
  constexpr int C = 1 + NF + NS;
  constexpr int NPR = BMAX / 2;                   // basis pairs
  const int PB = wf_pb(C, O);
  static_assert(BMAX % 4 == 0, "table rows are float4 aligned");
  extern __shared__ __align__(16) float wsm[];
  const int B = bc.B;
  const int QG = (int)blockDim.x / O;
  const int ring = (max(2 * PB * C * O, QG * D * B * O) + 3) & ~3;   // the table after it stays 16-B aligned
  float* ybs = wsm;                               // [2][PB][C][O] adjoint rows (bulk copies, 2-stage ring);
                                                  // at the end [QG][D*B][O] accumulators
  float* V = ybs + ring;                          // [PB][D][3][BMAX]
  float* red = V + PB * D * 3 * BMAX;             // [FL_THREADS] fixed-order point-group reduction
  __shared__ __align__(8) uint64_t full[2];
  const int qg = (int)threadIdx.x / O, o = (int)threadIdx.x % O;
  const bool active = qg < QG;
  uint64_t acc[D][NPR];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int j = 0; j < NPR; ++j) acc[a][j] = 0ull;   // (0.f, 0.f)
  float dbs = 0.f;
  const int64_t lo = (P * blockIdx.x) / gridDim.x, hi = (P * (blockIdx.x + 1)) / gridDim.x;
  const int nbat = (int)((hi - lo + PB - 1) / PB);
  const uint32_t row_bytes = (uint32_t)(C * O * 4);
  auto issue = [&](int b) {                       // thread 0: batch b -> stage b & 1
    const int64_t p0 = lo + (int64_t)b * PB;
    const int npb = (int)((hi - p0) < PB ? (hi - p0) : PB);
    tc::mbar_arrive_expect_tx(&full[b & 1], row_bytes * npb);
    tc::bulk_g2s(ybs + (b & 1) * (PB * C * O), Ybar + p0 * (int64_t)(C * O), row_bytes * npb, &full[b & 1]);
  };
  if (threadIdx.x == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_mbar_init();
    if (nbat > 0) issue(0);
    if (nbat > 1) issue(1);
  }
  for (int b = 0; b < nbat; ++b) {
    const int64_t p0 = lo + (int64_t)b * PB;
    const int nq = (int)((hi - p0) < PB ? (hi - p0) : PB);
    __syncthreads();                              // previous batch's table consumed (and barrier init visible)
    // table: task = (point q, coordinate a, 4 consecutive bases), each basis evaluated in place
    for (int e = threadIdx.x; e < PB * D * (BMAX / 4); e += blockDim.x) {
      const int n4 = 4 * (e % (BMAX / 4)), qa = e / (BMAX / 4);
      const int q = qa / D, a = qa - (qa / D) * D;
      const float x = (q < nq) ? __ldg(pts + (p0 + q) * D + a) : 0.f;
      const int n0 = first_basis(x, bc);
      float vd[3][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int n = n4 + u, r = n - n0;
        float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3;
        if (q < nq && r >= 0 && r <= bc.k && n < B) hr_eval<M, (NS > 0 ? 2 : 1)>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
        if (q < nq && x != x) v0 = v1 = v2 = x;   // NaN inputs poison their row (flagged downstream)
        vd[0][u] = v0;
        vd[1][u] = v1;
        vd[2][u] = v2;
      }
      float* row = V + qa * 3 * BMAX + n4;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        *reinterpret_cast<float4*>(row + d * BMAX) = make_float4(vd[d][0], vd[d][1], vd[d][2], vd[d][3]);
    }
    __syncthreads();
    tc::mbar_wait(&full[b & 1], (uint32_t)((b >> 1) & 1));
    const float* yst = ybs + (b & 1) * (PB * C * O) + o;
    if (active) {
      for (int q = qg; q < nq; q += QG) {
        float y[C];
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = yst[(q * C + c) * O];
        dbs += y[0];
        const uint64_t Y0 = tc::pk2(y[0], y[0]);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const uint64_t Y1 = tc::pk2(y[1 + a], y[1 + a]);
          const float y2 = (a < NS) ? y[1 + NF + (a < NS ? a : 0)] : 0.f;
          const uint64_t Y2 = tc::pk2(y2, y2);
          const float4* r0 = reinterpret_cast<const float4*>(V + (q * D + a) * 3 * BMAX);
#pragma unroll
          for (int j4 = 0; j4 < BMAX / 4; ++j4) {
            const float4 w0 = r0[j4], w1 = r0[BMAX / 4 + j4];
            uint64_t a0 = acc[a][2 * j4], a1 = acc[a][2 * j4 + 1];
            a0 = tc::fma2(Y0, tc::pk2(w0.x, w0.y), a0);
            a1 = tc::fma2(Y0, tc::pk2(w0.z, w0.w), a1);
            a0 = tc::fma2(Y1, tc::pk2(w1.x, w1.y), a0);
            a1 = tc::fma2(Y1, tc::pk2(w1.z, w1.w), a1);
            if (a < NS) {
              const float4 w2 = r0[2 * (BMAX / 4) + j4];
              a0 = tc::fma2(Y2, tc::pk2(w2.x, w2.y), a0);
              a1 = tc::fma2(Y2, tc::pk2(w2.z, w2.w), a1);
            }
            acc[a][2 * j4] = a0;
            acc[a][2 * j4 + 1] = a1;
          }
        }
      }
    }
    __syncthreads();                              // stage b & 1 fully read
    if (threadIdx.x == 0 && b + 2 < nbat) {
      tc::fence_proxy_async_smem();               // generic reads of the stage before the async-proxy refill
      issue(b + 2);
    }
  }
  // fixed-order sum over the point groups: accumulators -> shared [QG][D*B][O] (the stage ring is free now)
  const int64_t nW = (int64_t)O * D * B;
  float* dst = part + (int64_t)blockIdx.x * nW;
  float* accs = ybs;
  __syncthreads();
  if (active) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int j = 0; j < NPR; ++j) {
        float lo_, hi_;
        tc::upk2(acc[a][j], lo_, hi_);
        if (2 * j < B) accs[((qg * D + a) * B + 2 * j) * O + o] = lo_;
        if (2 * j + 1 < B) accs[((qg * D + a) * B + 2 * j + 1) * O + o] = hi_;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D * B * O; e += blockDim.x) {
    float v = 0.f;
    for (int g = 0; g < QG; ++g) v += accs[g * D * B * O + e];
    const int oo = e % O, an = e / O;            // accs index (a*B + n)*O + o
    dst[(int64_t)oo * D * B + an] = v;
  }
  __syncthreads();
  red[threadIdx.x] = active ? dbs : 0.f;
  __syncthreads();
  if (qg == 0) {
    float v = 0.f;
    for (int g = 0; g < QG; ++g) v += red[g * O + o];
    part_b[blockIdx.x * (int64_t)O + o] = v;
  }
}


// Band-limited variant of k_wgrad_first_r for k <= 3 (HRKAN_WF_WINDOW, default on): every thread of the block
// works on the SAME point, so the k+1 <= 4 non-zero bases of a coordinate sit at a block-uniform position --
// the update touches only the three accumulator pairs jp .. jp+2 (jp = floor(n0 / 2) clamped into the
// table, which covers n0 .. n0+3 and every in-range basis of an out-of-grid x) through a block-uniform
// switch over jp, 9 FFMA2 per coordinate instead of 3 * BMAX/2.  The per-batch table holds v, v', v'' of
// those six bases only and is double-buffered: batch b+1's table is built by the first threads while the
// block accumulates batch b (one __syncthreads per batch).
#ifndef HRKAN_WF_WINDOW
#define HRKAN_WF_WINDOW 1
#endif
// f(integral_constant<J>) for the block-uniform J = jp in [0, NPR-3] (NPR <= 10: at most 8 cases)
template <int NPR, class F>
__device__ __forceinline__ void wf_switch(int jp, F&& f) {
  static_assert(NPR - 3 <= 7, "extend the switch");
#define HRKAN_WF_CASE(J)                                                    \
  case J:                                                                   \
    if constexpr (J <= NPR - 3) f(std::integral_constant<int, J>{});        \
    break;
  switch (jp) {
    HRKAN_WF_CASE(0) HRKAN_WF_CASE(1) HRKAN_WF_CASE(2) HRKAN_WF_CASE(3)
    HRKAN_WF_CASE(4) HRKAN_WF_CASE(5) HRKAN_WF_CASE(6) HRKAN_WF_CASE(7)
  }
#undef HRKAN_WF_CASE
}

template <int NF, int NS, int M, int BMAX>
__global__ void __launch_bounds__(FL_THREADS) k_wgrad_first_w(const float* __restrict__ pts,
                                                              const float* __restrict__ Ybar, float* __restrict__ part,
                                                              float* __restrict__ part_b, int64_t P, int O,
                                                              BasisCfg bc) {
  constexpr int D = NF;
  constexpr int C = 1 + NF + NS;
  constexpr int NPR = BMAX / 2;                   // accumulator pairs per coordinate
  constexpr int TW = 3 * 6 + 2;                   // table row: [3 orders][6 bases] + jp + pad (8-B aligned)
  static_assert(NPR >= 3, "window of three pairs");
  const int PB = wf_pb(C, O);
  extern __shared__ __align__(16) float wsm[];
  const int B = bc.B;
  const int QG = (int)blockDim.x / O;
  const int ring = (max(2 * PB * C * O, QG * D * B * O) + 3) & ~3;   // the table after it stays 16-B aligned
  float* ybs = wsm;                               // [2][PB][C][O] adjoint rows (bulk copies, 2-stage ring);
                                                  // at the end [QG][D*B][O] accumulators
  float* V = ybs + ring;                          // [2][PB][D][TW]
  float* red = V + 2 * PB * D * TW;               // [FL_THREADS] fixed-order point-group reduction
  __shared__ __align__(8) uint64_t full[2];
  const int qg = (int)threadIdx.x / O, o = (int)threadIdx.x % O;
  const bool active = qg < QG;
  uint64_t acc[D][NPR];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int j = 0; j < NPR; ++j) acc[a][j] = 0ull;   // (0.f, 0.f)
  float dbs = 0.f;
  const int64_t lo = (P * blockIdx.x) / gridDim.x, hi = (P * (blockIdx.x + 1)) / gridDim.x;
  const int nbat = (int)((hi - lo + PB - 1) / PB);
  const uint32_t row_bytes = (uint32_t)(C * O * 4);
  auto issue = [&](int b) {                       // thread 0: batch b -> stage b & 1
    const int64_t p0 = lo + (int64_t)b * PB;
    const int npb = (int)((hi - p0) < PB ? (hi - p0) : PB);
    tc::mbar_arrive_expect_tx(&full[b & 1], row_bytes * npb);
    tc::bulk_g2s(ybs + (b & 1) * (PB * C * O), Ybar + p0 * (int64_t)(C * O), row_bytes * npb, &full[b & 1]);
  };
  // table of batch b: task = (point q, coordinate a, basis u of the six 2 jp .. 2 jp + 5), spread over the
  // warps (lanes 0 .. NTL-1 of each) so that no single warp carries the build
  const int warp_ = (int)threadIdx.x >> 5, lane_ = (int)threadIdx.x & 31, nwarp_ = (int)blockDim.x >> 5;
  const int ntask = PB * D * 6, NTL = (ntask + nwarp_ - 1) / nwarp_;
  auto build = [&](int b) {
    const int64_t p0 = lo + (int64_t)b * PB;
    const int nq = (int)((hi - p0) < PB ? (hi - p0) : PB);
    for (int l = lane_; l < NTL; l += 32) {
      const int e6 = warp_ * NTL + l;
      if (e6 >= ntask) break;
      const int e = e6 / 6, u = e6 - e * 6;
      const int q = e / D;
      float* row = V + ((b & 1) * PB * D + e) * TW;
      const float x = (q < nq) ? __ldg(pts + (p0 + q) * D + (e - q * D)) : 0.f;
      int jp = first_basis(x, bc) >> 1;           // floor(n0 / 2), also for negative n0
      jp = min(max(jp, 0), NPR - 3);
      const int n = 2 * jp + u;
      float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3;
      if (q < nq && n < B) hr_eval<M, (NS > 0 ? 2 : 1)>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
      if (q < nq && x != x) v0 = v1 = v2 = x;     // NaN inputs poison their row (flagged downstream)
      row[u] = v0;
      row[6 + u] = v1;
      row[12 + u] = v2;
      if (u == 0) reinterpret_cast<int*>(row)[18] = jp;
    }
  };
  if (threadIdx.x == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_mbar_init();
    if (nbat > 0) issue(0);
    if (nbat > 1) issue(1);
  }
  if (nbat > 0) build(0);
  __syncthreads();                                // barrier init and table 0 visible
  for (int b = 0; b < nbat; ++b) {
    const int64_t p0 = lo + (int64_t)b * PB;
    const int nq = (int)((hi - p0) < PB ? (hi - p0) : PB);
    if (b + 1 < nbat) build(b + 1);               // other half of the table ring (batch b-1 finished at the last barrier)
    tc::mbar_wait(&full[b & 1], (uint32_t)((b >> 1) & 1));
    const float* yst = ybs + (b & 1) * (PB * C * O) + o;
    const float* Vb = V + (b & 1) * PB * D * TW;
    if (active) {
      for (int q = qg; q < nq; q += QG) {
        float y[C];
#pragma unroll
        for (int c = 0; c < C; ++c) y[c] = yst[(q * C + c) * O];
        dbs += y[0];
        const uint64_t Y0 = tc::pk2(y[0], y[0]);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const uint64_t Y1 = tc::pk2(y[1 + a], y[1 + a]);
          const float y2 = (a < NS) ? y[1 + NF + (a < NS ? a : 0)] : 0.f;
          const uint64_t Y2 = tc::pk2(y2, y2);
          const float* row = Vb + (q * D + a) * TW;
          // the point's contribution to the three pairs (independent of the accumulators: full ILP) ...
          uint64_t c3[3];
#pragma unroll
          for (int w = 0; w < 3; ++w) {
            uint64_t t = tc::mul2(Y1, *reinterpret_cast<const uint64_t*>(row + 6 + 2 * w));
            if (a < NS) t = tc::fma2(Y2, *reinterpret_cast<const uint64_t*>(row + 12 + 2 * w), t);
            c3[w] = tc::fma2(Y0, *reinterpret_cast<const uint64_t*>(row + 2 * w), t);
          }
          // ... added to the accumulator pairs jp .. jp+2 (block-uniform jp)
          const int jp = reinterpret_cast<const int*>(row)[18];
          wf_switch<NPR>(jp, [&](auto Jc) {
            constexpr int J = decltype(Jc)::value;
            const uint64_t ONE2 = tc::pk2(1.f, 1.f);
#pragma unroll
            for (int w = 0; w < 3; ++w) acc[a][J + w] = tc::fma2(c3[w], ONE2, acc[a][J + w]);
          });
        }
      }
    }
    __syncthreads();                              // stage b & 1 and table b & 1 fully read; table (b+1) & 1 complete
    if (threadIdx.x == 0 && b + 2 < nbat) {
      tc::fence_proxy_async_smem();               // generic reads of the stage before the async-proxy refill
      issue(b + 2);
    }
  }
  // fixed-order sum over the point groups: accumulators -> shared [QG][D*B][O] (the stage ring is free now)
  const int64_t nW = (int64_t)O * D * B;
  float* dst = part + (int64_t)blockIdx.x * nW;
  float* accs = ybs;
  __syncthreads();
  if (active) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int j = 0; j < NPR; ++j) {
        float lo_, hi_;
        tc::upk2(acc[a][j], lo_, hi_);
        if (2 * j < B) accs[((qg * D + a) * B + 2 * j) * O + o] = lo_;
        if (2 * j + 1 < B) accs[((qg * D + a) * B + 2 * j + 1) * O + o] = hi_;
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < D * B * O; e += blockDim.x) {
    float v = 0.f;
    for (int g = 0; g < QG; ++g) v += accs[g * D * B * O + e];
    const int oo = e % O, an = e / O;            // accs index (a*B + n)*O + o
    dst[(int64_t)oo * D * B + an] = v;
  }
  __syncthreads();
  red[threadIdx.x] = active ? dbs : 0.f;
  __syncthreads();
  if (qg == 0) {
    float v = 0.f;
    for (int g = 0; g < QG; ++g) v += red[g * O + o];
    part_b[blockIdx.x * (int64_t)O + o] = v;
  }
}

}  // namespace
