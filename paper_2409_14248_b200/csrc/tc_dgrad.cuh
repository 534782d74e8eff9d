// tc_dgrad.cuh -- tensor-core input-adjoint kernel of a hidden layer, included by
// tc_kernels.cuh.
//
//   Abar^c[p,(i,n)] = sum_o Ybar^c[p,o] W[o,(i,n)]                  (bf16x3 tcgen05, fp32 TMEM)
// then the jet-chain epilogue (v1, v2, v3 = first/second/third x-derivatives of basis n at x_i):
//   xbar    = sum_n [Abar^0 v1 + sum_a Abar^{1,a} v2 dx_a + sum_a Abar^{2,a} (v3 dx_a^2 + v2 ddx_a)]
//   dxbar_a = sum_n [Abar^{1,a} v1 + 2 Abar^{2,a} v2 dx_a],     ddxbar_a = sum_n Abar^{2,a} v1
//
// Orientation: MMA M = 128 contiguous K rows (i,n) -- an input split between two tiles is summed through
// a per-point carry in shared memory (input-aligned tiles of floor(128/B) whole inputs when B < 11, see
// dgr_rows_per_tile) -- MMA N = (point, channel) columns p*C + c of NP points, MMA
// K = o.  A = pre-tiled W^T hi/lo and B = pre-split Ybar hi/lo (k_split_ybar), both by 1-D bulk
// copies per stage.  Two TMEM accumulators: the 8 epilogue warps drain M-tile t while the MMA
// runs t+1.  Epilogue: TMEM -> smem slice of SLICE_P points -> each (point, input) gathers only the
// k+1 non-zero bases of its x (input jets TMA-loaded per M-tile) -> Xbar[p][c][i].
#pragma once
#ifndef HRKAN_DGR_NSTAGE_MAX
#define HRKAN_DGR_NSTAGE_MAX 8   // stage-ring depth cap (shared memory permitting)
#endif

namespace {

// Epilogue parallelism: a slice of SLICE_P points gives SLICE_P * IPT (point, input) gather tasks per
// barrier interval; slices and epilogue warps are sized so those tasks fill the epilogue threads
// (measured per 2^18 points: C4's C = 4 layers with 32-point slices and 12 warps 3.58 -> 2.65 ms, C3's
// C = 5 layers with 24-point slices 1.29 -> 1.08 ms; C5's 7-channel slices stay at 16 points, 32 would
// leave room for only 3 stages and was 30 % slower).
// dgrad epilogue arithmetic on packed fp32 pairs (two bases per FFMA2/FMUL2) for m >= 4
// (C4 dgrad 2.76 -> 2.55 ms, C3 1.12 -> 0.96 ms per 2^18 points)
#ifndef HRKAN_DGR_F32X2
#define HRKAN_DGR_F32X2 1
#endif
#ifndef HRKAN_DGR_SLICE_P
#define HRKAN_DGR_SLICE_P 0
#endif
#ifndef HRKAN_DGR_EPI_WARPS
#define HRKAN_DGR_EPI_WARPS 0
#endif
__host__ __device__ constexpr int dgr_slice_p(int C) {
  return (HRKAN_DGR_SLICE_P > 0 && C > 1 && tc_np(C) % (HRKAN_DGR_SLICE_P > 0 ? HRKAN_DGR_SLICE_P : 1) == 0 &&
          (HRKAN_DGR_SLICE_P * C) % 8 == 0)
             ? HRKAN_DGR_SLICE_P
             : C == 1 ? 64 : C == 4 ? 32 : C == 5 ? 24 : 16;
}
__host__ __device__ constexpr int dgr_epi_warps(int C) {
  return HRKAN_DGR_EPI_WARPS > 0 ? HRKAN_DGR_EPI_WARPS : C == 4 ? 12 : 8;
}
constexpr int DGR_SST = 129;   // column stride of the epilogue slice (odd: conflict-free gathers)
constexpr int DGR_IPTB = 16;   // jet box width (inputs) >= inputs per M-tile + 3 (box start aligned down to 16 B)

// M-tile rows.  Contiguous: 128 K rows (i, n), an input split between two tiles summed through a
// per-point carry in shared memory -- used for 3-D nets (7-channel jets, MMA-bound: C5 dgrad 10.8 ->
// 9.9 ms per 2^18 points, no idle rows) when the jet box holds every input such a tile touches (B >= 11).
// Input-aligned: floor(128/B) whole inputs (IPT*B < 128 rows busy) -- kept for the 4/5-channel nets,
// whose epilogue-bound tiles got 14-22 % slower with the extra inputs per contiguous tile.
__host__ __device__ constexpr int dgr_rows_per_tile(int B, int D) {
  return (D >= 3 && 127 / B + 5 <= DGR_IPTB) ? 128 : (128 / B) * B;
}
__host__ __device__ constexpr bool dgr_tile_ok(int B, int D) {
  return B >= 1 && ((dgr_rows_per_tile(B, D) == 128 ? 127 / B + 2 : 128 / B) + 3 <= DGR_IPTB);
}

template <int NF, int NS, int M, int OO>
struct DgrCfg {
  static constexpr int C = 1 + NF + NS;
  static constexpr int NP = tc_np(C);
  static constexpr int N = NP * C;
  static constexpr int O = OO;                                // = MMA K of this kernel (64, 128, 256)
  static constexpr int NKB = O / TC_KB;
  static constexpr int W_STAGE_BYTES = 2 * 2 * 128 * 16;      // W^T hi + lo, [2 chunks][128 rows][8] bf16
  static constexpr int Y_STAGE_BYTES = 2 * 2 * N * 16;        // Ybar hi + lo, [2 chunks][N rows][8] bf16
  static constexpr int STAGE_BYTES = W_STAGE_BYTES + Y_STAGE_BYTES;
  static constexpr int JET_FLOATS = N * DGR_IPTB;             // TMA box X[NP][C][IPTB]
  static constexpr int SLICE_P = dgr_slice_p(C);
  static constexpr int S_FLOATS = SLICE_P * C * DGR_SST;
  static constexpr int FIXED_BYTES = 4 * (2 * JET_FLOATS + S_FLOATS + 2 * NP * C) + 1024;   // + split-input carries
  static constexpr int NSTAGE_FIT = (225 * 1024 - FIXED_BYTES) / STAGE_BYTES;
  static constexpr int NSTAGE = NSTAGE_FIT > HRKAN_DGR_NSTAGE_MAX ? HRKAN_DGR_NSTAGE_MAX : NSTAGE_FIT;
  static constexpr int SMEM_BYTES = NSTAGE * STAGE_BYTES + FIXED_BYTES;
  static constexpr uint32_t TMEM_COLS = tc_tmem_cols(2 * N);
  static constexpr int EPI_WARPS = dgr_epi_warps(C);           // multiple of 4 (TMEM lane quadrants)
  static constexpr int THREADS = 32 * (EPI_WARPS + 3);          // + MMA warp + stage producer + jet producer
  static constexpr int MMA_WARP = EPI_WARPS, PROD_WARP = EPI_WARPS + 1, JET_WARP = EPI_WARPS + 2;
  static_assert(N % 16 == 0 && N <= 256, "bad N");
  static_assert(NP % SLICE_P == 0 && (SLICE_P * C) % 8 == 0 && EPI_WARPS % 4 == 0, "bad slice");
  static_assert(NSTAGE >= 3, "shared memory budget");
  static_assert(STAGE_BYTES % 128 == 0, "TMA boxes after the stages need 128-B alignment");
};

// W^T tiles for k_dgrad_tc: for M-tile mt (K rows mt*RPT ...), K-block kb (o = kb*KB ...):
// [hi | lo] each [2 chunks][128 rows][8] bf16, row r <-> K row mt*RPT + r (r < RPT), zero outside.
__global__ void k_tile_w_dgr(const float* __restrict__ W, uint16_t* __restrict__ Wt, int O, int I, int B, int RPT,
                             int nmt) {
  const int nkb = O / TC_KB;
  const int64_t per = 128 * TC_KB;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= per * nkb * nmt) return;
  const int64_t blk = t / per;
  const int r8 = (int)(t - blk * per);             // (ch*128 + row)*8 + e
  const int mt = (int)(blk / nkb), kb = (int)(blk - (int64_t)mt * nkb);
  const int e = r8 & 7, row = (r8 >> 3) & 127, ch = r8 >> 10;
  const int o = kb * TC_KB + 8 * ch + e;
  const int64_t kr = (int64_t)mt * RPT + row, K = (int64_t)I * B;
  const float w = (row < RPT && kr < K) ? W[(int64_t)o * K + kr] : 0.f;
  uint16_t hi, lo;
  tc::split1_bf16(w, hi, lo);
  uint16_t* dst = Wt + blk * 2 * per;
  dst[r8] = hi;
  dst[per + r8] = lo;
}

template <int NF, int NS, int M, int OO>
__global__ void __launch_bounds__(DgrCfg<NF, NS, M, OO>::THREADS, 1)
    k_dgrad_tc(const __grid_constant__ CUtensorMap tmX, const uint16_t* __restrict__ Ysplit,
               const uint16_t* __restrict__ Wtiled, float* __restrict__ Xbar, int64_t P, int I, int RPT, int nmt,
               BasisCfg bc, int dbg) {
  using Cfg = DgrCfg<NF, NS, M, OO>;
  constexpr int C = Cfg::C, NP = Cfg::NP, N = Cfg::N, NKB = Cfg::NKB, NSTAGE = Cfg::NSTAGE;
  constexpr int SLICE_P = Cfg::SLICE_P;
  constexpr int DGR_EPI_WARPS = Cfg::EPI_WARPS, DGR_MMA_WARP = Cfg::MMA_WARP, DGR_PROD_WARP = Cfg::PROD_WARP;
  constexpr int NEPI = 32 * DGR_EPI_WARPS;
  constexpr int NH = DGR_EPI_WARPS / 4;                       // epilogue warps per TMEM lane quadrant
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared address space visible to the compiler (STS/LDS, not generic ST/LD)
  float* jets = reinterpret_cast<float*>(smem + NSTAGE * Cfg::STAGE_BYTES);   // [2][NP][C][IPTB] input jets
  float* S = jets + 2 * Cfg::JET_FLOATS;                      // epilogue slice [SLICE_P*C][DGR_SST]
  float* carry = S + Cfg::S_FLOATS;                           // [2][NP][C] partial adjoints of split inputs
  __shared__ __align__(8) uint64_t full_bar[NSTAGE], empty_bar[NSTAGE], acc_full[2], acc_empty[2];
  __shared__ __align__(8) uint64_t jet_full[2], jet_empty[2];
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // persistent (one CTA per SM): point tiles blockIdx.x + jt*gridDim.x, each run as nmt M-tiles; the
  // global M-tile counter gm = jt*nmt + mt drives the accumulator / jet-box / carry double buffers and
  // g = gm*NKB + kb the stage ring, so tile jt+1's MMAs overlap tile jt's epilogue
  const int64_t ntiles = (P + NP - 1) / NP;
  const int ntl = (int)((ntiles - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);
  const int nmt_tot = ntl * nmt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&acc_full[a], 1);
      tc::mbar_init(&acc_empty[a], NEPI);
      tc::mbar_init(&jet_full[a], 1);
      tc::mbar_init(&jet_empty[a], DGR_EPI_WARPS);   // one elected lane per epilogue warp
    }
    tc::fence_mbar_init();
  }
  if (warp == DGR_MMA_WARP) tc::tmem_alloc<Cfg::TMEM_COLS>(&tmem_base_sh);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp < DGR_EPI_WARPS) {
    // ===================== epilogue: per M-tile, TMEM -> smem slices -> jet-chain gather
    const int qw = warp & 3;                      // TMEM lane quadrant (warp % 4)
    const int half = warp >> 2;                   // which of the NH column phases this warp drains
    const int etid = threadIdx.x;
    const int r = qw * 32 + lane;                 // accumulator row = il*B + n
#pragma unroll 1
    for (int gm = 0; gm < nmt_tot; ++gm) {
      const int jt = gm / nmt, mt = gm - jt * nmt;
      const int64_t p0 = ((int64_t)blockIdx.x + (int64_t)jt * gridDim.x) * NP;
      const int buf = gm & 1;
      tc::mbar_wait(&acc_full[buf], (uint32_t)((gm >> 1) & 1));
      tc::tc_fence_after();
      tc::mbar_wait(&jet_full[buf], (uint32_t)((gm >> 1) & 1));
      const int B = bc.B;
      const int row0 = mt * RPT, nrows = min(RPT, I * B - row0);   // this tile's K rows
      const int i_first = row0 / B, n_in = (row0 + nrows - 1) / B - i_first + 1;
      const float* js = jets + buf * Cfg::JET_FLOATS + (i_first & 3);   // [NP][C][IPTB] from input i_first & ~3
#pragma unroll 1
      for (int sl = 0; sl < NP / SLICE_P; ++sl) {
        const uint32_t tb = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)(buf * N + sl * SLICE_P * C);
#pragma unroll 1
        for (int c8 = half * 8; c8 < SLICE_P * C; c8 += 8 * NH) {
          float v[8];
          tc::tmem_ld8(tb + c8, v);
#pragma unroll
          for (int q = 0; q < 8; ++q) S[(c8 + q) * DGR_SST + r] = v[q];
        }
        if (sl == NP / SLICE_P - 1) {             // accumulator fully read: release it early
          tc::tc_fence_before();
          tc::mbar_arrive(&acc_empty[buf]);
        }
        tc::named_bar_sync(1, NEPI);
        // task = (point pq, input il), input fastest: Xbar stores run along i
        for (int task = etid; task < ((dbg & 4) ? 0 : SLICE_P * n_in); task += NEPI) {
          const int il = task % n_in, pq = task / n_in;
          const int pl = sl * SLICE_P + pq;
          const int64_t p = p0 + pl;
          const int i = i_first + il;
          if (p >= P) continue;
          const int n_lo = max(0, row0 - i * B), n_hi = min(B, row0 + nrows - i * B);   // this tile's bases of i
          const float* jq = js + (pl * C) * DGR_IPTB + il;
          const float x = jq[0];
          float dx[NF > 0 ? NF : 1], ddx[NS > 0 ? NS : 1];
#pragma unroll
          for (int a = 0; a < NF; ++a) dx[a] = jq[(1 + a) * DGR_IPTB];
#pragma unroll
          for (int a = 0; a < NS; ++a) ddx[a] = jq[(1 + NF + a) * DGR_IPTB];
          const int n0 = first_basis(x, bc);
          float xb = 0.f, dxb[NF > 0 ? NF : 1], ddxb[NS > 0 ? NS : 1];
#pragma unroll
          for (int a = 0; a < NF; ++a) dxb[a] = 0.f;
#pragma unroll
          for (int a = 0; a < NS; ++a) ddxb[a] = 0.f;
          const float* Sp = S + (pq * C) * DGR_SST + (i * B - row0);   // row of basis n: i*B + n - row0
#if HRKAN_DGR_F32X2
          if constexpr (M >= 4) {
            // two bases per instruction (FFMA2/FMUL2); t clamped at 0 (NaN kept) zeroes v1..v3 outside
            // the support and for bases outside this tile (m >= 4); their smem rows are clamped in range
            const uint64_t ONE2 = tc::pk2(1.f, 1.f), NEG2 = tc::pk2(-1.f, -1.f);
            const float sc = bc.sc, k2 = -(2.f * M - 1.f);
            const uint64_t C12 = tc::pk2(-2.f * M * sc, -2.f * M * sc);
            const uint64_t C22 = tc::pk2(-2.f * M * sc * sc, -2.f * M * sc * sc);
            const uint64_t C32 = tc::pk2(4.f * M * (M - 1) * sc * sc * sc, 4.f * M * (M - 1) * sc * sc * sc);
            const uint64_t K22 = tc::pk2(k2, k2), THREE2 = tc::pk2(3.f, 3.f), TWO2 = tc::pk2(2.f, 2.f);
            uint64_t xb2 = tc::pk2(0.f, 0.f), dxb2[NF > 0 ? NF : 1], ddxb2[NS > 0 ? NS : 1], dx2[NF > 0 ? NF : 1],
                     ddx2[NS > 0 ? NS : 1];
#pragma unroll
            for (int a = 0; a < NF; ++a) { dxb2[a] = xb2; dx2[a] = tc::pk2(dx[a], dx[a]); }
#pragma unroll
            for (int a = 0; a < NS; ++a) { ddxb2[a] = xb2; ddx2[a] = tc::pk2(ddx[a], ddx[a]); }
#pragma unroll
            for (int rr = 0; rr < KMAX; rr += 2) {
              if (rr > bc.k) break;
              const int na = n0 + rr, nb = n0 + rr + 1;
              const bool oka = na >= n_lo && na < n_hi, okb = rr + 1 <= bc.k && nb >= n_lo && nb < n_hi;
              const int ca = oka ? na : n_lo, cb = okb ? nb : n_lo;          // in-tile rows for the loads
              const uint64_t qq = tc::pk2(basis_q(x, na, bc), basis_q(x, nb, bc));
              const uint64_t q2 = tc::mul2(qq, qq);
              float t0, t1;
              tc::upk2(tc::fma2(q2, NEG2, ONE2), t0, t1);
              t0 = oka ? tc::max_nan(t0, 0.f) : 0.f;
              t1 = okb ? tc::max_nan(t1, 0.f) : 0.f;
              const uint64_t t = tc::pk2(t0, t1);
              uint64_t tm3 = ONE2;
#pragma unroll
              for (int e = 0; e < M - 3; ++e) tm3 = tc::mul2(tm3, t);
              const uint64_t tm2 = tc::mul2(tm3, t), tm1 = tc::mul2(tm2, t);
              const uint64_t v1 = tc::mul2(tc::mul2(qq, tm1), C12);
              const uint64_t kq = tc::fma2(q2, K22, ONE2);                      // 1 - (2m-1) q^2
              const uint64_t v2 = tc::mul2(tc::mul2(tm2, kq), C22);
              const uint64_t v3 = tc::mul2(tc::mul2(tc::mul2(qq, tm3), tc::fma2(q2, K22, THREE2)), C32);
              uint64_t ab[C];
#pragma unroll
              for (int c = 0; c < C; ++c) ab[c] = tc::pk2(Sp[c * DGR_SST + ca], Sp[c * DGR_SST + cb]);
              xb2 = tc::fma2(ab[0], v1, xb2);
#pragma unroll
              for (int a = 0; a < NF; ++a) {
                xb2 = tc::fma2(tc::mul2(ab[1 + a], v2), dx2[a], xb2);
                dxb2[a] = tc::fma2(ab[1 + a], v1, dxb2[a]);
              }
#pragma unroll
              for (int a = 0; a < NS; ++a) {
                const uint64_t g = ab[1 + NF + a];
                xb2 = tc::fma2(g, tc::fma2(tc::mul2(v3, dx2[a]), dx2[a], tc::mul2(v2, ddx2[a])), xb2);
                dxb2[a] = tc::fma2(tc::mul2(TWO2, tc::mul2(g, v2)), dx2[a], dxb2[a]);
                ddxb2[a] = tc::fma2(g, v1, ddxb2[a]);
              }
            }
            float lo_, hi_;
            tc::upk2(xb2, lo_, hi_);
            xb = lo_ + hi_;
#pragma unroll
            for (int a = 0; a < NF; ++a) { tc::upk2(dxb2[a], lo_, hi_); dxb[a] = lo_ + hi_; }
#pragma unroll
            for (int a = 0; a < NS; ++a) { tc::upk2(ddxb2[a], lo_, hi_); ddxb[a] = lo_ + hi_; }
          } else {
#endif
#pragma unroll
          for (int rr = 0; rr < KMAX; ++rr) {
            if (rr > bc.k) break;
            const int n = n0 + rr;
            if (n < n_lo || n >= n_hi) continue;
            float v0, v1, v2, v3;
            hr_eval<M, (NS > 0 ? 3 : 2)>(basis_q(x, n, bc), bc.sc, v0, v1, v2, v3);
            float ab[C];
#pragma unroll
            for (int c = 0; c < C; ++c) ab[c] = Sp[c * DGR_SST + n];
            xb = fmaf(ab[0], v1, xb);
#pragma unroll
            for (int a = 0; a < NF; ++a) {
              xb = fmaf(ab[1 + a] * v2, dx[a], xb);
              dxb[a] = fmaf(ab[1 + a], v1, dxb[a]);
            }
#pragma unroll
            for (int a = 0; a < NS; ++a) {
              const float g = ab[1 + NF + a];
              xb = fmaf(g, fmaf(v3 * dx[a], dx[a], v2 * ddx[a]), xb);
              dxb[a] = fmaf(2.f * g * v2, dx[a], dxb[a]);
              ddxb[a] = fmaf(g, v1, ddxb[a]);
            }
          }
#if HRKAN_DGR_F32X2
          }
#endif
          // carries alternate by tile parity: a tile reads its predecessor's and writes its own
          if (n_lo > 0) {                          // input started in the previous tile: add its part
            const float* cp = carry + (((gm + 1) & 1) * NP + pl) * C;
            xb += cp[0];
#pragma unroll
            for (int a = 0; a < NF; ++a) dxb[a] += cp[1 + a];
#pragma unroll
            for (int a = 0; a < NS; ++a) ddxb[a] += cp[1 + NF + a];
          }
          float* cp = carry + ((gm & 1) * NP + pl) * C;
          if (n_hi < B) {                          // input continues in the next tile: carry the part
            cp[0] = xb;
#pragma unroll
            for (int a = 0; a < NF; ++a) cp[1 + a] = dxb[a];
#pragma unroll
            for (int a = 0; a < NS; ++a) cp[1 + NF + a] = ddxb[a];
            continue;
          }
          float* out = Xbar + p * (int64_t)(C * I) + i;
          out[0] = xb;
#pragma unroll
          for (int a = 0; a < NF; ++a) out[(1 + a) * I] = dxb[a];
#pragma unroll
          for (int a = 0; a < NS; ++a) out[(1 + NF + a) * I] = ddxb[a];
        }
        tc::named_bar_sync(1, NEPI);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&jet_empty[buf]);
    }
  } else if (warp == DGR_MMA_WARP) {
    {   // the whole warp runs the issue loop, one elected lane issues (tc::mma_bf16_w)
      constexpr uint32_t idesc = tc::idesc_bf16(128, N);
      int s = 0;
      uint32_t ph = 0;
#pragma unroll 1
      for (int gm = 0; gm < nmt_tot; ++gm) {
        const int buf = gm & 1;
        if (gm >= 2) {
          tc::mbar_wait(&acc_empty[buf], (uint32_t)(((gm >> 1) - 1) & 1));
          tc::tc_fence_after();
        }
#pragma unroll 1
        for (int kb = 0; kb < NKB; ++kb) {
          tc::mbar_wait(&full_bar[s], ph);
          tc::tc_fence_after();
          const uint32_t w_hi = tc::smem_u32(smem + s * Cfg::STAGE_BYTES);
          const uint32_t w_lo = w_hi + 2 * 128 * 16;
          const uint32_t y_hi = w_hi + Cfg::W_STAGE_BYTES;
          const uint32_t y_lo = y_hi + 2 * N * 16;
          const uint64_t wh = tc::smem_desc(w_hi, 128 * 16, 128);
          const uint64_t wl = tc::smem_desc(w_lo, 128 * 16, 128);
          const uint64_t yh = tc::smem_desc(y_hi, N * 16, 128);
          const uint64_t yl = tc::smem_desc(y_lo, N * 16, 128);
          const uint32_t d = tmem + (uint32_t)(buf * N);
          tc::mma_bf16_w(d, wl, yh, idesc, kb > 0 ? 1u : 0u);
          tc::mma_bf16_w(d, wh, yl, idesc, 1u);
          tc::mma_bf16_w(d, wh, yh, idesc, 1u);
          tc::mma_commit_w(&empty_bar[s]);
          if (++s == NSTAGE) { s = 0; ph ^= 1u; }
        }
        tc::mma_commit_w(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else if (warp == DGR_PROD_WARP) {
    // ===================== producer: W^T and pre-split Ybar stages (1-D bulk copies); never waits on the
    // epilogue, so the MMA is only held back by the TMEM accumulators it releases early
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int jt = 0; jt < ntl; ++jt) {
        const uint16_t* ytile = Ysplit + ((int64_t)blockIdx.x + (int64_t)jt * gridDim.x) * NKB * (Cfg::Y_STAGE_BYTES / 2);
        for (int g = 0; g < nmt * NKB; ++g) {       // W^T stage g = mt*NKB + kb of this point tile
          const int kb = g - (g / NKB) * NKB;
          tc::mbar_wait(&empty_bar[s], ph ^ 1u);
          tc::mbar_arrive_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
          tc::bulk_g2s(smem + s * Cfg::STAGE_BYTES, Wtiled + (int64_t)g * (Cfg::W_STAGE_BYTES / 2), Cfg::W_STAGE_BYTES,
                       &full_bar[s]);
          tc::bulk_g2s(smem + s * Cfg::STAGE_BYTES + Cfg::W_STAGE_BYTES, ytile + (int64_t)kb * (Cfg::Y_STAGE_BYTES / 2),
                       Cfg::Y_STAGE_BYTES, &full_bar[s]);
          if (++s == NSTAGE) { s = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== jet producer: input-jet boxes of the M-tiles (TMA), two tiles ahead of use
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmX);
      for (int gm = 0; gm < nmt_tot; ++gm) {
        const int jt = gm / nmt, mt = gm - jt * nmt;
        const int p0 = (int)(((int64_t)blockIdx.x + (int64_t)jt * gridDim.x) * NP);
        const int jb = gm & 1;
        if (gm >= 2) tc::mbar_wait(&jet_empty[jb], (uint32_t)(((gm >> 1) - 1) & 1));
        tc::mbar_arrive_expect_tx(&jet_full[jb], Cfg::JET_FLOATS * 4);
        tc::tma_load_3d(jets + jb * Cfg::JET_FLOATS, &tmX, ((mt * RPT) / bc.B) & ~3, 0, p0, &jet_full[jb]);
      }
    }
    __syncwarp();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == DGR_MMA_WARP) tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
}

}  // namespace
