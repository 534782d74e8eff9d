// tc_kernels.cuh -- tcgen05 / TMEM tensor-core engine for the wide hidden layers (sm_100a).
//
// The hidden KAN layer is the dense contraction of PAPER.md:45/:87 ("KAN layer as a matrix
// operation") applied to every jet channel:
//     Y[(p,c), o] = sum_{K=(i,n)} A^c[p, K] W[o, K]      (+ b_o on the value channel c = 0)
// with A^c generated on the fly from the saved input jet.  It runs as bf16x3 on
// the 5th-generation tensor cores: W and A are split into bf16 hi/lo parts and
//     D += W_lo A_hi + W_hi A_lo + W_hi A_hi
// accumulate in fp32 TMEM, which meets the north-star tolerance.
//
// Forward kernel k_fwd_tc (orientation "W rows x (point,channel) columns"):
//   MMA M = output neurons o (128-row tiles; O = 64/128 -> 1 zero-padded or full tile, 256 -> 2 tiles
//   sharing the B tile), MMA N = NP points x C channels of one point tile (channel-major columns
//   n = c*NP + p), MMA K = I*B (dense over all bases, zero-padded to a multiple of KB).
//   smem stage = { W_hi, W_lo tiles [2 chunks][OP rows][8] bf16 via one 1-D bulk copy of a pre-tiled
//                  global copy;  A_hi, A_lo tiles [2 chunks][N rows][8] written by the generator
//                  warps }, NSTAGE-deep mbarrier ring.  The generators read the saved input jet from
//   a ring of TMA-loaded windows X[tile points][C|1][4 inputs] (coalesced, prefetched ahead).
//   warps 0 .. 4*NGEN-1: NGEN generator groups (K-blocks kb = grp mod NGEN), which also drain the
//   TMEM segments (+bias -> Y[p][c][o], coalesced); then the MMA warp (TMEM allocator + single-thread
//   tcgen05.mma issuer), the W bulk-copy warp and the jet-window TMA warp (FwdCfg::*_WARP).
#pragma once
#ifndef HRKAN_FWD_NSTAGE_MAX
#define HRKAN_FWD_NSTAGE_MAX 6   // stage-ring depth cap (shared memory permitting)
#endif
#include "tc_ptx.cuh"

namespace {

using namespace hrkan;

constexpr int TC_KB = 16;          // K per pipeline stage (one bf16 MMA K-step)
constexpr int TC_GEN_THREADS = 128;   // one generator group (4 warps); the group handles every other K-block
// Generator groups (all also drain the accumulators): 4 where the register budget of 19 warps allows
// it without spills (measured: C4 forward 4.24 -> 3.78 ms, C3 1.83 -> 1.68 ms per 2^18 points), else 3
// (C = 3 and C = 5 at O >= 128 spill with 4; C5's C = 7 layer was 2 % slower with 4).
// forward generator arithmetic on packed fp32 pairs (two K slots per FFMA2/FMUL2) for m >= 3
// (C4 forward 3.16 -> 2.75 ms, C3 1.42 -> 1.25 ms, C5 10.8 -> 10.5 ms per 2^18 points)
#ifndef HRKAN_FWD_F32X2
#define HRKAN_FWD_F32X2 1
#endif
#ifndef HRKAN_FWD_NGEN
#define HRKAN_FWD_NGEN 0
#endif
__host__ __device__ constexpr int tc_ngen(int C, int O) {
  return HRKAN_FWD_NGEN > 0 ? HRKAN_FWD_NGEN : (C == 1 || C == 4 || O <= 64) ? 4 : 3;
}
#ifndef HRKAN_FWD_NOCROSS
#define HRKAN_FWD_NOCROSS 0       // 1: TIMING EXPERIMENT ONLY (wrong results): K chunks never read the next input's jets
#endif
#ifndef HRKAN_FWD_SWAP
#define HRKAN_FWD_SWAP 0          // 1: O = 64 forward with (channel, point) rows on the MMA M side (FwdCfg::SW; measured 12 % slower on C3, off)
#endif
constexpr int TC_WIN = 4;             // inputs per jet window (16-B TMA rows)
constexpr int TC_NWIN = 8;            // jet-window ring depth

// Points per tile so that N = NP*C is a multiple of 16 and <= 256.
__host__ __device__ constexpr int tc_np(int C) {
  return C == 7 ? 32 : C == 5 ? 48 : C == 4 ? 64 : C == 3 ? 80 : C == 1 ? 256 : 0;
}

__host__ __device__ constexpr uint32_t tc_tmem_cols(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int NF, int NS, int M, int OO>
struct FwdCfg {
  static constexpr int C = 1 + NF + NS;
  static constexpr int NP = tc_np(C);
  static constexpr int N = NP * C;
  static constexpr int O = OO;                               // output neurons (64, 128 or 256)
  // O = 64 runs SWAPPED: M = 128 generated (channel, point) rows, two M-tiles over a 256-row operand,
  // N = the 64 output neurons -- the MMA then costs 2 x 128x64 instead of a zero-padded 128 x N
  // (tcgen05 issue floor max(M,128)*N/256 cycles: 64 vs 120 per K-step for C = 5)
  static constexpr bool SW = HRKAN_FWD_SWAP && (OO == 64);
  static constexpr int NROW = SW ? 256 : N;                  // rows of the generated operand buffer
  static constexpr int NMT = SW ? 2 : (OO + 127) / 128;      // 128-row M-tiles (of W, or of the generated rows)
  static constexpr int OP = SW ? 64 : 128 * NMT;             // rows of the W tiles (zero-padded when not swapped)
  static constexpr int ACC_COLS = SW ? NMT * O : NMT * N;    // TMEM columns of one accumulator
  // bf16 operands, K-major, SWIZZLE_NONE: a K-block of 16 = 2 chunks of 8 elements (16 B per row).
  // Generated operand chunk stride padded to 64 B (mod 128 B): the generators' 8-B stores
  // (4 consecutive K of one row, chunk-fastest lanes) are bank-conflict free.
  static constexpr int ACSB = NROW * 16 + 64;                // chunk stride (bytes)
  static constexpr int W_STAGE_BYTES = 2 * 2 * OP * 16;      // hi + lo, [2 chunks][OP rows][8] each
  static constexpr int A_STAGE_BYTES = 2 * 2 * ACSB;         // hi + lo, [2 chunks][N rows][8] each
  static constexpr int STAGE_BYTES = W_STAGE_BYTES + A_STAGE_BYTES;
  static constexpr int CB = C | 1;                           // box channels (odd: conflict-free window reads)
  static constexpr int WIN_FLOATS = NP * CB * TC_WIN;        // TMA box [NP points][CB][TC_WIN inputs]
  static constexpr int FIXED_BYTES = 4 * TC_NWIN * WIN_FLOATS + 2 * 4 * 256 + 1024;   // windows, ctr, -ctr*sc
  static constexpr int NSTAGE_FIT = (225 * 1024 - FIXED_BYTES) / STAGE_BYTES;   // static smem + margin
  static constexpr int NSTAGE = NSTAGE_FIT > HRKAN_FWD_NSTAGE_MAX ? HRKAN_FWD_NSTAGE_MAX : NSTAGE_FIT;
  static constexpr int SMEM_BYTES = NSTAGE * STAGE_BYTES + FIXED_BYTES;
  static constexpr int NACC = (2 * ACC_COLS <= 512) ? 2 : 1;  // double-buffered accumulators if they fit
  static constexpr int NGEN = tc_ngen(C, OO);
  static constexpr int MMA_WARP = 4 * NGEN, PROD_WARP = 4 * NGEN + 1, WIN_WARP = 4 * NGEN + 2;
  static constexpr int THREADS = 32 * (4 * NGEN + 3);        // + MMA warp + W producer warp + jet-window TMA warp
  static constexpr uint32_t TMEM_COLS = tc_tmem_cols(NACC * ACC_COLS);
  static_assert(N % 16 == 0 && N <= 256, "bad N");
  static_assert(ACC_COLS <= 512, "accumulators exceed TMEM");
  static_assert(NSTAGE >= 2, "shared memory budget");
  static_assert(STAGE_BYTES % 128 == 0, "TMA windows after the stages need 128-B alignment");
  // groups write alternate K-blocks: a group's previous stage is NGEN back, so its lead over the oldest
  // unconsumed stage stays below two laps of the ring (no parity aliasing on empty_bar) iff NGEN <= NSTAGE
  static_assert(NGEN <= NSTAGE, "stage ring shallower than the generator groups");
};

// Pre-tiled, pre-split weights for k_fwd_tc: for K-block kb: [hi | lo] each [2 chunks][OP][8] bf16
// (rows o >= O are zero: a 64-neuron layer runs as one zero-padded 128-row M-tile).
__global__ void k_tile_w_fwd(const float* __restrict__ W, uint16_t* __restrict__ Wt, int O, int OP, int K, int nkb) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per_kb = (int64_t)OP * TC_KB;        // elements of one of hi / lo per K-block
  if (t >= per_kb * nkb) return;
  const int kb = (int)(t / per_kb);
  const int r = (int)(t - (int64_t)kb * per_kb);     // r = (chunk*OP + o)*8 + e
  const int e = r & 7, o = (r >> 3) % OP, ch = (r >> 3) / OP;
  const int k = kb * TC_KB + 8 * ch + e;
  const float w = (k < K && o < O) ? W[(int64_t)o * K + k] : 0.f;
  uint16_t hi, lo;
  tc::split1_bf16(w, hi, lo);
  uint16_t* dst = Wt + (int64_t)kb * 2 * per_kb;
  dst[r] = hi;
  dst[per_kb + r] = lo;
}

// Forward hidden layer.  Warp roles (FwdCfg: NGEN = 3 or 4 generator groups of 4 warps):
//   warps 0 .. 4*NGEN-1   generator groups (K-blocks kb = grp mod NGEN), then the segment drains;
//   MMA_WARP              TMEM allocator + single-thread tcgen05.mma issuer;
//   PROD_WARP             1-D bulk copies of the pre-tiled W_hi/W_lo stage;
//   WIN_WARP              TMA loads of jet windows X[p0 .. p0+NP)[C|1][4w .. 4w+4) -> smem ring
//                         (TC_NWIN deep), so the generators read the jets from shared memory.
template <int NF, int NS, int M, int OO>
__global__ void __launch_bounds__(FwdCfg<NF, NS, M, OO>::THREADS, 1)
    k_fwd_tc(const __grid_constant__ CUtensorMap tmX, const uint16_t* __restrict__ Wtiled, const float* __restrict__ bias,
             float* __restrict__ Y, int64_t P, int I, int nkb, int seg, BasisCfg bc, int dbg) {
  using Cfg = FwdCfg<NF, NS, M, OO>;
  constexpr int C = Cfg::C, NP = Cfg::NP, N = Cfg::N, O = Cfg::O, NACC = Cfg::NACC, NSTAGE = Cfg::NSTAGE;
  constexpr int NMT = Cfg::NMT, OP = Cfg::OP;
  constexpr int ACSB = Cfg::ACSB;
  constexpr int TC_NGEN = Cfg::NGEN, TC_MMA_WARP = Cfg::MMA_WARP, TC_PROD_WARP = Cfg::PROD_WARP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps the shared address space visible to the compiler (STS/LDS, not generic ST/LD)
  float* win = reinterpret_cast<float*>(smem + NSTAGE * Cfg::STAGE_BYTES);   // [TC_NWIN][NP][C][TC_WIN]
  float* ctr = win + TC_NWIN * Cfg::WIN_FLOATS;              // basis centres mid_n, n < B
  float* ncs = ctr + 256;                                     // -mid_n * sc (packed-pair generator)
  __shared__ __align__(8) uint64_t full_bar[NSTAGE], empty_bar[NSTAGE], acc_full[NACC], acc_empty[NACC];
  __shared__ __align__(8) uint64_t win_full[TC_NWIN], win_empty[TC_NWIN];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)blockIdx.x * NP;
  const int K = I * bc.B;
  const int nseg = (nkb + seg - 1) / seg;
  const int nwin = (I + TC_WIN - 1) / TC_WIN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      tc::mbar_init(&full_bar[s], (TC_GEN_THREADS / 32) * tc::ARRIVALS_PER_WARP + 1);   // one generator group + W producer
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      tc::mbar_init(&acc_full[a], 1);
      tc::mbar_init(&acc_empty[a], TC_GEN_THREADS * TC_NGEN);
    }
    for (int w = 0; w < TC_NWIN; ++w) {
      tc::mbar_init(&win_full[w], 1);
      tc::mbar_init(&win_empty[w], 4 * TC_NGEN);           // one elected lane per generator warp
    }
    tc::fence_mbar_init();
  }
  for (int n = threadIdx.x; n < bc.B; n += blockDim.x) {
    ctr[n] = fmaf((float)n, bc.h, bc.mid0);
    ncs[n] = -ctr[n] * bc.sc;
  }
  if (warp == TC_MMA_WARP) tc::tmem_alloc<Cfg::TMEM_COLS>(&tmem_base_sh);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp < 4 * TC_NGEN) {
    const int grp = warp >> 2;                 // generator group: K-blocks kb = grp (mod TC_NGEN)
    const int gtid = threadIdx.x & (TC_GEN_THREADS - 1);
    const int qw = warp & 3;                   // TMEM lane quadrant of this warp
    // Drain K-segment sg: TMEM accumulator -> Y (first segment: = D + bias; later: += D), fp32 RN.
    // Bounds the tensor core's accumulation error to one segment.
    auto drain = [&](int sg) {
      const int buf = sg % NACC;
      tc::mbar_wait(&acc_full[buf], (uint32_t)((sg / NACC) & 1));
      tc::tc_fence_after();
      if constexpr (Cfg::SW) {
        // swapped: TMEM lane = generated row (c, p) of M-tile t, columns = the 64 outputs; the
        // (M-tile, 16-output chunk) units are shared round-robin by the generator groups
#pragma unroll 1
        for (int u = grp; u < NMT * (O / 16); u += TC_NGEN) {
          const int t = u / (O / 16), o0 = (u % (O / 16)) * 16;
          const int r = t * 128 + qw * 32 + lane;
          const int c = r / NP, pl = r - (r / NP) * NP;
          const int64_t p = p0 + pl;
          const bool ok = r < N && p < P;
          float v[16];
          tc::tmem_ld16(tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)((buf * NMT + t) * O + o0), v);
          float4* yp = reinterpret_cast<float4*>(Y + (p * C + c) * (int64_t)O + o0);
          if (ok) {
            if (sg == 0 && c == 0) {
#pragma unroll
              for (int q = 0; q < 16; ++q) v[q] += __ldg(bias + o0 + q);
            }
            if (sg > 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 old = yp[q];
                v[4 * q] += old.x; v[4 * q + 1] += old.y; v[4 * q + 2] += old.z; v[4 * q + 3] += old.w;
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) yp[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      } else {
#pragma unroll 1
      for (int t = 0; t < NMT; ++t) {
        if (t * 128 + qw * 32 >= O) continue;        // zero-padded rows of a 64-neuron layer: nothing to store
        const int o = t * 128 + qw * 32 + lane;
        const float b = (sg == 0) ? __ldg(bias + o) : 0.f;
        const uint32_t tbase = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)((buf * NMT + t) * N);
        // 16-column chunks are shared round-robin by the generator groups (same lane quadrant); column
        // col = c*NP + pl -> Y[p0 + pl][c][o] at a 32-bit offset from this lane's base (few live registers)
        const int lim = (P - p0 < (int64_t)NP) ? (int)(P - p0) : NP;
        float* yb = Y + p0 * (C * O) + o;
#pragma unroll 1
        for (int c0 = 16 * grp; c0 < N; c0 += 16 * TC_NGEN) {
          float v[16];
          tc::tmem_ld16(tbase + c0, v);
          if (sg == 0) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < NP) v[q] += b;             // value channel c = 0
          } else {
            float old[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {             // 16 loads in flight
              const int col = c0 + q, c = col / NP, pl = col - c * NP;
              old[q] = (pl < lim) ? yb[(pl * C + c) * O] : 0.f;
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += old[q];
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int col = c0 + q, c = col / NP, pl = col - c * NP;
            if (pl < lim) yb[(pl * C + c) * O] = v[q];
          }
        }
      }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[buf]);
    };
    // ===================== generators: A^c[p, k] for the stage's KB columns.
    // Task = (point pl, 4-wide K chunk j), chunk fastest across lanes; the jets come from the TMA
    // window ring.  K positions advance incrementally (no integer division in the loop).
    constexpr int NTASK = NP * (TC_KB / 4);
    constexpr int TPT = (NTASK + TC_GEN_THREADS - 1) / TC_GEN_THREADS;
    const int j = gtid & 3;                    // fixed chunk of this thread (TC_GEN_THREADS % 4 == 0)
    const int B = bc.B;
    int i0, n0;                                // task K position k0 = kb*KB + 4j -> (input i0, basis n0)
    int ilo, nlo;                              // K-block start kb*KB -> (ilo, nlo)
    {
      const int k0 = grp * TC_KB + 4 * j;
      i0 = k0 / B;
      n0 = k0 - i0 * B;
      ilo = (grp * TC_KB) / B;
      nlo = grp * TC_KB - ilo * B;
    }
    const int dstep = TC_KB * TC_NGEN;         // K advance per group step
    const int di = dstep / B, dn = dstep - (dstep / B) * B;
    int wwait = 0, wrel = 0;                   // next window to wait for / to release
    int next_drain = 0;
    for (int kb = grp; kb < nkb; kb += TC_NGEN) {
      while (next_drain < nseg - 1 && kb >= (next_drain + 1) * seg + NSTAGE) drain(next_drain++);
      // windows: release those below this K-block's first input, wait for those up to its last
      const int ihi = min(I - 1, ilo + (nlo + TC_KB - 1 >= B) + (nlo + TC_KB - 1 >= 2 * B));
      while (wrel < ilo / TC_WIN) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&win_empty[wrel % TC_NWIN]);
        ++wrel;
      }
      while (wwait <= ihi / TC_WIN) {
        tc::mbar_wait(&win_full[wwait % TC_NWIN], (uint32_t)((wwait / TC_NWIN) & 1));
        ++wwait;
      }
      const int s = kb % NSTAGE;
      tc::mbar_wait(&empty_bar[s], ((kb / NSTAGE) & 1) ^ 1);
      uint8_t* a_hi = smem + s * Cfg::STAGE_BYTES + Cfg::W_STAGE_BYTES;
      uint8_t* a_lo = a_hi + 2 * ACSB;
      const int aoff = (j >> 1) * ACSB + (j & 1) * 8;    // chunk j/2, half j%2 of the 16-B row
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int task = gtid + u * TC_GEN_THREADS;
        if (task >= NTASK || (dbg & 1)) break;    // dbg bit 0: skip generation (timing experiments only)
        const int pl = task >> 2;
        // jets of inputs i0 and i0+1 (the chunk crosses into i0+1 when n0 + 3 >= B)
        float jx[2], jdx[2][NF > 0 ? NF : 1], jddx[2][NS > 0 ? NS : 1];
#pragma unroll
        for (int h = 0; h < (HRKAN_FWD_NOCROSS ? 1 : 2); ++h) {
          const int i = i0 + h;
          const float* wp = win + ((i / TC_WIN) % TC_NWIN) * Cfg::WIN_FLOATS + (pl * Cfg::CB) * TC_WIN + (i % TC_WIN);
          jx[h] = wp[0];
#pragma unroll
          for (int a = 0; a < NF; ++a) jdx[h][a] = wp[(1 + a) * TC_WIN];
#pragma unroll
          for (int a = 0; a < NS; ++a) jddx[h][a] = wp[(1 + NF + a) * TC_WIN];
        }
        float va[C][4];
#if HRKAN_FWD_F32X2
        if constexpr (M >= 3) {
          // two K slots per instruction (FFMA2/FMUL2); same formulas as hr_eval with t clamped at 0
          // (NaN kept), so every derivative vanishes outside the support (m >= 3)
          const uint64_t SC2 = tc::pk2(bc.sc, bc.sc), ONE2 = tc::pk2(1.f, 1.f), NEG2 = tc::pk2(-1.f, -1.f);
          const float c1 = -2.f * M * bc.sc, c2 = -2.f * M * bc.sc * bc.sc, k2 = -(2.f * M - 1.f);
          const uint64_t C12 = tc::pk2(c1, c1), C22 = tc::pk2(c2, c2), K22 = tc::pk2(k2, k2);
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int na = n0 + e, nb = n0 + e + 1;
            const bool ha = !HRKAN_FWD_NOCROSS && na >= B, hb = !HRKAN_FWD_NOCROSS && nb >= B;
            const int nna = ha ? na - B : (HRKAN_FWD_NOCROSS ? min(na, B - 1) : na), nnb = hb ? nb - B : (HRKAN_FWD_NOCROSS ? min(nb, B - 1) : nb);
            const uint64_t qq = tc::fma2(tc::pk2(ha ? jx[1] : jx[0], hb ? jx[1] : jx[0]), SC2, tc::pk2(ncs[nna], ncs[nnb]));
            const uint64_t q2 = tc::mul2(qq, qq);
            float t0, t1;
            tc::upk2(tc::fma2(q2, NEG2, ONE2), t0, t1);
            t0 = (i0 * B + na < K) ? tc::max_nan(t0, 0.f) : 0.f;
            t1 = (i0 * B + nb < K) ? tc::max_nan(t1, 0.f) : 0.f;
            const uint64_t t = tc::pk2(t0, t1);
            uint64_t tm2 = ONE2;
#pragma unroll
            for (int k = 0; k < M - 2; ++k) tm2 = tc::mul2(tm2, t);
            const uint64_t tm1 = tc::mul2(tm2, t);
            tc::upk2(tc::mul2(tm1, t), va[0][e], va[0][e + 1]);
            const uint64_t v1 = tc::mul2(tc::mul2(qq, tm1), C12);
            const uint64_t v2 = tc::mul2(tc::mul2(tm2, tc::fma2(q2, K22, ONE2)), C22);
#pragma unroll
            for (int a = 0; a < NF; ++a) {
              const uint64_t d = tc::pk2(ha ? jdx[1][a] : jdx[0][a], hb ? jdx[1][a] : jdx[0][a]);
              tc::upk2(tc::mul2(v1, d), va[1 + a][e], va[1 + a][e + 1]);
            }
#pragma unroll
            for (int a = 0; a < NS; ++a) {
              const uint64_t d = tc::pk2(ha ? jdx[1][a] : jdx[0][a], hb ? jdx[1][a] : jdx[0][a]);
              const uint64_t dd = tc::pk2(ha ? jddx[1][a] : jddx[0][a], hb ? jddx[1][a] : jddx[0][a]);
              tc::upk2(tc::fma2(tc::mul2(v2, d), d, tc::mul2(v1, dd)), va[1 + NF + a][e], va[1 + NF + a][e + 1]);
            }
          }
        } else {
#endif
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n = n0 + e;
          const bool h = n >= B;                      // chunk crosses into input i0+1
          const int nn = h ? n - B : n;
          const float x = h ? jx[1] : jx[0];
          float v0, v1, v2, v3;
          hr_eval<M, (NS > 0 ? 2 : 1)>((x - ctr[nn]) * bc.sc, bc.sc, v0, v1, v2, v3);
          if (i0 * B + n >= K) v0 = v1 = v2 = 0.f;
          va[0][e] = v0;
#pragma unroll
          for (int a = 0; a < NF; ++a) va[1 + a][e] = v1 * (h ? jdx[1][a] : jdx[0][a]);
#pragma unroll
          for (int a = 0; a < NS; ++a) {
            const float d1 = h ? jdx[1][a] : jdx[0][a];
            const float d2 = h ? jddx[1][a] : jddx[0][a];
            va[1 + NF + a][e] = fmaf(v2 * d1, d1, v1 * d2);
          }
        }
#if HRKAN_FWD_F32X2
        }
#endif
#pragma unroll
        for (int c = 0; c < C; ++c) {
          uint2 hh, ll;
          tc::split4_bf16(make_float4(va[c][0], va[c][1], va[c][2], va[c][3]), hh, ll);
          const int row = c * NP + pl;                  // channel-major columns of the MMA N
          *reinterpret_cast<uint2*>(a_hi + aoff + row * 16) = hh;
          *reinterpret_cast<uint2*>(a_lo + aoff + row * 16) = ll;
        }
      }
      tc::warp_arrive_after_writes(&full_bar[s]);
      // advance to this group's next K-block
      n0 += dn; i0 += di;
      if (n0 >= B) { n0 -= B; ++i0; }
      nlo += dn; ilo += di;
      if (nlo >= B) { nlo -= B; ++ilo; }
    }
    while (next_drain < nseg) drain(next_drain++);
  } else if (warp == TC_MMA_WARP) {
    // ===================== MMA issuer: the whole warp runs the loop, one elected lane issues (tc::mma_bf16_w)
    {
      // dbg bit 6: deliberate deadlock (the issuer waits for its own first commit) -- exercises the hang
      // guard of debug builds (tests/test_gpu_hang_guard.py); never set in production
      if (dbg & 64) tc::mbar_wait(&acc_full[0], 0);
      constexpr uint32_t idesc = Cfg::SW ? tc::idesc_bf16(128, O) : tc::idesc_bf16(128, N);
      // counters and descriptors advance incrementally (no integer division per K-block)
      const uint32_t base = tc::smem_u32(smem);
      const uint64_t bh0 = tc::smem_desc(base + Cfg::W_STAGE_BYTES, ACSB, 128);
      const uint64_t bl0 = tc::smem_desc(base + Cfg::W_STAGE_BYTES + 2 * ACSB, ACSB, 128);
      const uint64_t wh0 = tc::smem_desc(base, OP * 16, 128);
      const uint64_t wl0 = tc::smem_desc(base + 2 * OP * 16, OP * 16, 128);
      int s = 0, segc = 0, buf = 0, sgi = 0;
      uint32_t ph = 0, use0 = 0u, use1 = 0u;
      for (int kb = 0; kb < nkb; ++kb) {
        const bool seg_first = segc == 0;
        if (seg_first && sgi >= NACC) {
          tc::mbar_wait(&acc_empty[buf], ((buf ? use1 : use0) - 1) & 1);
          tc::tc_fence_after();
        }
        tc::mbar_wait(&full_bar[s], ph);
        tc::tc_fence_after();
        const uint64_t off = (uint64_t)((uint32_t)(s * Cfg::STAGE_BYTES) >> 4);
#pragma unroll
        for (int t = 0; t < NMT; ++t) {
          const uint64_t toff = off + (uint64_t)((t * 128 * 16) >> 4);
          if constexpr (Cfg::SW) {            // A = generated rows of M-tile t, B = W (64 rows)
            const uint32_t d = tmem + (uint32_t)((buf * NMT + t) * O);
            tc::mma_bf16_w(d, bl0 + toff, wh0 + off, idesc, seg_first ? 0u : 1u);
            tc::mma_bf16_w(d, bh0 + toff, wl0 + off, idesc, 1u);
            tc::mma_bf16_w(d, bh0 + toff, wh0 + off, idesc, 1u);
          } else {
            const uint32_t d = tmem + (uint32_t)((buf * NMT + t) * N);
            tc::mma_bf16_w(d, wl0 + toff, bh0 + off, idesc, seg_first ? 0u : 1u);
            tc::mma_bf16_w(d, wh0 + toff, bl0 + off, idesc, 1u);
            tc::mma_bf16_w(d, wh0 + toff, bh0 + off, idesc, 1u);
          }
        }
        tc::mma_commit_w(&empty_bar[s]);
        if (++segc == seg || kb == nkb - 1) {
          tc::mma_commit_w(&acc_full[buf]);
          segc = 0;
          if (buf) ++use1; else ++use0;
          ++sgi;
          if (NACC == 2) buf ^= 1;
        }
        if (++s == NSTAGE) { s = 0; ph ^= 1u; }
      }
    }
    __syncwarp();
  } else if (warp == TC_PROD_WARP) {
    // ===================== bulk-copy producer of the pre-tiled W_hi/W_lo stage
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % NSTAGE;
        tc::mbar_wait(&empty_bar[s], ((kb / NSTAGE) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&full_bar[s], Cfg::W_STAGE_BYTES);
        tc::bulk_g2s(smem + s * Cfg::STAGE_BYTES, Wtiled + (int64_t)kb * (Cfg::W_STAGE_BYTES / 2), Cfg::W_STAGE_BYTES,
                     &full_bar[s]);
      }
    }
    __syncwarp();
  } else {
    // ===================== TMA producer of the jet windows
    if (lane == 0) {
      tc::tma_prefetch_desc(&tmX);
      for (int w = 0; w < nwin; ++w) {
        const int slot = w % TC_NWIN;
        if (w >= TC_NWIN) tc::mbar_wait(&win_empty[slot], (uint32_t)(((w / TC_NWIN) - 1) & 1));
        tc::mbar_arrive_expect_tx(&win_full[slot], Cfg::WIN_FLOATS * 4);
        tc::tma_load_3d(win + slot * Cfg::WIN_FLOATS, &tmX, w * TC_WIN, 0, (int)p0, &win_full[slot]);
      }
    }
    __syncwarp();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == TC_MMA_WARP) tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
}

}  // namespace

#include "tc_dgrad.cuh"
#include "tc_wgrad.cuh"

namespace {

// Pre-split the output-jet adjoint Ybar[P][C][O] of a tensor-core layer into the bf16 hi/lo operand
// stages both reverse kernels bulk-copy (every CTA of k_wgrad_tc and every
// M-tile of k_dgrad_tc would otherwise re-split the same values):
//   YW (k_wgrad_tc B operand, K = 8 points x channel pair):
//       [8-point block b][stage ss][hi|lo][chunk ch = channel 2ss+ch][O rows][8 points]
//   YD (k_dgrad_tc B operand, K = 16 outputs):
//       [point tile t (NP points)][K-block kb][hi|lo][chunk = 8 outputs][N rows = p*C + c][8]
// One block per 8 points; the block stages Ybar[8][C][O] in shared memory (coalesced float4 loads).
template <int C, int O>
__global__ void __launch_bounds__(256) k_split_ybar(const float* __restrict__ Ybar, int64_t P,
                                                    uint16_t* __restrict__ YW, uint16_t* __restrict__ YD) {
  constexpr int NP = tc_np(C), N = NP * C, NKB = O / TC_KB;
  constexpr int OS = O + 4;                       // padded row stride: the YD pass reads rows at stride OS
  extern __shared__ float ys[];                   // [8*C rows = q*C + c][OS]
  const int64_t b = blockIdx.x;
  const int64_t p0 = b * 8;
  const float4* src = reinterpret_cast<const float4*>(Ybar + p0 * (int64_t)(C * O));
  constexpr int NV = 8 * C * O / 4;               // float4s of the 8-point block
  constexpr int UNR = 8;                          // loads in flight per thread (the kernel is HBM-latency bound)
  for (int e0 = threadIdx.x; e0 < NV; e0 += UNR * 256) {
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int e = e0 + u * 256;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < NV && p0 + (e * 4) / (C * O) < P) v[u] = __ldg(src + e);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int e = e0 + u * 256;
      if (e < NV) reinterpret_cast<float4*>(ys + ((e * 4) / O) * OS)[((e * 4) % O) / 4] = v[u];
    }
  }
  __syncthreads();
  // wgrad operand: K chunks of 8 points are packed densely over (block, channel): chunk z = b*C + c
  // goes to stage z/2, half z%2 (no zero channel for odd C); the chunk after the last block of an odd
  // total is zero-filled (it pairs with that block's last channel in the final stage).  Lanes run
  // along o: 16-B stores are contiguous.
  const bool tail = (b == (int64_t)gridDim.x - 1) && ((gridDim.x * (int64_t)C) & 1);
  for (int t = threadIdx.x; t < (C + (tail ? 1 : 0)) * O; t += blockDim.x) {
    const int o = t % O, c = t / O;
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = (c < C) ? ys[(q * C + c) * OS + o] : 0.f;
    uint4 hi, lo;
    tc::split8_bf16(v, hi, lo);
    const int64_t z = b * C + c;
    const int ch = (int)(z & 1);
    uint16_t* dst = YW + (z >> 1) * (int64_t)(2 * 2 * O * 8);
    *reinterpret_cast<uint4*>(dst + (ch * O + o) * 8) = hi;
    *reinterpret_cast<uint4*>(dst + 2 * O * 8 + (ch * O + o) * 8) = lo;
  }
  // dgrad operand: lanes run along the 8*C rows (p*C + c) of this block, which are contiguous rows
  // of the tile's N -- 16-B stores are contiguous (the row-fastest order also keeps the float4 reads
  // of the padded smem rows conflict-free).
  const int64_t tile = p0 / NP;
  const int row0 = (int)(p0 - tile * NP) * C;
  for (int t = threadIdx.x; t < 8 * C * (O / 8); t += blockDim.x) {
    const int rw = t % (8 * C), og = t / (8 * C);
    const float4* sp = reinterpret_cast<const float4*>(ys + rw * OS + og * 8);
    const float4 a0 = sp[0], a1 = sp[1];
    float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    uint4 hi, lo;
    tc::split8_bf16(v, hi, lo);
    uint16_t* dst = YD + (tile * NKB + og / 2) * (int64_t)(2 * 2 * N * 8);
    *reinterpret_cast<uint4*>(dst + ((og & 1) * N + row0 + rw) * 8) = hi;
    *reinterpret_cast<uint4*>(dst + 2 * N * 8 + ((og & 1) * N + row0 + rw) * 8) = lo;
  }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
bool tc_layer_ok(const hrkan_net* net, int l) {
  if (net->engine == 1) return false;
  const int L = net->L;
  if (l <= 0 || l >= L - 1) return false;          // hidden layers only
  const int O = net->widths[l + 1], I = net->widths[l];
  if (O != 64 && O != 128 && O != 256) return false;
  if (net->engine == 0 && (int64_t)I * net->B < 256) return false;   // K too small to pay off
  if (net->B < 8) return false;                   // a K chunk spans at most 2 inputs; <= 17 inputs per M-tile
  if (I % 8 != 0) return false;                    // jet windows / boxes (TMA rows 16-B aligned)
  return true;
}

hrkan_status tc_refresh_weights(hrkan_net* net, cudaStream_t st) {
  if (net->tc_layers.empty()) net->tc_layers.assign(net->L, TcLayerState{});
  for (int l = 0; l < net->L; ++l) {
    if (!tc_layer_ok(net, l)) continue;
    const int O = net->widths[l + 1], I = net->widths[l];
    TcLayerState& ls = net->tc_layers[l];
    const int K = I * net->B;
    ls.nkb = (K + TC_KB - 1) / TC_KB;
    const int OP = (HRKAN_FWD_SWAP && O == 64) ? 64 : (O + 127) / 128 * 128;   // FwdCfg::OP (O = 64 runs swapped)
    const size_t n = (size_t)ls.nkb * 2 * OP * TC_KB;
    if (!ls.w_fwd) {
      if (cudaMalloc(&ls.w_fwd, n * sizeof(uint16_t)) != cudaSuccess) return fail(HRKAN_ENOMEM, "tc weight alloc");
    }
    const int64_t tot = (int64_t)ls.nkb * OP * TC_KB;
    HR_LAUNCH(HRKAN_K_OTHER, "k_tile_w_fwd",
              k_tile_w_fwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(net->params + net->w_off[l], ls.w_fwd, O, OP, K,
                                                                          ls.nkb));
    // W^T tiles for the dgrad kernel (contiguous 128-row M-tiles, or input-aligned for B < 11)
    const int RPT = dgr_rows_per_tile(net->B, net->D);
    ls.ntile_dgr = (int)((K + RPT - 1) / RPT);
    const size_t nd = (size_t)ls.ntile_dgr * (O / TC_KB) * 2 * 128 * TC_KB;
    if (!ls.w_dgr) {
      if (cudaMalloc(&ls.w_dgr, nd * sizeof(uint16_t)) != cudaSuccess) return fail(HRKAN_ENOMEM, "tc weight alloc");
    }
    const int64_t totd = (int64_t)ls.ntile_dgr * (O / TC_KB) * 128 * TC_KB;
    HR_LAUNCH(HRKAN_K_OTHER, "k_tile_w_dgr",
              k_tile_w_dgr<<<(unsigned)((totd + 255) / 256), 256, 0, st>>>(net->params + net->w_off[l], ls.w_dgr, O, I,
                                                                          net->B, RPT, ls.ntile_dgr));
  }
  return HRKAN_OK;
}

template <int NF, int NS, int M, int OO>
hrkan_status launch_fwd_tc(hrkan_net* net, int l, const float* X, float* Y, int64_t n, cudaStream_t st) {
  using Cfg = FwdCfg<NF, NS, M, OO>;
  auto kfn = k_fwd_tc<NF, NS, M, OO>;
  static uint64_t attr_dev = 0;                   // function attributes are per device (context)
  if (!((attr_dev >> (net->device & 63)) & 1)) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_dev |= 1ull << (net->device & 63);
  }
  const int I = net->widths[l];
  CUtensorMap tm;
  HR_TRY(make_tmap_f32_3d(&tm, X, (uint64_t)I, (uint64_t)Cfg::C, (uint64_t)n, TC_WIN, Cfg::CB, Cfg::NP));
  const TcLayerState& ls = net->tc_layers[l];
  const unsigned grid = (unsigned)((n + Cfg::NP - 1) / Cfg::NP);
  const int cls = HRKAN_K_FWD_HIDDEN;
  HR_LAUNCH(cls, "k_fwd_tc",
            kfn<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(tm, ls.w_fwd, net->params + net->b_off[l], Y, n, I, ls.nkb,
                                                           Cfg::NACC == 2 ? net->tc_seg : net->tc_seg_single, net->bc,
                                                           net->tc_dbg));
  return HRKAN_OK;
}

template <int NF, int NS, int M>
hrkan_status tc_forward_layer(hrkan_net* net, int l, const float* X, float* Y, int64_t n, cudaStream_t st, bool* done) {
  *done = false;
  constexpr int C = 1 + NF + NS;
  if constexpr (tc_np(C) == 0) {
    return HRKAN_OK;
  } else {
    if (!tc_layer_ok(net, l) || l >= (int)net->tc_layers.size() || !net->tc_layers[l].w_fwd) return HRKAN_OK;
    const int O = net->widths[l + 1];
    if (O == 64) HR_TRY(launch_fwd_tc<NF, NS, M, 64>(net, l, X, Y, n, st));
    else if (O == 128) HR_TRY(launch_fwd_tc<NF, NS, M, 128>(net, l, X, Y, n, st));
    else HR_TRY(launch_fwd_tc<NF, NS, M, 256>(net, l, X, Y, n, st));
    *done = true;
    return HRKAN_OK;
  }
}

// Sizes the pre-split operand buffers (net->tc_yw, net->tc_yd) of a C-channel layer with O outputs, n points.
template <int C>
hrkan_status tc_split_buffers(hrkan_net* net, int O, int64_t n) {
  const int64_t nb8 = (n + 7) / 8;
  const int64_t ntile = (n + tc_np(C) - 1) / tc_np(C);
  const size_t yw = (size_t)((nb8 * C + 1) / 2) * 2 * 2 * O * 8;        // densely packed K chunks
  const size_t yd = (size_t)ntile * (O / TC_KB) * 2 * 2 * tc_np(C) * C * 8;
  HR_CUDA(net->tc_yw.ensure(yw * sizeof(uint16_t)));
  HR_CUDA(net->tc_yd.ensure(yd * sizeof(uint16_t)));
  return HRKAN_OK;
}

// Both reverse kernels of hidden layer l run on the tensor cores for n points (so its Ybar is consumed only
// as the pre-split operands + bias partials, and an upstream kernel may emit those instead of fp32 Ybar).
bool tc_reverse_ok(const hrkan_net* net, int l, int64_t n) {
  return tc_layer_ok(net, l) && n >= 8 && l < (int)net->tc_layers.size() && net->tc_layers[l].w_dgr &&
         dgr_tile_ok(net->B, net->D);
}

// Pre-split Ybar of tensor-core layer l for both reverse kernels (net->tc_yw, net->tc_yd).
template <int NF, int NS, int M>
hrkan_status tc_split_ybar(hrkan_net* net, int l, const float* Ybar, int64_t n, cudaStream_t st) {
  constexpr int C = 1 + NF + NS;
  if constexpr (tc_np(C) == 0) {
    return HRKAN_OK;
  } else {
    if (!tc_layer_ok(net, l) || n <= 0) return HRKAN_OK;
    const int O = net->widths[l + 1];
    const int64_t nb8 = (n + 7) / 8;
    HR_TRY(tc_split_buffers<C>(net, O, n));
    auto launch = [&](auto OC) -> hrkan_status {
      constexpr int OO = decltype(OC)::value;
      auto kfn = k_split_ybar<C, OO>;
      constexpr int smem = 8 * C * (OO + 4) * 4;
      HR_CUDA(smem_optin(kfn, smem));
      HR_LAUNCH(HRKAN_K_OTHER, "k_split_ybar",
                kfn<<<(unsigned)nb8, 256, smem, st>>>(Ybar, n, (uint16_t*)net->tc_yw.p, (uint16_t*)net->tc_yd.p));
      return HRKAN_OK;
    };
    if (O == 64) return launch(std::integral_constant<int, 64>{});
    if (O == 128) return launch(std::integral_constant<int, 128>{});
    return launch(std::integral_constant<int, 256>{});
  }
}

template <int NF, int NS, int M, int OO>
hrkan_status launch_wgrad_tc(hrkan_net* net, int l, const float* X, const float* Ybar, float* dW, float* db,
                             int64_t n, cudaStream_t st, const float* bias_part, int bias_nz) {
  using Cfg = WgrCfg<NF, NS, M, OO>;
  constexpr int C = Cfg::C, O = Cfg::O;
  auto kfn = k_wgrad_tc<NF, NS, M, OO>;
  static uint64_t attr_dev = 0;                   // function attributes are per device (context)
  if (!((attr_dev >> (net->device & 63)) & 1)) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_dev |= 1ull << (net->device & 63);
  }
  const int I = net->widths[l];
  const int64_t K = (int64_t)I * net->B;
  const int nmt = (int)((K + 127) / 128);
  // slabs per M-tile: 3-6 waves of one CTA per SM, chosen to minimise the idle tail of the last wave
  int nslab = 1;
  {
    double best = -1.0;
    const int lo = std::max(1, (3 * net->num_sms) / nmt), hi = std::max(lo, (6 * net->num_sms) / nmt);
    for (int c = lo; c <= hi; ++c) {
      const int64_t units = (int64_t)c * nmt;
      const double eff = (double)units / (double)(((units + net->num_sms - 1) / net->num_sms) * net->num_sms);
      if (eff > best + 1e-9) { best = eff; nslab = c; }
    }
  }
  nslab = (int)std::min<int64_t>(nslab, std::max<int64_t>(1, n / 64));
  int64_t slab = (n + nslab - 1) / nslab;
  slab = (slab + WGR_JP - 1) / WGR_JP * WGR_JP;       // jet boxes of 32 points never straddle slabs
  nslab = (int)((n + slab - 1) / slab);
  const size_t part_bytes = sizeof(float) * ((size_t)nslab * O * K + (size_t)1024 * O);
  HR_CUDA(net->tc_ws.ensure(part_bytes));
  float* part = net->tc_ws.f();
  float* part_b = part + (size_t)nslab * O * K;
  CUtensorMap tmX;
  HR_TRY(make_tmap_f32_3d(&tmX, X, (uint64_t)I, (uint64_t)C, (uint64_t)n, WGR_IW, C, WGR_JP));
  {
    HR_LAUNCH(HRKAN_K_WGRAD_HIDDEN, "k_wgrad_tc",
              kfn<<<(unsigned)(nslab * nmt), WGR_THREADS, Cfg::SMEM_BYTES, st>>>(
                  tmX, (const uint16_t*)net->tc_yw.p, part, n, I, nmt, slab, net->tc_wseg, net->bc, net->tc_dbg));
  }
  HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_slabs",
            k_reduce_slabs<<<(unsigned)((O * K + 255) / 256), 256, 0, st>>>(part, nslab, (int64_t)O * K, dW));
  if (bias_part) {                                   // emitted by the fused output layer
    HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_bias", k_reduce_bias<<<(O + 31) / 32, 256, 0, st>>>(bias_part, bias_nz, O, db));
    return HRKAN_OK;
  }
  const int nz = (int)std::min<int64_t>(1024, std::max<int64_t>(1, n / 256));
  HR_LAUNCH(HRKAN_K_REDUCE, "k_bias_part",
            k_bias_part<<<dim3((O + 127) / 128, nz), 128, 0, st>>>(Ybar, C, O, n, part_b));
  HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_bias", k_reduce_bias<<<(O + 31) / 32, 256, 0, st>>>(part_b, nz, O, db));
  return HRKAN_OK;
}

template <int NF, int NS, int M>
hrkan_status tc_wgrad_layer(hrkan_net* net, int l, const float* X, const float* Ybar, float* dW, float* db, int64_t n,
                            cudaStream_t st, bool* done, const float* bias_part = nullptr, int bias_nz = 0) {
  *done = false;
  if (!tc_layer_ok(net, l) || n < 8) return HRKAN_OK;
  const int O = net->widths[l + 1];
  if (O == 64) HR_TRY(launch_wgrad_tc<NF, NS, M, 64>(net, l, X, Ybar, dW, db, n, st, bias_part, bias_nz));
  else if (O == 128) HR_TRY(launch_wgrad_tc<NF, NS, M, 128>(net, l, X, Ybar, dW, db, n, st, bias_part, bias_nz));
  else HR_TRY(launch_wgrad_tc<NF, NS, M, 256>(net, l, X, Ybar, dW, db, n, st, bias_part, bias_nz));
  *done = true;
  return HRKAN_OK;
}

template <int NF, int NS, int M, int OO>
hrkan_status launch_dgrad_tc(hrkan_net* net, int l, const float* X, const float* Ybar, float* Xbar, int64_t n,
                             cudaStream_t st) {
  using Cfg = DgrCfg<NF, NS, M, OO>;
  auto kfn = k_dgrad_tc<NF, NS, M, OO>;
  static uint64_t attr_dev = 0;                   // function attributes are per device (context)
  if (!((attr_dev >> (net->device & 63)) & 1)) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_dev |= 1ull << (net->device & 63);
  }
  const TcLayerState& ls = net->tc_layers[l];
  const int I = net->widths[l];
  CUtensorMap tmX;
  HR_TRY(make_tmap_f32_3d(&tmX, X, (uint64_t)I, (uint64_t)Cfg::C, (uint64_t)n, DGR_IPTB, Cfg::C, Cfg::NP));
  const int64_t ntiles = (n + Cfg::NP - 1) / Cfg::NP;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, net->num_sms));   // persistent
  HR_LAUNCH(HRKAN_K_DGRAD_HIDDEN, "k_dgrad_tc",
            kfn<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, st>>>(tmX, (const uint16_t*)net->tc_yd.p, ls.w_dgr, Xbar, n, I,
                                                            dgr_rows_per_tile(net->B, net->D), ls.ntile_dgr, net->bc,
                                                            net->tc_dbg));
  return HRKAN_OK;
}

template <int NF, int NS, int M>
hrkan_status tc_dgrad_layer(hrkan_net* net, int l, const float* X, const float* Ybar, float* Xbar, int64_t n,
                            cudaStream_t st, bool* done) {
  *done = false;
  constexpr int C = 1 + NF + NS;
  if constexpr (tc_np(C) == 0) {
    return HRKAN_OK;
  } else {
    if (!tc_layer_ok(net, l) || l >= (int)net->tc_layers.size() || !net->tc_layers[l].w_dgr) return HRKAN_OK;
    if (!dgr_tile_ok(net->B, net->D)) return HRKAN_OK;   // an M-tile's inputs would not fit the jet box
    const int O = net->widths[l + 1];
    if (O == 64) HR_TRY(launch_dgrad_tc<NF, NS, M, 64>(net, l, X, Ybar, Xbar, n, st));
    else if (O == 128) HR_TRY(launch_dgrad_tc<NF, NS, M, 128>(net, l, X, Ybar, Xbar, n, st));
    else HR_TRY(launch_dgrad_tc<NF, NS, M, 256>(net, l, X, Ybar, Xbar, n, st));
    *done = true;
    return HRKAN_OK;
  }
}

void tc_free(hrkan_net* net) {
  for (auto& ls : net->tc_layers) {
    if (ls.w_fwd) cudaFree(ls.w_fwd);
    if (ls.w_dgr) cudaFree(ls.w_dgr);
    ls.w_fwd = ls.w_dgr = nullptr;
  }
}

}  // namespace
