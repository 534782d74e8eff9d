// tc_kernels.cuh -- tcgen05 / TMEM tensor-core engine for the wide hidden layers (sm_100a).
//
// The hidden KAN layer is the dense contraction of PAPER.md:45/:87 ("KAN layer as a matrix
// operation") applied to every jet channel:
//     Y[(p,c), o] = sum_{K=(i,n)} A^c[p, K] W[o, K]      (+ b_o on the value channel c = 0)
// with A^c generated on the fly from the saved input jet.  It runs as 3xTF32
// on the 5th-generation tensor cores: W and A are split into tf32 hi/lo parts and
//     D += W_hi A_hi + W_hi A_lo + W_lo A_hi
// accumulate in fp32 TMEM, which meets the north-star tolerance.
//
// Forward kernel k_fwd_tc (orientation "W rows x (point,channel) columns"):
//   MMA M = output neurons o (128-row tiles; O = 128 or 256 -> 1 or 2 tiles, both share the B tile),
//   MMA N = NP points x C channels of one point tile (channel-major columns n = c*NP + p),
//   MMA K = I*B (dense over all bases, zero-padded to a multiple of KB).
//   smem stage = { W_hi, W_lo tiles [KB/4 chunks][O rows][4] via one 1-D bulk copy of a
//                  pre-tiled global copy;  A_hi, A_lo tiles [KB/4][N][4] written by 4 generator
//                  warps from the jet }, NSTAGE-deep mbarrier ring.
//   warps 0-3: generators, then epilogue (TMEM -> registers -> +bias -> Y[p][c][o], coalesced);
//   warp 4: TMEM allocator + single-thread MMA issuer; warp 5: bulk-copy producer.
#pragma once
#include "tc_ptx.cuh"

namespace {

using namespace hrkan;

constexpr int TC_KB = 16;          // K per pipeline stage (two tf32 MMA K-steps of 8)
constexpr int TC_NSTAGE = 3;
constexpr int TC_GEN_THREADS = 128;   // one generator group (4 warps); the group handles every other K-block
constexpr int TC_NGEN = 2;            // generator groups (group 0 also drains the accumulators)
constexpr int TC_THREADS = 32 * (4 * TC_NGEN + 2);   // + MMA warp + producer warp
constexpr int TC_MMA_WARP = 4 * TC_NGEN, TC_PROD_WARP = 4 * TC_NGEN + 1;

// Points per tile so that N = NP*C is a multiple of 16 and <= 256.
__host__ __device__ constexpr int tc_np(int C) {
  return C == 7 ? 32 : C == 5 ? 48 : C == 4 ? 64 : C == 3 ? 80 : C == 1 ? 256 : 0;
}

__host__ __device__ constexpr uint32_t tc_tmem_cols(uint32_t c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int NF, int NS, int M, int NMT>
struct FwdCfg {
  static constexpr int C = 1 + NF + NS;
  static constexpr int NP = tc_np(C);
  static constexpr int N = NP * C;
  static constexpr int O = 128 * NMT;
  static constexpr int W_STAGE_FLOATS = 2 * O * TC_KB;     // hi + lo
  static constexpr int A_STAGE_FLOATS = 2 * N * TC_KB;
  static constexpr int STAGE_BYTES = 4 * (W_STAGE_FLOATS + A_STAGE_FLOATS);
  static constexpr int SMEM_BYTES = TC_NSTAGE * STAGE_BYTES + 1024;
  static constexpr int NACC = (2 * NMT * N <= 512) ? 2 : 1;   // double-buffered accumulators if they fit
  static constexpr uint32_t TMEM_COLS = tc_tmem_cols(NACC * NMT * N);
  static_assert(N % 16 == 0 && N <= 256, "bad N");
  static_assert(NMT * N <= 512, "accumulators exceed TMEM");
};

// Pre-tiled, pre-split weights for k_fwd_tc: for K-block kb: [hi | lo] each [KB/4][O][4].
__global__ void k_tile_w_fwd(const float* __restrict__ W, float* __restrict__ Wt, int O, int K, int nkb) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per_kb = (int64_t)O * TC_KB;
  if (t >= per_kb * nkb) return;
  const int kb = (int)(t / per_kb);
  const int r = (int)(t - (int64_t)kb * per_kb);     // r = (j*O + o)*4 + e
  const int e = r & 3, o = (r >> 2) % O, j = (r >> 2) / O;
  const int k = kb * TC_KB + 4 * j + e;
  const float w = (k < K) ? W[(int64_t)o * K + k] : 0.f;
  float hi, lo;
  tc::split_tf32(w, hi, lo);
  float* dst = Wt + (int64_t)kb * 2 * per_kb;
  dst[r] = hi;
  dst[per_kb + r] = lo;
}

template <int NF, int NS, int M, int NMT>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_fwd_tc(const float* __restrict__ X, const float* __restrict__ Wtiled, const float* __restrict__ bias,
             float* __restrict__ Y, int64_t P, int I, int nkb, int seg, BasisCfg bc) {
  using Cfg = FwdCfg<NF, NS, M, NMT>;
  constexpr int C = Cfg::C, NP = Cfg::NP, N = Cfg::N, O = Cfg::O, NACC = Cfg::NACC;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* smem = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[TC_NSTAGE], empty_bar[TC_NSTAGE], acc_full[NACC], acc_empty[NACC];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = (int64_t)blockIdx.x * NP;
  const int K = I * bc.B;
  const int nseg = (nkb + seg - 1) / seg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_NSTAGE; ++s) {
      tc::mbar_init(&full_bar[s], TC_GEN_THREADS + 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      tc::mbar_init(&acc_full[a], 1);
      tc::mbar_init(&acc_empty[a], TC_GEN_THREADS * TC_NGEN);
    }
    tc::fence_mbar_init();
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
#pragma unroll 1
      for (int t = 0; t < NMT; ++t) {
        const int o = t * 128 + qw * 32 + lane;
        const float b = (sg == 0) ? __ldg(bias + o) : 0.f;
        const uint32_t tbase = tmem + ((uint32_t)(qw * 32) << 16) + (uint32_t)((buf * NMT + t) * N);
        // 16-column chunks are shared round-robin by the generator groups (same lane quadrant)
#pragma unroll 1
        for (int c0 = 16 * grp; c0 < N; c0 += 16 * TC_NGEN) {
          float v[16];
          tc::tmem_ld16(tbase + c0, v);
          float* yp[16];
          bool ok[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int col = c0 + q;
            const int c = col / NP, pl = col - c * NP;
            const int64_t p = p0 + pl;
            ok[q] = p < P;
            yp[q] = Y + (p * C + c) * (int64_t)O + o;
            if (sg == 0 && c == 0) v[q] += b;
          }
          if (sg > 0) {
            float old[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) old[q] = ok[q] ? *yp[q] : 0.f;   // 16 loads in flight
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += old[q];
          }
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (ok[q]) *yp[q] = v[q];
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&acc_empty[buf]);
    };
    // ===================== generators: A^c[p, k] for the stage's KB columns.
    // Each thread owns TPT tasks (point pl, 4-wide K chunk j) per block; the jets of the next
    // block are prefetched into registers while the current block is generated.
    constexpr int NTASK = NP * (TC_KB / 4);
    constexpr int TPT = (NTASK + TC_GEN_THREADS - 1) / TC_GEN_THREADS;
    float jx[2][TPT][2], jdx[2][TPT][2][NF > 0 ? NF : 1], jddx[2][TPT][2][NS > 0 ? NS : 1];
    auto prefetch = [&](int kb, auto SLOT) {
      constexpr int slot = decltype(SLOT)::value;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int task = gtid + u * TC_GEN_THREADS;
        const int pl = task % NP, j = task / NP;
        const int64_t p = p0 + pl;
        const int k0 = kb * TC_KB + 4 * j;
        const int i0 = k0 / bc.B;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = i0 + h;
          jx[slot][u][h] = 0.f;
#pragma unroll
          for (int a = 0; a < NF; ++a) jdx[slot][u][h][a] = 0.f;
#pragma unroll
          for (int a = 0; a < NS; ++a) jddx[slot][u][h][a] = 0.f;
          if (task < NTASK && p < P && i < I && kb < nkb) {
            const float* base = X + p * (int64_t)(C * I) + i;
            jx[slot][u][h] = __ldg(base);
#pragma unroll
            for (int a = 0; a < NF; ++a) jdx[slot][u][h][a] = __ldg(base + (1 + a) * I);
#pragma unroll
            for (int a = 0; a < NS; ++a) jddx[slot][u][h][a] = __ldg(base + (1 + NF + a) * I);
          }
        }
      }
    };
    int next_drain = 0;
    // one K-block: prefetch the group's next block into the other register slot, then generate
    auto step = [&](int kb, auto SLOT) {
      constexpr int slot = decltype(SLOT)::value;
      while (next_drain < nseg - 1 && kb >= (next_drain + 1) * seg + TC_NSTAGE) drain(next_drain++);
      prefetch(kb + TC_NGEN, std::integral_constant<int, slot ^ 1>{});
      const int s = kb % TC_NSTAGE;
      const uint32_t ph = (kb / TC_NSTAGE) & 1;
      tc::mbar_wait(&empty_bar[s], ph ^ 1);
      float* a_hi = smem + s * (Cfg::W_STAGE_FLOATS + Cfg::A_STAGE_FLOATS) + Cfg::W_STAGE_FLOATS;
      float* a_lo = a_hi + N * TC_KB;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int task = gtid + u * TC_GEN_THREADS;
        if (task >= NTASK) break;
        const int pl = task % NP, j = task / NP;
        const int k0 = kb * TC_KB + 4 * j;
        const int i0 = k0 / bc.B;
        int n = k0 - i0 * bc.B;
        float va[C][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool h = n >= bc.B;                   // chunk crosses into input i0+1
          const int nn = h ? n - bc.B : n;
          const float x = h ? jx[slot][u][1] : jx[slot][u][0];
          float v0, v1, v2, v3;
          hr_eval<M, (NS > 0 ? 2 : 1)>(basis_q(x, nn, bc), bc.sc, v0, v1, v2, v3);
          if (k0 + e >= K) v0 = v1 = v2 = 0.f;
          va[0][e] = v0;
#pragma unroll
          for (int a = 0; a < NF; ++a) va[1 + a][e] = v1 * (h ? jdx[slot][u][1][a] : jdx[slot][u][0][a]);
#pragma unroll
          for (int a = 0; a < NS; ++a) {
            const float d1 = h ? jdx[slot][u][1][a] : jdx[slot][u][0][a];
            const float d2 = h ? jddx[slot][u][1][a] : jddx[slot][u][0][a];
            va[1 + NF + a][e] = fmaf(v2 * d1, d1, v1 * d2);
          }
          ++n;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          float4 hh, ll;
          tc::split_tf32(va[c][0], hh.x, ll.x);
          tc::split_tf32(va[c][1], hh.y, ll.y);
          tc::split_tf32(va[c][2], hh.z, ll.z);
          tc::split_tf32(va[c][3], hh.w, ll.w);
          const int row = c * NP + pl;                  // channel-major columns of the MMA N
          *reinterpret_cast<float4*>(a_hi + (j * N + row) * 4) = hh;
          *reinterpret_cast<float4*>(a_lo + (j * N + row) * 4) = ll;
        }
      }
      tc::fence_proxy_async_smem();
      tc::mbar_arrive(&full_bar[s]);
    };
    prefetch(grp, std::integral_constant<int, 0>{});
    for (int kb = grp; kb < nkb; kb += 2 * TC_NGEN) {
      step(kb, std::integral_constant<int, 0>{});
      if (kb + TC_NGEN < nkb) step(kb + TC_NGEN, std::integral_constant<int, 1>{});
    }
    while (next_drain < nseg) drain(next_drain++);
  } else if (warp == TC_MMA_WARP) {
    // ===================== MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, N);
      for (int kb = 0; kb < nkb; ++kb) {
        const int sg = kb / seg, buf = sg % NACC;
        const bool seg_first = (kb % seg) == 0;
        if (seg_first && sg >= NACC) {
          tc::mbar_wait(&acc_empty[buf], (uint32_t)((sg / NACC - 1) & 1));
          tc::tc_fence_after();
        }
        const int s = kb % TC_NSTAGE;
        const uint32_t ph = (kb / TC_NSTAGE) & 1;
        tc::mbar_wait(&full_bar[s], ph);
        tc::tc_fence_after();
        const float* w_hi = smem + s * (Cfg::W_STAGE_FLOATS + Cfg::A_STAGE_FLOATS);
        const float* w_lo = w_hi + O * TC_KB;
        const float* a_hi = w_hi + Cfg::W_STAGE_FLOATS;
        const float* a_lo = a_hi + N * TC_KB;
#pragma unroll
        for (int ks = 0; ks < TC_KB / 8; ++ks) {
          // K-step ks covers chunks 2ks, 2ks+1: LBO = chunk stride = rows*16 B, SBO = 8 rows = 128 B
          const uint32_t aoff = (uint32_t)(2 * ks * N * 16);
          const uint64_t bh = tc::smem_desc(tc::smem_u32(a_hi) + aoff, N * 16, 128);
          const uint64_t bl = tc::smem_desc(tc::smem_u32(a_lo) + aoff, N * 16, 128);
#pragma unroll
          for (int t = 0; t < NMT; ++t) {
            const uint32_t woff = (uint32_t)(2 * ks * O * 16 + t * 128 * 16);
            const uint64_t wh = tc::smem_desc(tc::smem_u32(w_hi) + woff, O * 16, 128);
            const uint64_t wl = tc::smem_desc(tc::smem_u32(w_lo) + woff, O * 16, 128);
            const uint32_t d = tmem + (uint32_t)((buf * NMT + t) * N);
            const uint32_t acc0 = (seg_first && ks == 0) ? 0u : 1u;
            tc::mma_tf32(d, wl, bh, idesc, acc0);
            tc::mma_tf32(d, wh, bl, idesc, 1u);
            tc::mma_tf32(d, wh, bh, idesc, 1u);
          }
        }
        tc::mma_commit(&empty_bar[s]);
        if ((kb % seg) == seg - 1 || kb == nkb - 1) tc::mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ===================== bulk-copy producer of the pre-tiled W_hi/W_lo stage
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % TC_NSTAGE;
        const uint32_t ph = (kb / TC_NSTAGE) & 1;
        tc::mbar_wait(&empty_bar[s], ph ^ 1);
        float* w_dst = smem + s * (Cfg::W_STAGE_FLOATS + Cfg::A_STAGE_FLOATS);
        tc::mbar_arrive_expect_tx(&full_bar[s], Cfg::W_STAGE_FLOATS * 4);
        tc::bulk_g2s(w_dst, Wtiled + (int64_t)kb * Cfg::W_STAGE_FLOATS, Cfg::W_STAGE_FLOATS * 4, &full_bar[s]);
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

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
bool tc_layer_ok(const hrkan_net* net, int l) {
  if (net->engine == 1) return false;
  const int L = net->L;
  if (l <= 0 || l >= L - 1) return false;          // hidden layers only
  const int O = net->widths[l + 1], I = net->widths[l];
  if (O != 128 && O != 256) return false;
  if (net->engine == 0 && (int64_t)I * net->B < 256) return false;   // K too small to pay off
  if (net->B < 4) return false;                   // a 4-wide K chunk spans at most 2 inputs
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
    const size_t n = (size_t)ls.nkb * 2 * O * TC_KB;
    if (!ls.w_fwd) {
      if (cudaMalloc(&ls.w_fwd, n * sizeof(float)) != cudaSuccess) return fail(HRKAN_ENOMEM, "tc weight alloc");
    }
    const int64_t tot = (int64_t)ls.nkb * O * TC_KB;
    HR_LAUNCH(HRKAN_K_OTHER, "k_tile_w_fwd",
              k_tile_w_fwd<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(net->params + net->w_off[l], ls.w_fwd, O, K, ls.nkb));
    // W^T tiles for the dgrad kernel (input-aligned M-tiles)
    const int IPT = 128 / net->B;
    ls.ntile_dgr = (I + IPT - 1) / IPT;
    const size_t nd = (size_t)ls.ntile_dgr * (O / TC_KB) * 2 * 128 * TC_KB;
    if (!ls.w_dgr) {
      if (cudaMalloc(&ls.w_dgr, nd * sizeof(float)) != cudaSuccess) return fail(HRKAN_ENOMEM, "tc weight alloc");
    }
    const int64_t totd = (int64_t)ls.ntile_dgr * (O / TC_KB) * 128 * TC_KB;
    HR_LAUNCH(HRKAN_K_OTHER, "k_tile_w_dgr",
              k_tile_w_dgr<<<(unsigned)((totd + 255) / 256), 256, 0, st>>>(net->params + net->w_off[l], ls.w_dgr, O, I,
                                                                          net->B, IPT, ls.ntile_dgr));
  }
  return HRKAN_OK;
}

template <int NF, int NS, int M, int NMT>
hrkan_status launch_fwd_tc(hrkan_net* net, int l, const float* X, float* Y, int64_t n, cudaStream_t st) {
  using Cfg = FwdCfg<NF, NS, M, NMT>;
  auto kfn = k_fwd_tc<NF, NS, M, NMT>;
  static bool attr_set = false;
  if (!attr_set) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_set = true;
  }
  const TcLayerState& ls = net->tc_layers[l];
  const unsigned grid = (unsigned)((n + Cfg::NP - 1) / Cfg::NP);
  const int cls = HRKAN_K_FWD_HIDDEN;
  HR_LAUNCH(cls, "k_fwd_tc",
            kfn<<<grid, TC_THREADS, Cfg::SMEM_BYTES, st>>>(X, ls.w_fwd, net->params + net->b_off[l], Y, n,
                                                           net->widths[l], ls.nkb, Cfg::NACC == 2 ? net->tc_seg : 2 * net->tc_seg, net->bc));
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
    if (O == 128) HR_TRY(launch_fwd_tc<NF, NS, M, 1>(net, l, X, Y, n, st));
    else HR_TRY(launch_fwd_tc<NF, NS, M, 2>(net, l, X, Y, n, st));
    *done = true;
    return HRKAN_OK;
  }
}

template <int NF, int NS, int M, int OT>
hrkan_status launch_wgrad_tc(hrkan_net* net, int l, const float* X, const float* Ybar, float* dW, float* db,
                             int64_t n, cudaStream_t st) {
  using Cfg = WgrCfg<NF, NS, M, OT>;
  constexpr int C = Cfg::C, O = Cfg::O;
  auto kfn = k_wgrad_tc<NF, NS, M, OT>;
  static bool attr_set = false;
  if (!attr_set) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_set = true;
  }
  const int I = net->widths[l];
  const int64_t K = (int64_t)I * net->B;
  const int nmt = (int)((K + 127) / 128);
  int nslab = (int)std::max<int64_t>(1, (4 * net->num_sms + nmt / 2) / nmt);
  nslab = (int)std::min<int64_t>(nslab, std::max<int64_t>(1, n / 64));
  int64_t slab = (n + nslab - 1) / nslab;
  slab = (slab + 7) / 8 * 8;
  nslab = (int)((n + slab - 1) / slab);
  const size_t part_bytes = sizeof(float) * ((size_t)nslab * O * K + (size_t)64 * O);
  HR_CUDA(net->tc_ws.ensure(part_bytes));
  float* part = net->tc_ws.f();
  float* part_b = part + (size_t)nslab * O * K;
  HR_LAUNCH(HRKAN_K_WGRAD_HIDDEN, "k_wgrad_tc",
            kfn<<<(unsigned)(nslab * nmt), WGR_THREADS, Cfg::SMEM_BYTES, st>>>(X, Ybar, part, n, I, nmt, slab,
                                                                               net->tc_wseg, net->bc));
  HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_slabs",
            k_reduce_slabs<<<(unsigned)((O * K + 255) / 256), 256, 0, st>>>(part, nslab, (int64_t)O * K, dW));
  const int nz = (int)std::min<int64_t>(64, std::max<int64_t>(1, n / 256));
  HR_LAUNCH(HRKAN_K_REDUCE, "k_bias_part",
            k_bias_part<<<dim3((O + 127) / 128, nz), 128, 0, st>>>(Ybar, C, O, n, part_b));
  HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_bias", k_reduce_bias<<<(O + 127) / 128, 128, 0, st>>>(part_b, nz, O, db));
  return HRKAN_OK;
}

template <int NF, int NS, int M>
hrkan_status tc_wgrad_layer(hrkan_net* net, int l, const float* X, const float* Ybar, float* dW, float* db, int64_t n,
                            cudaStream_t st, bool* done) {
  *done = false;
  if (!tc_layer_ok(net, l) || n < 8) return HRKAN_OK;
  const int O = net->widths[l + 1];
  if (O == 128) HR_TRY(launch_wgrad_tc<NF, NS, M, 1>(net, l, X, Ybar, dW, db, n, st));
  else HR_TRY(launch_wgrad_tc<NF, NS, M, 2>(net, l, X, Ybar, dW, db, n, st));
  *done = true;
  return HRKAN_OK;
}

template <int NF, int NS, int M, int OT>
hrkan_status launch_dgrad_tc(hrkan_net* net, int l, const float* X, const float* Ybar, float* Xbar, int64_t n,
                             cudaStream_t st) {
  using Cfg = DgrCfg<NF, NS, M, OT>;
  auto kfn = k_dgrad_tc<NF, NS, M, OT>;
  static bool attr_set = false;
  if (!attr_set) {
    HR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_set = true;
  }
  const TcLayerState& ls = net->tc_layers[l];
  const unsigned grid = (unsigned)((n + Cfg::NP - 1) / Cfg::NP);
  HR_LAUNCH(HRKAN_K_DGRAD_HIDDEN, "k_dgrad_tc",
            kfn<<<grid, DGR_THREADS, Cfg::SMEM_BYTES, st>>>(X, Ybar, ls.w_dgr, Xbar, n, net->widths[l], 128 / net->B,
                                                            ls.ntile_dgr, net->bc));
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
    const int O = net->widths[l + 1];
    if (O == 128) HR_TRY(launch_dgrad_tc<NF, NS, M, 1>(net, l, X, Ybar, Xbar, n, st));
    else HR_TRY(launch_dgrad_tc<NF, NS, M, 2>(net, l, X, Ybar, Xbar, n, st));
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
