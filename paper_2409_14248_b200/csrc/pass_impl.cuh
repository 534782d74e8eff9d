// pass_impl.cuh -- the chunked scheduler of one PINN loss+gradient (or forward-jet) pass, included by
// pass_m<M>.cu with HRKAN_M set: forward through the hidden layers (SIMT or tcgen05), the fused
// output-layer/loss kernel, then the reverse through the hidden layers (SURVEY §3 call stack).
#pragma once
#include "hrkan_internal.cuh"
#include "simt_kernels.cuh"
#include "tc_kernels.cuh"
#include "last_kernels.cuh"
#include "first_kernels.cuh"
#include "tiny_kernels.cuh"
#include "jet_kernels.cuh"

namespace {

// want_split: the preceding hidden layer runs both reverse kernels on the tensor cores, so the output layer may
// emit their pre-split bf16 operands and bias partials directly (k_last_v3<..., SPLIT>); *split_nb is then set
// to the number of bias-partial rows in net->tc_bias_part (0 when the fp32 adjoint was written instead).
template <int NF, int NS, int M, int MODE, bool FIRST>
hrkan_status launch_last(hrkan_net* net, const float* in, int64_t n, const PassArgs& a, int64_t c0, float* xbar,
                         cudaStream_t st, bool want_split = false, int* split_nb = nullptr) {
  if (split_nb) *split_nb = 0;
  const int l = net->L - 1;
  const int I = net->widths[l];
  const int IB = I * net->B;
  constexpr int C = 1 + NF + NS;
  if constexpr (!FIRST && MODE != LAST_JET && M >= 4) {
    if (I % 32 == 0 && I <= 256 && net->bc.k + 1 <= LV3_KT) {
      // input-parallel, bulk-copied jet batches, cached basis values (k_last_v3)
      constexpr bool CAN_SPLIT = tc_np(C) > 0;
      const bool split = CAN_SPLIT && want_split && split_nb;
      auto kv = split ? k_last_v3<NF, NS, M, MODE, CAN_SPLIT> : k_last_v3<NF, NS, M, MODE, false>;
      const int nw = I / 32, BP = lv3_bp(net->B);
      const size_t smem = sizeof(float) * ((size_t)2 * LV3_PB * C * (I + 4) + 2 * (size_t)I * BP + (size_t)LV3_PB * nw * C + LV3_PB * C);
      HR_CUDA(smem_optin(kv, smem));
      int per_sm = 0;
      HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kv, I, smem));
      per_sm = std::max(1, per_sm);
      const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * net->num_sms, (n + LV3_PB - 1) / LV3_PB));
      HR_CUDA(net->last_part.ensure(sizeof(float) * (size_t)nb * (IB + 4)));
      const hrkan_pde* pde = a.pde;
      const float* pts = a.pts + c0 * net->D;
      const float* f = a.forcing ? a.forcing + c0 : nullptr;
      const float* g = a.g ? a.g + c0 : nullptr;
      uint16_t *yw = nullptr, *yd = nullptr;
      float* pbias = nullptr;
      if (split) {
        if constexpr (CAN_SPLIT) HR_TRY(tc_split_buffers<C>(net, I, n));
        HR_CUDA(net->tc_bias_part.ensure(sizeof(float) * (size_t)nb * I));
        yw = (uint16_t*)net->tc_yw.p;
        yd = (uint16_t*)net->tc_yd.p;
        pbias = net->tc_bias_part.f();
        *split_nb = nb;
      }
      HR_LAUNCH(HRKAN_K_FWD_LAST, split ? "k_last_v3 (split)" : "k_last_v3",
                kv<<<nb, I, smem, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], n, I, net->bc, pts, f,
                                        g, pde->alpha, pde->adv, pde->visc, a.inv_n, xbar, net->last_part.f(), yw, yd, pbias));
      const float scale = (MODE == LAST_BOUNDARY) ? a.inv_n : pde->alpha * a.inv_n;
      HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_last",
                k_reduce_last<<<(IB + 3 + RL_COLS - 1) / RL_COLS, RL_COLS * RL_CHAINS, 0, st>>>(net->last_part.f(), nb, IB, a.grad + net->w_off[l],
                                                                     a.grad + net->b_off[l], scale, a.out_loss, a.out_flag));
      return HRKAN_OK;
    }
  }
  if (!FIRST && I % 32 == 0 && I <= 256) {
    // input-parallel variant: I/32 warps per block, block-shared dW accumulator
    auto kv = k_last_v2<NF, NS, M, MODE>;
    const int nw = I / 32;
    const size_t fixed = sizeof(float) * ((MODE == LAST_JET ? 0 : (size_t)IB) + (size_t)LV_PB * nw * C + LV_PB * C);
    const size_t per_pt = sizeof(float) * (size_t)nw * C * 32;
    const int pbm = (int)std::max<int64_t>(1, std::min<int64_t>(LV_PB, ((int64_t)47 * 1024 - (int64_t)fixed) / (int64_t)per_pt));
    const size_t smem = fixed + per_pt * pbm;
    int per_sm = 0;
    HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kv, I, smem));
    per_sm = std::max(1, per_sm);
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * net->num_sms, (n + LV_PB - 1) / LV_PB));
    const hrkan_pde* pde = a.pde;
    if (MODE == LAST_JET) {
      HR_LAUNCH(HRKAN_K_FWD_LAST, "k_last_v2",
                kv<<<nb, I, smem, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], n, I, net->bc,
                                        a.u ? a.u + c0 : nullptr, a.du ? a.du + c0 * NF : nullptr,
                                        a.d2u ? a.d2u + c0 * NF : nullptr, nullptr, nullptr, nullptr, 0.f, 0.f, 0.f, 0.f,
                                        nullptr, nullptr, pbm));
      return HRKAN_OK;
    }
    HR_CUDA(net->last_part.ensure(sizeof(float) * (size_t)nb * (IB + 4)));
    const float* pts = a.pts + c0 * net->D;
    const float* f = a.forcing ? a.forcing + c0 : nullptr;
    const float* g = a.g ? a.g + c0 : nullptr;
    const std::string lname = "k_last_v2 (grid " + std::to_string(nb) + ", block " + std::to_string(I) + ", smem " +
                              std::to_string(smem) + ", per_sm " + std::to_string(per_sm) + ")";
    HR_LAUNCH(HRKAN_K_FWD_LAST, lname.c_str(),
              kv<<<nb, I, smem, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], n, I, net->bc,
                                      nullptr, nullptr, nullptr, pts, f, g, pde->alpha, pde->adv, pde->visc, a.inv_n,
                                      xbar, net->last_part.f(), pbm));
    const float scale = (MODE == LAST_BOUNDARY) ? a.inv_n : pde->alpha * a.inv_n;
    HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_last",
              k_reduce_last<<<(IB + 3 + RL_COLS - 1) / RL_COLS, RL_COLS * RL_CHAINS, 0, st>>>(net->last_part.f(), nb, IB, a.grad + net->w_off[l],
                                                                   a.grad + net->b_off[l], scale, a.out_loss, a.out_flag));
    return HRKAN_OK;
  }
  auto kfn = k_last_fused<NF, NS, M, MODE, FIRST>;
  if (MODE == LAST_JET) {
    const unsigned grid = (unsigned)std::min<int64_t>(8 * net->num_sms, (n + LF_WARPS - 1) / LF_WARPS);
    HR_LAUNCH(HRKAN_K_FWD_LAST, "k_last_fused",
              kfn<<<grid, 32 * LF_WARPS, 0, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], n, I,
                                                  net->bc, a.u ? a.u + c0 : nullptr, a.du ? a.du + c0 * NF : nullptr,
                                                  a.d2u ? a.d2u + c0 * NF : nullptr, nullptr, nullptr, nullptr, 0.f,
                                                  0.f, 0.f, 0.f, nullptr, nullptr));
    return HRKAN_OK;
  }
  const size_t smem = sizeof(float) * (size_t)LF_WARPS * IB;
  if (smem > 200 * 1024) return fail(HRKAN_EUNSUPPORTED, "output layer too wide for the fused last-layer kernel");
  HR_CUDA(smem_optin(kfn, smem));
  const int per_sm = std::max(1, std::min(4, (int)((220 * 1024) / std::max<size_t>(smem, 1))));
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * net->num_sms, (n + LF_WARPS - 1) / LF_WARPS));
  HR_CUDA(net->last_part.ensure(sizeof(float) * (size_t)nb * (IB + 4)));
  const float* pts = a.pts + c0 * net->D;
  const float* f = a.forcing ? a.forcing + c0 : nullptr;
  const float* g = a.g ? a.g + c0 : nullptr;
  const hrkan_pde* pde = a.pde;
  HR_LAUNCH(HRKAN_K_FWD_LAST, "k_last_fused",
            kfn<<<nb, 32 * LF_WARPS, smem, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], n, I,
                                                 net->bc, nullptr, nullptr, nullptr, pts, f, g, pde->alpha, pde->adv,
                                                 pde->visc, a.inv_n, xbar, net->last_part.f()));
  const float scale = (MODE == LAST_BOUNDARY) ? a.inv_n : pde->alpha * a.inv_n;
  HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_last",
            k_reduce_last<<<(IB + 3 + RL_COLS - 1) / RL_COLS, RL_COLS * RL_CHAINS, 0, st>>>(net->last_part.f(), nb, IB, a.grad + net->w_off[l],
                                                                 a.grad + net->b_off[l], scale, a.out_loss, a.out_flag));
  return HRKAN_OK;
}

// First-layer forward with W staged in shared memory (k_fwd_first_s) when it fits; *done = false otherwise.
template <int NF, int NS, int M>
hrkan_status launch_fwd_first_s(hrkan_net* net, const float* X0, float* Y, int64_t n, int O, cudaStream_t st, bool* done) {
  *done = false;
  const int B = net->B;
  if (O > FL_THREADS || net->bc.k + 1 > KMAX) return HRKAN_OK;
  auto go = [&](auto KTc) -> hrkan_status {
    constexpr int KT = decltype(KTc)::value;
    const size_t smem = sizeof(FlTab<KT>) * FL_BATCH * NF + sizeof(float) * (size_t)NF * (B + 2 * KT) * O;
    if (smem > 200 * 1024) return HRKAN_OK;
    auto kfn = k_fwd_first_s<NF, NS, M, KT>;
    HR_CUDA(smem_optin(kfn, smem));
    int per_sm = 0;
    HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, FL_THREADS, smem));
    per_sm = std::max(1, per_sm);
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + FL_BATCH - 1) / FL_BATCH, (int64_t)per_sm * net->num_sms));
    HR_LAUNCH(HRKAN_K_FWD_FIRST, "k_fwd_first_s",
              kfn<<<g, FL_THREADS, smem, st>>>(X0, net->wt[0], net->params + net->b_off[0], Y, n, O, net->bc));
    *done = true;
    return HRKAN_OK;
  };
  if (net->bc.k + 1 <= 4) return go(std::integral_constant<int, 4>{});
  return go(std::integral_constant<int, 8>{});
}

// First-layer weight gradient with register accumulators (k_wgrad_first_r) for B <= 20; *done = false otherwise.
template <int NF, int NS, int M>
hrkan_status launch_wgrad_first_r(hrkan_net* net, const float* X0, const float* Ybar, float* dW, float* db, int64_t n,
                                  int O, cudaStream_t st, bool* done) {
  *done = false;
  const int B = net->B;
  if (O > FL_THREADS || B > 20 || ((1 + NF + NS) * O * 4) % 16 != 0) return HRKAN_OK;
  auto go = [&](auto BMc) -> hrkan_status {
    constexpr int BMAX = decltype(BMc)::value;
    const bool window = HRKAN_WF_WINDOW && net->bc.k <= 3;     // band-limited update (k + 1 <= 4 active bases)
    auto kfn = window ? k_wgrad_first_w<NF, NS, M, BMAX> : k_wgrad_first_r<NF, NS, M, BMAX>;
    const int pb = wf_pb(1 + NF + NS, O);
    const size_t ring = (std::max<size_t>((size_t)2 * pb * (1 + NF + NS) * O, (size_t)(FL_THREADS / O) * NF * B * O) + 3) & ~(size_t)3;
    const size_t smem = sizeof(float) * (ring + (window ? (size_t)2 * pb * NF * 20 : (size_t)pb * NF * 3 * BMAX) + FL_THREADS);
    HR_CUDA(smem_optin(kfn, smem));
    int per_sm = 0;
    HR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, FL_THREADS, smem));
    per_sm = std::max(1, per_sm);
    const int nzf = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * net->num_sms, n / 64));
    const int64_t nWf = (int64_t)O * NF * B;
    HR_CUDA(net->first_part.ensure(sizeof(float) * (size_t)nzf * (nWf + O)));
    float* fpart = net->first_part.f();
    float* fpart_b = fpart + (size_t)nzf * nWf;
    HR_LAUNCH(HRKAN_K_WGRAD_FIRST, window ? "k_wgrad_first_w" : "k_wgrad_first_r",
              kfn<<<nzf, FL_THREADS, smem, st>>>(X0, Ybar, fpart, fpart_b, n, O, net->bc));
    HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_parts",
              k_reduce_parts<<<(unsigned)((nWf + O + 255) / 256), 256, 0, st>>>(fpart, fpart_b, nzf, nWf, O, dW, db));
    *done = true;
    return HRKAN_OK;
  };
  if (B <= 12) return go(std::integral_constant<int, 12>{});
  if (B <= 16) return go(std::integral_constant<int, 16>{});
  return go(std::integral_constant<int, 20>{});
}

// Forward + (optional) loss/seeds + reverse over one point set, chunk by chunk.
template <int NF, int NS, int M>
hrkan_status run_pass(hrkan_net* net, const PassArgs& a, cudaStream_t st) {
  constexpr int C = 1 + NF + NS;
  const int L = net->L, D = net->D;
  const int64_t Pc = std::min<int64_t>(auto_chunk(net), std::max<int64_t>(a.P, 1));
  HR_TRY(ensure_workspace(net, Pc, C));
  // layer-input jet buffers: jet[l] for l = 1..L-1 (the output layer is fused with the loss)
  std::vector<float*> jet(L + 1, nullptr);
  {
    float* q = net->jets.f();
    for (int l = 1; l <= L; ++l) {
      jet[l] = q;
      q += (size_t)Pc * C * net->widths[l];
    }
  }
  const BasisCfg bc = net->bc;
  for (int64_t c0 = 0; c0 < a.P; c0 += Pc) {
    const int64_t n = std::min(Pc, a.P - c0);
    const float* X0 = a.pts + c0 * D;
    // ---------------- forward through the hidden layers
    for (int l = 0; l < L - 1; ++l) {
      const int I = net->widths[l], O = net->widths[l + 1];
      const float* in = (l == 0) ? X0 : jet[l];
      bool done = false;
      if (l > 0) HR_TRY(tc_forward_layer<NF, NS, M>(net, l, in, jet[l + 1], n, st, &done));
      if (!done) {
        const int64_t tot = n * O;
        const unsigned grid = (unsigned)((tot + 255) / 256);
        const int cls = (l == 0) ? HRKAN_K_FWD_FIRST : HRKAN_K_FWD_HIDDEN;
        if (l == 0) {
          const int bd = FL_THREADS;
          bool fast = false;
          if constexpr (NF > 0) HR_TRY(launch_fwd_first_s<NF, NS, M>(net, in, jet[l + 1], n, O, st, &fast));
          if (!fast) {
            const unsigned gf = (unsigned)std::min<int64_t>((n + FL_BATCH - 1) / FL_BATCH, 16 * net->num_sms);
            HR_LAUNCH(cls, "k_fwd_first", k_fwd_first<NF, NS, M><<<gf, bd, 0, st>>>(in, net->wt[l], net->params + net->b_off[l], jet[l + 1], n, I, O, bc));
          }
        } else
          HR_LAUNCH(cls, "k_fwd_simt", k_fwd_simt<NF, NS, M, false><<<grid, 256, 0, st>>>(in, net->wt[l], net->params + net->b_off[l], jet[l + 1], n, I, O, bc));
      }
    }
    // ---------------- output layer fused with residual, loss, seeds and its reverse (a3, a4, a8)
    const float* in_last = (L == 1) ? X0 : jet[L - 1];
    float* ybar = net->adj_a.f();
    float* xbar = net->adj_b.f();
    if (a.kind == PASS_JET) {
      if constexpr (NF == NS && NF >= 1) {
        if (L == 1) HR_TRY((launch_last<NF, NS, M, LAST_JET, true>(net, in_last, n, a, c0, nullptr, st)));
        else HR_TRY((launch_last<NF, NS, M, LAST_JET, false>(net, in_last, n, a, c0, nullptr, st)));
      }
      continue;
    }
    // the output layer emits the last hidden layer's pre-split reverse operands when that layer runs both
    // reverse kernels on the tensor cores (HRKAN_FUSE_SPLIT=0 in the environment at create time disables it)
    const bool want_split = L >= 3 && net->fuse_split && tc_reverse_ok(net, L - 2, n);
    int split_nb = 0;
    auto last = [&](auto MODEc) -> hrkan_status {
      constexpr int MODE = decltype(MODEc)::value;
      if (L == 1) return launch_last<NF, NS, M, MODE, true>(net, in_last, n, a, c0, nullptr, st);
      return launch_last<NF, NS, M, MODE, false>(net, in_last, n, a, c0, ybar, st, want_split, &split_nb);
    };
    if (a.kind == PASS_INTERIOR) {
      if (a.pde->kind == HRKAN_BURGERS) {
        if constexpr (NF == 2 && NS == 1) HR_TRY(last(std::integral_constant<int, LAST_BURGERS>{}));
        else return fail(HRKAN_EINVAL, "internal: Burgers pass needs NF=2, NS=1");
      } else {
        if constexpr (NF == NS && NF >= 1) HR_TRY(last(std::integral_constant<int, LAST_POISSON>{}));
        else return fail(HRKAN_EINVAL, "internal: Poisson pass needs NF=NS=D");
      }
    } else {
      if constexpr (NF == 0 && NS == 0) HR_TRY(last(std::integral_constant<int, LAST_BOUNDARY>{}));
      else return fail(HRKAN_EINVAL, "internal: boundary pass needs C=1");
    }
    // ---------------- reverse through the hidden layers (a5, a6, a7), last to first
    for (int l = L - 2; l >= 0; --l) {
      const int I = net->widths[l], O = net->widths[l + 1];
      const float* in = (l == 0) ? X0 : jet[l];
      float* dW = a.grad + net->w_off[l];
      float* db = a.grad + net->b_off[l];
      bool done = false;
      const bool fused = (l == L - 2) && split_nb > 0;   // operands + bias partials from the output layer
      if (l > 0 && !fused) HR_TRY(tc_split_ybar<NF, NS, M>(net, l, ybar, n, st));   // bf16 hi/lo operands of both kernels
      if (l > 0) HR_TRY(tc_wgrad_layer<NF, NS, M>(net, l, in, ybar, dW, db, n, st, &done,
                                                 fused ? net->tc_bias_part.f() : nullptr, split_nb));
      if (!done) {
        const dim3 blk(WG_J, WG_I);
        const int gx = (O + WG_J - 1) / WG_J, gy = (I + WG_I - 1) / WG_I;
        int nz = (int)std::max<int64_t>(1, (4 * net->num_sms + gx * gy - 1) / (gx * gy));
        nz = (int)std::min<int64_t>(nz, std::max<int64_t>(1, n / 64));
        nz = std::min(nz, NZ_MAX);
        const dim3 grid(gx, gy, nz);
        const size_t smem = sizeof(float) * WG_I * net->B * WG_J;
        const int cls = (l == 0) ? HRKAN_K_WGRAD_FIRST : HRKAN_K_WGRAD_HIDDEN;
        if (l == 0) {
          bool fast = false;
          if constexpr (NF > 0) HR_TRY(launch_wgrad_first_r<NF, NS, M>(net, in, ybar, dW, db, n, O, st, &fast));
          if (fast) continue;
          // first layer: batched shared basis tables, one thread per output neuron
          auto kfn = k_wgrad_first<NF, NS, M>;
          const int QG = O <= FL_THREADS ? FL_THREADS / O : 1;
          const size_t fsm = sizeof(float) * (size_t)QG * I * net->B * O;
          if (fsm > 200 * 1024 || O > 2 * FL_THREADS) return fail(HRKAN_EUNSUPPORTED, "first layer too wide");
          HR_CUDA(smem_optin(kfn, fsm));
          const int bd = FL_THREADS;
          const int nzf = (int)std::max<int64_t>(1, std::min<int64_t>(2 * net->num_sms, n / 64));
          const int64_t nWf = (int64_t)O * I * net->B;
          HR_CUDA(net->first_part.ensure(sizeof(float) * (size_t)nzf * (nWf + O)));
          float* fpart = net->first_part.f();
          float* fpart_b = fpart + (size_t)nzf * nWf;
          HR_LAUNCH(cls, "k_wgrad_first", kfn<<<nzf, bd, fsm, st>>>(in, ybar, fpart, fpart_b, n, I, O, bc));
          HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_parts",
                    k_reduce_parts<<<(unsigned)((nWf + O + 255) / 256), 256, 0, st>>>(fpart, fpart_b, nzf, nWf, O, dW, db));
          continue;
        } else {
          auto kfn = k_wgrad_simt<NF, NS, M, false>;
          HR_CUDA(smem_optin(kfn, smem));
          HR_LAUNCH(cls, "k_wgrad_simt", kfn<<<grid, blk, smem, st>>>(in, ybar, net->w_part.f(), net->b_part.f(), n, I, O, bc));
        }
        const int64_t nW = (int64_t)O * I * net->B;
        HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_parts",
                  k_reduce_parts<<<(unsigned)((nW + O + 255) / 256), 256, 0, st>>>(net->w_part.f(), net->b_part.f(), nz, nW, O, dW, db));
      }
      if (l > 0) {
        bool ddone = false;
        HR_TRY(tc_dgrad_layer<NF, NS, M>(net, l, in, ybar, xbar, n, st, &ddone));
        if (!ddone) {
          const int64_t tot = n * I;
          HR_LAUNCH(HRKAN_K_DGRAD_HIDDEN, "k_dgrad_simt",
                    k_dgrad_simt<NF, NS, M><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(in, net->params + net->w_off[l], ybar, xbar, n, I, O, bc));
        }
        std::swap(ybar, xbar);
      }
    }
  }
  return HRKAN_OK;
}

// Forward + loss/seeds + reverse of a generic jet spec S (jet_kernels.cuh), chunk by
// chunk: seeded layer-0 jet, every layer on the band-limited FFMA kernels, the Kawahara / anisotropic
// residual of the output jet, then wgrad + input adjoint from the last layer to the first.
template <class S, int M>
hrkan_status run_pass_spec(hrkan_net* net, const PassArgs& a, cudaStream_t st) {
  constexpr int C = S::C;
  const int L = net->L, D = net->D;
  if (D != S::D) return fail(HRKAN_EINVAL, "internal: jet spec dimension mismatch");
  int64_t sumw = 0;
  for (int l = 1; l <= L; ++l) sumw += net->widths[l];
  const int maxw = std::max(net->max_width, D);
  int64_t Pc = net->chunk;
  if (Pc <= 0) {
    Pc = (int64_t)(12.0e9 / (4.0 * C * (double)(sumw + 2 * maxw)));
    Pc = std::max<int64_t>(256, std::min<int64_t>(Pc, 1 << 20) / 256 * 256);
  }
  Pc = std::min<int64_t>(Pc, std::max<int64_t>(a.P, 1));
  for (int l = 0; l < L; ++l)
    if (net->widths[l + 1] > 256) return fail(HRKAN_EUNSUPPORTED, "jet-spec engine: widths up to 256");
  HR_CUDA(net->jets.ensure(sizeof(float) * (size_t)Pc * C * sumw));
  HR_CUDA(net->adj_a.ensure(sizeof(float) * (size_t)Pc * C * maxw));
  HR_CUDA(net->adj_b.ensure(sizeof(float) * (size_t)Pc * C * maxw));
  HR_CUDA(net->loss_part.ensure(sizeof(float) * 2 * (size_t)((Pc + 255) / 256 + 1)));
  HR_CUDA(net->w_part.ensure(sizeof(float) * (size_t)NZ_MAX * net->max_layer_w));
  HR_CUDA(net->b_part.ensure(sizeof(float) * (size_t)NZ_MAX * net->max_width));
  std::vector<float*> jet(L + 1, nullptr);
  {
    float* q = net->jets.f();
    for (int l = 1; l <= L; ++l) {
      jet[l] = q;
      q += (size_t)Pc * C * net->widths[l];
    }
  }
  const BasisCfg bc = net->bc;
  JsPdeArgs pa{};
  if (a.kind == PASS_INTERIOR) {
    pa.alpha = a.pde->alpha;
    pa.adv = a.pde->adv;
    pa.disp3 = a.pde->disp3;
    pa.disp5 = a.pde->disp5;
    for (int q = 0; q < 6; ++q) pa.K[q] = a.pde->aniso[q];
    pa.inv_n = a.inv_n;
  }
  for (int64_t c0 = 0; c0 < a.P; c0 += Pc) {
    const int64_t n = std::min(Pc, a.P - c0);
    const float* X0 = a.pts + c0 * D;
    float* U = (a.kind == PASS_JET) ? a.jet_out + c0 * C : jet[L];
    // ---------------- forward through every layer (a1, a2 on the generic jet)
    for (int l = 0; l < L; ++l) {
      const int I = net->widths[l], O = net->widths[l + 1];
      const float* in = (l == 0) ? X0 : jet[l];
      float* out = (l == L - 1) ? U : jet[l + 1];
      const int cls = (l == 0) ? HRKAN_K_FWD_FIRST : (l == L - 1 ? HRKAN_K_FWD_LAST : HRKAN_K_FWD_HIDDEN);
      if (O == 1) {
        const unsigned g = (unsigned)((n + JS_LW - 1) / JS_LW);
        if (l == 0) HR_LAUNCH(cls, "k_js_fwd_o1", (k_js_fwd_o1<S, M, true><<<g, 32 * JS_LW, 0, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], out, n, I, bc)));
        else HR_LAUNCH(cls, "k_js_fwd_o1", (k_js_fwd_o1<S, M, false><<<g, 32 * JS_LW, 0, st>>>(in, net->params + net->w_off[l], net->params + net->b_off[l], out, n, I, bc)));
      } else {
        const unsigned g = (unsigned)((n + JS_PT - 1) / JS_PT);
        const int bd = (O + 31) / 32 * 32;
        if (l == 0) HR_LAUNCH(cls, "k_js_fwd", (k_js_fwd<S, M, true><<<g, bd, 0, st>>>(in, net->wt[l], net->params + net->b_off[l], out, n, I, O, bc)));
        else HR_LAUNCH(cls, "k_js_fwd", (k_js_fwd<S, M, false><<<g, bd, 0, st>>>(in, net->wt[l], net->params + net->b_off[l], out, n, I, O, bc)));
      }
    }
    if (a.kind == PASS_JET) continue;
    // ---------------- residual, loss and seeds (a3 on the generic jet)
    float* ybar = net->adj_a.f();
    float* xbar = net->adj_b.f();
    const int nbl = (int)((n + 255) / 256);
    if (a.pde->kind == HRKAN_KAWAHARA) {
      if constexpr (C == 7) HR_LAUNCH(HRKAN_K_LOSS, "k_js_loss", (k_js_loss<S, JS_KAWAHARA><<<nbl, 256, 0, st>>>(U, a.forcing ? a.forcing + c0 : nullptr, ybar, net->loss_part.f(), n, pa)));
      else return fail(HRKAN_EINVAL, "internal: Kawahara needs the Taylor-5 jet");
    } else {
      if constexpr (C != 7) HR_LAUNCH(HRKAN_K_LOSS, "k_js_loss", (k_js_loss<S, JS_ANISO><<<nbl, 256, 0, st>>>(U, a.forcing + c0, ybar, net->loss_part.f(), n, pa)));
      else return fail(HRKAN_EINVAL, "internal: the anisotropic operator needs the Hessian jet");
    }
    HR_LAUNCH(HRKAN_K_REDUCE, "k_js_reduce_loss", (k_js_reduce_loss<<<1, 256, 0, st>>>(net->loss_part.f(), nbl, pa.alpha * pa.inv_n, a.out_loss, a.out_flag)));
    // ---------------- reverse, last layer to first (a4-a7 on the generic jet)
    for (int l = L - 1; l >= 0; --l) {
      const int I = net->widths[l], O = net->widths[l + 1];
      const float* in = (l == 0) ? X0 : jet[l];
      float* dW = a.grad + net->w_off[l];
      float* db = a.grad + net->b_off[l];
      const int cls = (l == 0) ? HRKAN_K_WGRAD_FIRST : (l == L - 1 ? HRKAN_K_WGRAD_LAST : HRKAN_K_WGRAD_HIDDEN);
      const int JW = (O == 1) ? 1 : 32;
      const int IW = (O == 1) ? std::min(256, (I + 31) / 32 * 32) : 8;
      const int gx = (O + JW - 1) / JW, gy = (I + IW - 1) / IW;
      int nz = (int)std::max<int64_t>(1, (4 * net->num_sms + gx * gy - 1) / (gx * gy));
      nz = (int)std::min<int64_t>(nz, std::max<int64_t>(1, n / 64));
      nz = std::min(nz, NZ_MAX);
      const size_t smem = sizeof(float) * (size_t)IW * net->B * JW;
      if (smem > 200 * 1024) return fail(HRKAN_EUNSUPPORTED, "jet-spec wgrad tile exceeds shared memory");
      auto wg = [&](auto kfn) -> hrkan_status {
        HR_CUDA(smem_optin(kfn, smem));
        HR_LAUNCH(cls, "k_js_wgrad", (kfn<<<dim3(gx, gy, nz), dim3(JW, IW), smem, st>>>(in, ybar, net->w_part.f(), net->b_part.f(), n, I, O, bc)));
        return HRKAN_OK;
      };
      if (O == 1) {
        if (l == 0) HR_TRY(wg(k_js_wgrad<S, M, true, 1>));
        else HR_TRY(wg(k_js_wgrad<S, M, false, 1>));
      } else {
        if (l == 0) HR_TRY(wg(k_js_wgrad<S, M, true, 32>));
        else HR_TRY(wg(k_js_wgrad<S, M, false, 32>));
      }
      const int64_t nW = (int64_t)O * I * net->B;
      HR_LAUNCH(HRKAN_K_REDUCE, "k_reduce_parts",
                k_reduce_parts<<<(unsigned)((nW + O + 255) / 256), 256, 0, st>>>(net->w_part.f(), net->b_part.f(), nz, nW, O, dW, db));
      if (l > 0) {
        const int64_t tot = n * I;
        HR_LAUNCH(l == L - 1 ? HRKAN_K_DGRAD_LAST : HRKAN_K_DGRAD_HIDDEN, "k_js_dgrad",
                  (k_js_dgrad<S, M><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(in, net->params + net->w_off[l], ybar, xbar, n, I, O, bc)));
        std::swap(ybar, xbar);
      }
    }
  }
  return HRKAN_OK;
}

template <class F>
hrkan_status with_channels(int nf, int ns, F&& f) {
  if (nf == 0 && ns == 0) return f(IC<0>{}, IC<0>{});
  if (nf == 1 && ns == 1) return f(IC<1>{}, IC<1>{});
  if (nf == 2 && ns == 1) return f(IC<2>{}, IC<1>{});
  if (nf == 2 && ns == 2) return f(IC<2>{}, IC<2>{});
  if (nf == 3 && ns == 3) return f(IC<3>{}, IC<3>{});
  return fail(HRKAN_EINVAL, "internal: unsupported channel set");
}

}  // namespace

// Whole loss + gradient of a tiny net in one launch (+ one reduction launch), tiny_kernels.cuh.
template <int M>
hrkan_status run_tiny(hrkan_net* net, const TinyArgs& t, cudaStream_t st) {
  TinyNet tn{};
  tn.L = net->L;
  tn.B = net->B;
  tn.np = (int)net->n_params;
  for (int l = 0; l <= net->L; ++l) tn.w[l] = net->widths[l];
  for (int l = 0; l < net->L; ++l) {
    tn.woff[l] = (int)net->w_off[l];
    tn.boff[l] = (int)net->b_off[l];
  }
  const int nb_int = (int)((t.Ni + TINY_THREADS - 1) / TINY_THREADS);
  const int nb_bnd = (int)((t.Nb + TINY_THREADS - 1) / TINY_THREADS);
  const int nb_ini = (int)((t.N0 + TINY_THREADS - 1) / TINY_THREADS);
  const int nb = std::max(1, nb_int + nb_bnd + nb_ini);
  HR_CUDA(net->last_part.ensure(sizeof(float) * (size_t)nb * (tn.np + 4)));
  if (!net->tiny_cnt.p) {                          // first call is never captured (graph mode captures the 2nd)
    HR_CUDA(net->tiny_cnt.ensure(sizeof(unsigned)));
    HR_CUDA(cudaMemsetAsync(net->tiny_cnt.p, 0, sizeof(unsigned), st));
  }
  const hrkan_pde* pde = t.pde;
  auto go = [&](auto NFc, auto NSc, auto BUR) -> hrkan_status {
    constexpr int NF = decltype(NFc)::value, NS = decltype(NSc)::value;
    constexpr bool BURGERS = decltype(BUR)::value;
    HR_LAUNCH(HRKAN_K_FUSED_STEP, "k_tiny_step",
              (k_tiny_step<NF, NS, M, BURGERS><<<nb, TINY_THREADS, 0, st>>>(
                  tn, net->params, net->bc, net->D, t.interior, t.forcing, t.Ni, nb_int, t.boundary, t.g_boundary, t.Nb,
                  nb_bnd, t.initial, t.g_initial, t.N0, pde->alpha, pde->adv, pde->visc, t.inv_int, t.inv_bi,
                  net->last_part.f(), (unsigned*)net->tiny_cnt.p, pde->alpha * t.inv_int, t.out)));
    return HRKAN_OK;
  };
  if (pde->kind == HRKAN_BURGERS) HR_TRY(go(IC<2>{}, IC<1>{}, std::true_type{}));
  else if (net->D == 1) HR_TRY(go(IC<1>{}, IC<1>{}, std::false_type{}));
  else if (net->D == 2) HR_TRY(go(IC<2>{}, IC<2>{}, std::false_type{}));
  else HR_TRY(go(IC<3>{}, IC<3>{}, std::false_type{}));
  return HRKAN_OK;
}

#define HRKAN_DEFINE_DISPATCH(MM)                                                                   \
  namespace hrkan {                                                                                \
  hrkan_status dispatch_pass_m##MM(hrkan_net* net, int nf, int ns, const PassArgs& a, cudaStream_t st) { \
    return with_channels(nf, ns, [&](auto NFc, auto NSc) {                                        \
      return run_pass<decltype(NFc)::value, decltype(NSc)::value, MM>(net, a, st);                \
    });                                                                                            \
  }                                                                                                \
  hrkan_status tiny_step_m##MM(hrkan_net* net, const TinyArgs& t, cudaStream_t st) {             \
    return run_tiny<MM>(net, t, st);                                                               \
  }                                                                                                \
  hrkan_status dispatch_spec_m##MM(hrkan_net* net, int spec, const PassArgs& a, cudaStream_t st) { \
    if (spec == JSPEC_TAYLOR5) return run_pass_spec<JsTaylor5, MM>(net, a, st);                    \
    if (spec == JSPEC_HESS2) return run_pass_spec<JsHess<2>, MM>(net, a, st);                      \
    if (spec == JSPEC_HESS3) return run_pass_spec<JsHess<3>, MM>(net, a, st);                      \
    return fail(HRKAN_EINVAL, "internal: unknown jet spec");                                       \
  }                                                                                                \
  }
