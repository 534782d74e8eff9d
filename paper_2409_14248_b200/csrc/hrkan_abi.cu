// hrkan_abi.cu -- libhrkan.so: the C ABI of include/hrkan.h, the network object and the host->device
// staging of host buffers.  The chunked loss+gradient scheduler lives in pass_impl.cuh (one
// translation unit per HR order m, pass_m<m>.cu).
//
// Every arithmetic step of the hot path runs in the kernels of simt_kernels.cuh, last_kernels.cuh
// and tc_*.cuh; this file only validates arguments, owns device memory and sequences launches on
// the caller's stream (SURVEY §3 "New build" call stack).
#include <atomic>
#include <cstdlib>

#include "hrkan_internal.cuh"
#include "simt_kernels.cuh"
#include "tc_kernels.cuh"   // weight tiling for the tensor-core engine (tc_refresh_weights, tc_free)

namespace hrkan {

thread_local std::string g_err;
static std::atomic<uint64_t> g_ws_gen{0};
uint64_t workspace_generation() { return g_ws_gen.load(std::memory_order_relaxed); }
void bump_workspace_generation() { g_ws_gen.fetch_add(1, std::memory_order_relaxed); }

hrkan_status fail(hrkan_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
void clear_error() { g_err.clear(); }

}  // namespace hrkan

namespace {

// Width padding (hrkan_net::padded): one layer of the caller's compact vector <-> the padded layout.
// dir 0: padded[o][i][n] = compact[o][i][n], padded b[o] = compact b[o] (padding stays zero);
// dir 1: the reverse gather (gradients).
__global__ void k_pad_layer(float* __restrict__ cW, float* __restrict__ cb, float* __restrict__ pW,
                            float* __restrict__ pb, int O, int IB, int IBp, int dir) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nW = (int64_t)O * IB;
  if (t >= nW + O) return;
  float *c, *q;
  if (t < nW) {
    const int64_t o = t / IB;
    c = cW + t;
    q = pW + o * IBp + (t - o * IB);
  } else {
    c = cb + (t - nW);
    q = pb + (t - nW);
  }
  if (dir == 0) *q = *c; else *c = *q;
}

// hidden width -> the width the tensor-core kernels take (64, 128, 256), or unchanged
int tc_pad_width(int w) { return w <= 64 ? 64 : w <= 128 ? 128 : 256; }

// The widths the kernels run on (see hrkan_net::padded): with at least two hidden layers, every hidden
// width in (32, 256] and B >= 8 (the tensor-core conditions of tc_layer_ok), hidden widths are
// zero-padded to 64 / 128 / 256 so that every hidden->hidden layer runs on the tensor cores
// (HRKAN_PAD_WIDTHS=0 disables it).  Returns whether any width changed.
bool execution_widths(const int32_t* widths, int n_widths, int B, std::vector<int>& out) {
  out.assign(widths, widths + n_widths);
  bool pad_ok = n_widths >= 4 && B >= 8, any = false;
  if (const char* e = std::getenv("HRKAN_PAD_WIDTHS")) pad_ok = pad_ok && std::atoi(e) != 0;
  for (int i = 1; i + 1 < n_widths; ++i) {
    pad_ok = pad_ok && widths[i] > 32 && widths[i] <= 256;
    any = any || tc_pad_width(widths[i]) != widths[i];
  }
  if (!(pad_ok && any)) return false;
  for (int i = 1; i + 1 < n_widths; ++i) out[i] = tc_pad_width(widths[i]);
  return true;
}

hrkan_status pad_copy(hrkan_net* net, float* compact, float* padded, int dir, cudaStream_t st) {
  for (int l = 0; l < net->L; ++l) {
    const int O = net->pub_widths[l + 1], IB = net->pub_widths[l] * net->B, IBp = net->widths[l] * net->B;
    const int64_t n = (int64_t)O * IB + O;
    HR_LAUNCH(HRKAN_K_OTHER, "k_pad_layer",
              k_pad_layer<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
                  compact + net->pub_w_off[l], compact + net->pub_b_off[l], padded + net->w_off[l],
                  padded + net->b_off[l], O, IB, IBp, dir));
  }
  return HRKAN_OK;
}

hrkan_status refresh_derived(hrkan_net* net, cudaStream_t st, bool force = false) {
  if (!net->derived_dirty && !force) return HRKAN_OK;
  if (net->padded) HR_TRY(pad_copy(net, net->pub_params, net->params, 0, st));
  for (int l = 0; l < net->L; ++l) {
    const int I = net->widths[l], O = net->widths[l + 1];
    const int64_t n = (int64_t)O * I * net->B;
    HR_LAUNCH(HRKAN_K_OTHER, "k_transpose_w",
              k_transpose_w<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(net->params + net->w_off[l], net->wt[l], O, I * net->B));
  }
  HR_TRY(tc_refresh_weights(net, st));
  net->derived_dirty = false;
  net->body_refreshed = true;
  return HRKAN_OK;
}

// Stage a host input (n floats) into `buf`, or pass a device pointer through.
hrkan_status stage_in(const float* src, int64_t n, DevBuf& buf, cudaStream_t st, const float** out) {
  if (!src || n == 0 || is_device_ptr(src)) {
    *out = src;
    return HRKAN_OK;
  }
  HR_CUDA(buf.ensure(sizeof(float) * (size_t)n));
  HR_CUDA(cudaMemcpyAsync(buf.p, src, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, st));
  *out = buf.f();
  return HRKAN_OK;
}


hrkan_status tiny_step(hrkan_net* net, const TinyArgs& t, cudaStream_t st) {
  switch (net->m) {
    case 2: return tiny_step_m2(net, t, st);
    case 3: return tiny_step_m3(net, t, st);
    case 4: return tiny_step_m4(net, t, st);
    case 5: return tiny_step_m5(net, t, st);
    case 6: return tiny_step_m6(net, t, st);
    case 7: return tiny_step_m7(net, t, st);
    case 8: return tiny_step_m8(net, t, st);
  }
  return fail(HRKAN_EINVAL, "m must be in [2, 8]");
}

// The one-launch tiny-net step applies: every width <= 8, <= 4 layers, few parameters.
bool tiny_eligible(const hrkan_net* net) {
  if (net->engine != 0 || net->L > 4 || net->n_params > 2048 || net->k + 1 > KMAX) return false;
  for (int w : net->widths)
    if (w > 8) return false;
  return true;
}

hrkan_status dispatch_pass(hrkan_net* net, int nf, int ns, const PassArgs& a, cudaStream_t st) {
  switch (net->m) {
    case 2: return dispatch_pass_m2(net, nf, ns, a, st);
    case 3: return dispatch_pass_m3(net, nf, ns, a, st);
    case 4: return dispatch_pass_m4(net, nf, ns, a, st);
    case 5: return dispatch_pass_m5(net, nf, ns, a, st);
    case 6: return dispatch_pass_m6(net, nf, ns, a, st);
    case 7: return dispatch_pass_m7(net, nf, ns, a, st);
    case 8: return dispatch_pass_m8(net, nf, ns, a, st);
  }
  return fail(HRKAN_EINVAL, "m must be in [2, 8]");
}

hrkan_status dispatch_spec(hrkan_net* net, int spec, const PassArgs& a, cudaStream_t st) {
  switch (net->m) {
    case 2: return dispatch_spec_m2(net, spec, a, st);
    case 3: return dispatch_spec_m3(net, spec, a, st);
    case 4: return dispatch_spec_m4(net, spec, a, st);
    case 5: return dispatch_spec_m5(net, spec, a, st);
    case 6: return dispatch_spec_m6(net, spec, a, st);
    case 7: return dispatch_spec_m7(net, spec, a, st);
    case 8: return dispatch_spec_m8(net, spec, a, st);
  }
  return fail(HRKAN_EINVAL, "m must be in [2, 8]");
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* hrkan_last_error(void) { return hrkan::g_err.c_str(); }

hrkan_status hrkan_create(const int32_t* widths, int32_t n_widths, int32_t G, int32_t k, int32_t m, float grid_lo,
                          float grid_hi, uint64_t seed, int32_t device, hrkan_net_t* out) {
  clear_error();
  if (!out) return fail(HRKAN_EINVAL, "out is NULL");
  *out = nullptr;
  if (!widths || n_widths < 2) return fail(HRKAN_EINVAL, "need at least 2 widths");
  for (int i = 0; i < n_widths; ++i)
    if (widths[i] < 1) return fail(HRKAN_EINVAL, "widths must be >= 1");
  if (widths[0] < 1 || widths[0] > 3) return fail(HRKAN_EINVAL, "widths[0] (input dimension D) must be 1, 2 or 3");
  if (widths[n_widths - 1] != 1) return fail(HRKAN_EINVAL, "the last width must be 1 (scalar PDE solution)");
  if (G < 1 || k < 1) return fail(HRKAN_EINVAL, "G and k must be >= 1");
  if (k + 1 > KMAX) return fail(HRKAN_EUNSUPPORTED, "k > 7 is not supported");
  if (G + k > 200) return fail(HRKAN_EUNSUPPORTED, "G + k > 200 is not supported");
  if (m < 2 || m > 8) return fail(HRKAN_EINVAL, "m must be in [2, 8] (second derivatives need m >= 2)");
  if (!std::isfinite(grid_lo) || !std::isfinite(grid_hi) || !(grid_lo < grid_hi))
    return fail(HRKAN_EINVAL, "grid_lo < grid_hi (finite) required");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return fail(HRKAN_EINVAL, "invalid CUDA device index");
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(HRKAN_ECUDA, "cudaGetDeviceProperties failed");
  if (prop.major != 10 || prop.minor != 0)
    return fail(HRKAN_EUNSUPPORTED, "libhrkan is built for sm_100a (B200) only; device is sm_" +
                                        std::to_string(prop.major) + std::to_string(prop.minor));
  DeviceGuard dg(device);
  hrkan_net* net = new hrkan_net();
  net->device = device;
  net->num_sms = prop.multiProcessorCount;
  net->pub_widths.assign(widths, widths + n_widths);
  net->widths = net->pub_widths;
  net->L = n_widths - 1;
  net->D = widths[0];
  net->G = G;
  net->k = k;
  net->m = m;
  net->B = G + k;
  net->lo = grid_lo;
  net->hi = grid_hi;
  const double h = ((double)grid_hi - grid_lo) / G;
  net->bc.lo = grid_lo;
  net->bc.h = (float)h;
  net->bc.inv_h = (float)(1.0 / h);
  net->bc.sc = (float)(2.0 / ((k + 1) * h));
  net->bc.mid0 = (float)(grid_lo + 0.5 * (1 - k) * h);
  net->bc.k = k;
  net->bc.B = G + k;
  net->padded = execution_widths(widths, n_widths, net->B, net->widths);
  int64_t off = 0, poff = 0;
  for (int l = 0; l < net->L; ++l) {
    const int64_t nW = (int64_t)net->widths[l + 1] * net->widths[l] * net->B;
    net->w_off.push_back(off);
    off += nW;
    net->b_off.push_back(off);
    off += net->widths[l + 1];
    net->max_layer_w = std::max(net->max_layer_w, nW);
    net->max_width = std::max(net->max_width, net->widths[l + 1]);
    net->pub_w_off.push_back(poff);
    poff += (int64_t)widths[l + 1] * widths[l] * net->B;
    net->pub_b_off.push_back(poff);
    poff += widths[l + 1];
  }
  net->n_params = off;
  net->pub_n_params = poff;
  // tuning overrides for experiments (precision/speed trade-off of the TMEM drain segments)
  if (const char* e = std::getenv("HRKAN_TC_SEG")) net->tc_seg = net->tc_seg_single = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("HRKAN_TC_WSEG")) net->tc_wseg = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("HRKAN_FUSE_SPLIT")) net->fuse_split = std::atoi(e) != 0;
  if (const char* e = std::getenv("HRKAN_TC_DBG")) net->tc_dbg = std::atoi(e);
  auto cleanup = [&](hrkan_status s) {
    hrkan_free(net);
    return s;
  };
  if (cudaMalloc(&net->params, sizeof(float) * off) != cudaSuccess ||
      cudaMalloc(&net->adam_m, sizeof(float) * poff) != cudaSuccess ||
      cudaMalloc(&net->adam_v, sizeof(float) * poff) != cudaSuccess ||
      cudaMalloc(&net->adam_t, 2 * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    return cleanup(fail(HRKAN_ENOMEM, "parameter allocation failed"));
  }
  net->pub_params = net->params;
  if (net->padded) {
    net->pub_params = nullptr;
    if (cudaMalloc(&net->pub_params, sizeof(float) * poff) != cudaSuccess ||
        cudaMemset(net->params, 0, sizeof(float) * off) != cudaSuccess) {   // the padding stays zero for good
      cudaGetLastError();
      return cleanup(fail(HRKAN_ENOMEM, "parameter allocation failed"));
    }
  }
  net->wt.assign(net->L, nullptr);
  for (int l = 0; l < net->L; ++l) {
    if (cudaMalloc(&net->wt[l], sizeof(float) * (size_t)net->widths[l + 1] * net->widths[l] * net->B) != cudaSuccess) {
      cudaGetLastError();
      return cleanup(fail(HRKAN_ENOMEM, "weight copy allocation failed"));
    }
  }
  hrkan_status s = hrkan_init_params(net, seed, nullptr);
  if (s != HRKAN_OK) return cleanup(s);
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(HRKAN_ECUDA, "init failed"));
  *out = net;
  return HRKAN_OK;
}

hrkan_status hrkan_execution_widths(const int32_t* widths, int32_t n_widths, int32_t G, int32_t k, int32_t* out) {
  if (!widths || !out || n_widths < 2) return fail(HRKAN_EINVAL, "NULL argument or fewer than 2 widths");
  if (G < 1 || k < 1) return fail(HRKAN_EINVAL, "G and k must be >= 1");
  for (int i = 0; i < n_widths; ++i)
    if (widths[i] < 1) return fail(HRKAN_EINVAL, "widths must be >= 1");
  std::vector<int> w;
  execution_widths(widths, n_widths, G + k, w);
  for (int i = 0; i < n_widths; ++i) out[i] = w[i];
  return HRKAN_OK;
}

int64_t hrkan_num_params(hrkan_net_t net) { return net ? net->pub_n_params : -1; }

int64_t hrkan_launch_count(hrkan_net_t net) { return net ? net->launches : -1; }

hrkan_status hrkan_set_chunk_points(hrkan_net_t net, int64_t chunk) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  if (chunk < 0) return fail(HRKAN_EINVAL, "chunk must be >= 0");
  net->chunk = chunk == 0 ? 0 : std::max<int64_t>(1, chunk);
  return HRKAN_OK;
}

hrkan_status hrkan_set_engine(hrkan_net_t net, int32_t mode) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  if (mode < 0 || mode > 2) return fail(HRKAN_EINVAL, "engine mode must be 0, 1 or 2");
  // the engine decides which derived weight copies refresh_derived maintains (engine 1 skips the
  // tensor-core tiles): any change re-derives all of them before the next call
  if (mode != net->engine) net->derived_dirty = true;
  net->engine = mode;
  return HRKAN_OK;
}

hrkan_status hrkan_init_params(hrkan_net_t net, uint64_t seed, void* stream) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  DeviceGuard dg(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  for (int l = 0; l < net->L; ++l) {
    const int I = net->pub_widths[l], O = net->pub_widths[l + 1];     // the caller's (unpadded) layer
    const int64_t nW = (int64_t)O * I * net->B;
    const float stdv = (float)(1.0 / std::sqrt((double)I * net->B));
    const int64_t n = std::max<int64_t>(nW, O);
    k_init_layer<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(net->pub_params + net->pub_w_off[l],
                                                              net->pub_params + net->pub_b_off[l], nW, O, stdv, seed,
                                                              (uint32_t)l);
    HR_TRY(check_launch(net, "k_init_layer"));
  }
  HR_CUDA(cudaMemsetAsync(net->adam_m, 0, sizeof(float) * net->pub_n_params, st));
  HR_CUDA(cudaMemsetAsync(net->adam_v, 0, sizeof(float) * net->pub_n_params, st));
  HR_CUDA(cudaMemsetAsync(net->adam_t, 0, 2 * sizeof(int), st));
  net->derived_dirty = true;
  return HRKAN_OK;
}

hrkan_status hrkan_get_params(hrkan_net_t net, float* dst, void* stream) {
  if (!net || !dst) return fail(HRKAN_EINVAL, "NULL argument");
  DeviceGuard dg(net->device);
  HR_CUDA(cudaMemcpyAsync(dst, net->pub_params, sizeof(float) * net->pub_n_params, cudaMemcpyDefault, (cudaStream_t)stream));
  return HRKAN_OK;
}

hrkan_status hrkan_set_params(hrkan_net_t net, const float* src, void* stream) {
  if (!net || !src) return fail(HRKAN_EINVAL, "NULL argument");
  DeviceGuard dg(net->device);
  HR_CUDA(cudaMemcpyAsync(net->pub_params, src, sizeof(float) * net->pub_n_params, cudaMemcpyDefault, (cudaStream_t)stream));
  net->derived_dirty = true;
  return HRKAN_OK;
}

hrkan_status hrkan_forward_jet(hrkan_net_t net, const float* pts, int64_t P, float* u, float* du, float* d2u,
                               void* stream) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  if (P < 0) return fail(HRKAN_EINVAL, "P must be >= 0");
  if (P == 0) return HRKAN_OK;
  if (!pts) return fail(HRKAN_EINVAL, "pts is NULL");
  clear_error();
  DeviceGuard dg(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int D = net->D;
  const float* dpts;
  HR_TRY(stage_in(pts, P * D, net->st_pts, st, &dpts));
  float* du_dev = du;
  float* u_dev = u;
  float* d2u_dev = d2u;
  const bool hu = u && !is_device_ptr(u), hdu = du && !is_device_ptr(du), hd2u = d2u && !is_device_ptr(d2u);
  if (hu) { HR_CUDA(net->st_u.ensure(sizeof(float) * P)); u_dev = net->st_u.f(); }
  if (hdu) { HR_CUDA(net->st_du.ensure(sizeof(float) * P * D)); du_dev = net->st_du.f(); }
  if (hd2u) { HR_CUDA(net->st_d2u.ensure(sizeof(float) * P * D)); d2u_dev = net->st_d2u.f(); }
  HR_TRY(refresh_derived(net, st));
  PassArgs a{};
  a.kind = PASS_JET;
  a.pts = dpts;
  a.P = P;
  a.u = u_dev;
  a.du = du_dev;
  a.d2u = d2u_dev;
  HR_TRY(dispatch_pass(net, D, D, a, st));
  if (hu) HR_CUDA(cudaMemcpyAsync(u, u_dev, sizeof(float) * P, cudaMemcpyDeviceToHost, st));
  if (hdu) HR_CUDA(cudaMemcpyAsync(du, du_dev, sizeof(float) * P * D, cudaMemcpyDeviceToHost, st));
  if (hd2u) HR_CUDA(cudaMemcpyAsync(d2u, d2u_dev, sizeof(float) * P * D, cudaMemcpyDeviceToHost, st));
  return HRKAN_OK;
}

hrkan_status hrkan_forward_jet_ex(hrkan_net_t net, int32_t kind, const float* pts, int64_t P, float* jet, void* stream) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  if (P < 0) return fail(HRKAN_EINVAL, "P must be >= 0");
  if (kind != HRKAN_JET_TAYLOR5 && kind != HRKAN_JET_HESSIAN) return fail(HRKAN_EINVAL, "unknown jet kind");
  if (kind == HRKAN_JET_TAYLOR5 && (net->D != 2 || net->m < 3))
    return fail(HRKAN_EINVAL, "the Taylor-5 jet needs D = 2 (x, t) and m >= 3");
  if (kind == HRKAN_JET_HESSIAN && net->D < 2) return fail(HRKAN_EINVAL, "the Hessian jet needs D = 2 or 3");
  if (P == 0) return HRKAN_OK;
  if (!pts || !jet) return fail(HRKAN_EINVAL, "NULL pts / jet");
  clear_error();
  DeviceGuard dg(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const int D = net->D;
  const int C = kind == HRKAN_JET_TAYLOR5 ? 7 : 1 + D + D * (D + 1) / 2;
  const float* dpts;
  HR_TRY(stage_in(pts, P * D, net->st_pts, st, &dpts));
  float* jet_dev = jet;
  const bool hj = !is_device_ptr(jet);
  if (hj) {
    HR_CUDA(net->st_u.ensure(sizeof(float) * P * C));
    jet_dev = net->st_u.f();
  }
  HR_TRY(refresh_derived(net, st));
  PassArgs a{};
  a.kind = PASS_JET;
  a.pts = dpts;
  a.P = P;
  a.jet_out = jet_dev;
  const int spec = kind == HRKAN_JET_TAYLOR5 ? JSPEC_TAYLOR5 : (D == 2 ? JSPEC_HESS2 : JSPEC_HESS3);
  HR_TRY(dispatch_spec(net, spec, a, st));
  if (hj) HR_CUDA(cudaMemcpyAsync(jet, jet_dev, sizeof(float) * P * C, cudaMemcpyDeviceToHost, st));
  return HRKAN_OK;
}

}  // extern "C"

namespace {

// The work of hrkan_pinn_loss_grad after argument validation (stream-ordered launches only).
hrkan_status loss_grad_body(hrkan_net* net, const hrkan_pde* pde, const float* interior, const float* forcing,
                            int64_t Ni, const float* boundary, const float* g_boundary, int64_t Nb,
                            const float* initial, const float* g_initial, int64_t N0, int64_t Ni_global,
                            int64_t Nbi_global, float* out, cudaStream_t st, bool force_refresh) {
  const int D = net->D;
  const int64_t np = net->n_params;        // gradient length of the net the kernels run on (padded or not)
  const int64_t pnp = net->pub_n_params;   // the caller's vector: [dθ (pnp) | aL_pde | L_bi | flag | pad]
  const float *d_int, *d_f = nullptr, *d_bnd, *d_gb, *d_ini, *d_gi;
  HR_TRY(stage_in(interior, Ni * D, net->st_int, st, &d_int));
  if (forcing && (pde->kind == HRKAN_POISSON || pde->kind == HRKAN_ANISO)) HR_TRY(stage_in(forcing, Ni, net->st_f, st, &d_f));
  HR_TRY(stage_in(boundary, Nb * D, net->st_bnd, st, &d_bnd));
  HR_TRY(stage_in(g_boundary, Nb, net->st_gb, st, &d_gb));
  HR_TRY(stage_in(initial, N0 * D, net->st_ini, st, &d_ini));
  HR_TRY(stage_in(g_initial, N0, net->st_gi, st, &d_gi));
  float* dout = out;
  const bool host_out = !is_device_ptr(out);
  if (host_out) {
    HR_CUDA(net->st_out.ensure(sizeof(float) * (pnp + 4)));
    dout = net->st_out.f();
  }
  float* const cout_ = dout;               // compact result (device)
  if (net->padded) {                        // the passes accumulate into the padded layout, gathered at the end
    HR_CUDA(net->pad_grad.ensure(sizeof(float) * (np + 4)));
    dout = net->pad_grad.f();
  }
  if (tiny_eligible(net) && (pde->kind == HRKAN_POISSON || pde->kind == HRKAN_BURGERS)) {
    TinyArgs t{pde, d_int, d_f, d_bnd, d_gb, d_ini, d_gi, Ni, Nb, N0, (float)(1.0 / (double)std::max<int64_t>(1, Ni_global)),
               Nbi_global > 0 ? (float)(1.0 / (double)Nbi_global) : 0.f, dout};
    HR_TRY(tiny_step(net, t, st));
    if (host_out) HR_CUDA(cudaMemcpyAsync(out, dout, sizeof(float) * (pnp + 4), cudaMemcpyDeviceToHost, st));
    return HRKAN_OK;
  }
  HR_CUDA(cudaMemsetAsync(dout, 0, sizeof(float) * (np + 4), st));
  HR_TRY(refresh_derived(net, st, force_refresh));
  PassArgs a{};
  a.grad = dout;
  a.pde = pde;
  a.out_flag = dout + np + 2;
  if (Ni > 0) {
    a.kind = PASS_INTERIOR;
    a.pts = d_int;
    a.P = Ni;
    a.forcing = d_f;
    a.out_loss = dout + np;
    a.inv_n = (float)(1.0 / (double)Ni_global);
    if (pde->kind == HRKAN_KAWAHARA) {
      HR_TRY(dispatch_spec(net, JSPEC_TAYLOR5, a, st));
    } else if (pde->kind == HRKAN_ANISO) {
      HR_TRY(dispatch_spec(net, D == 2 ? JSPEC_HESS2 : JSPEC_HESS3, a, st));
    } else {
      const int nf = D, ns = (pde->kind == HRKAN_BURGERS) ? 1 : D;
      HR_TRY(dispatch_pass(net, nf, ns, a, st));
    }
  }
  a.kind = PASS_BOUNDARY;
  a.out_loss = dout + np + 1;
  a.inv_n = Nbi_global > 0 ? (float)(1.0 / (double)Nbi_global) : 0.f;
  a.forcing = nullptr;
  if (Nb > 0) {
    a.pts = d_bnd;
    a.P = Nb;
    a.g = d_gb;
    HR_TRY(dispatch_pass(net, 0, 0, a, st));
  }
  if (N0 > 0) {
    a.pts = d_ini;
    a.P = N0;
    a.g = d_gi;
    HR_TRY(dispatch_pass(net, 0, 0, a, st));
  }
  if (net->padded) {
    HR_TRY(pad_copy(net, cout_, dout, 1, st));
    HR_CUDA(cudaMemcpyAsync(cout_ + pnp, dout + np, 4 * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  if (host_out) HR_CUDA(cudaMemcpyAsync(out, cout_, sizeof(float) * (pnp + 4), cudaMemcpyDeviceToHost, st));
  return HRKAN_OK;
}


bool same_key(const GraphKey& a, const GraphKey& b) { return std::memcmp(&a, &b, sizeof(GraphKey)) == 0; }

}  // namespace

extern "C" {

hrkan_status hrkan_pinn_loss_grad(hrkan_net_t net, const hrkan_pde* pde, const float* interior, const float* forcing,
                                  int64_t Ni, const float* boundary, const float* g_boundary, int64_t Nb,
                                  const float* initial, const float* g_initial, int64_t N0, int64_t Ni_global,
                                  int64_t Nbi_global, float* out, void* stream) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  if (!pde) return fail(HRKAN_EINVAL, "pde is NULL");
  if (!out) return fail(HRKAN_EINVAL, "out is NULL");
  if (Ni < 0 || Nb < 0 || N0 < 0) return fail(HRKAN_EINVAL, "negative point count");
  if ((Ni > 0 && !interior) || (Nb > 0 && (!boundary || !g_boundary)) || (N0 > 0 && (!initial || !g_initial)))
    return fail(HRKAN_EINVAL, "NULL point/target buffer with a non-zero count");
  if (Ni_global < Ni || Nbi_global < Nb + N0) return fail(HRKAN_EINVAL, "global normalisers smaller than local counts");
  if (pde->kind < HRKAN_POISSON || pde->kind > HRKAN_ANISO) return fail(HRKAN_EINVAL, "unknown pde kind");
  if (pde->kind == HRKAN_BURGERS && net->D != 2) return fail(HRKAN_EINVAL, "Burgers needs D = 2 (x, t)");
  if (pde->kind == HRKAN_KAWAHARA && net->D != 2) return fail(HRKAN_EINVAL, "Kawahara needs D = 2 (x, t)");
  if (pde->kind == HRKAN_KAWAHARA && net->m < 3)
    return fail(HRKAN_EINVAL, "u_xxxxx needs m >= 3 (v^(5) = 0 for m = 2; m >= 6 makes it continuous, P:102)");
  if (pde->kind == HRKAN_ANISO && net->D < 2) return fail(HRKAN_EINVAL, "the anisotropic operator needs D = 2 or 3");
  if (pde->kind == HRKAN_ANISO && Ni > 0 && !forcing) return fail(HRKAN_EINVAL, "the anisotropic operator needs a forcing");
  if (!std::isfinite(pde->alpha)) return fail(HRKAN_EINVAL, "alpha must be finite");
  clear_error();
  DeviceGuard dg(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  // CUDA-graph replay (hrkan_set_graph_mode): device buffers only, non-legacy stream, not already
  // inside a caller's capture, no per-launch profiling.  The first call with a new argument
  // signature runs eagerly (allocating every workspace), the second captures the whole call
  // (weight re-tiling included, since Adam changes the parameters between calls) and every later
  // call replays it with one cudaGraphLaunch.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  bool graph_ok = net->graph_mode && !net->prof_on && st != nullptr &&
                  cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone;
  if (graph_ok) {
    const void* ptrs[] = {interior, forcing, boundary, g_boundary, initial, g_initial, out};
    for (const void* q : ptrs) graph_ok = graph_ok && is_device_ptr(q);
  }
  cudaGetLastError();
  if (!graph_ok)
    return loss_grad_body(net, pde, interior, forcing, Ni, boundary, g_boundary, Nb, initial, g_initial, N0, Ni_global,
                          Nbi_global, out, st, false);
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  const void* kp[] = {interior, forcing, boundary, g_boundary, initial, g_initial, out, st};
  std::memcpy(key.ptrs, kp, sizeof(kp));
  key.n[0] = Ni; key.n[1] = Nb; key.n[2] = N0; key.n[3] = Ni_global; key.n[4] = Nbi_global; key.n[5] = net->chunk;
  key.kind = pde->kind; key.engine = net->engine;
  key.f[0] = pde->alpha; key.f[1] = pde->adv; key.f[2] = pde->visc; key.f[3] = pde->disp3; key.f[4] = pde->disp5;
  for (int q = 0; q < 6; ++q) key.f[5 + q] = pde->aniso[q];
  key.ws_gen = workspace_generation();
  if (net->graph_exec && same_key(key, net->graph_key)) {
    HR_CUDA(cudaGraphLaunch(net->graph_exec, st));
    net->launches += net->graph_launches;
    if (net->graph_refreshes) net->derived_dirty = false;   // the tiny-net body never re-derives
    return HRKAN_OK;
  }
  if (!same_key(key, net->graph_key)) {           // new signature: run eagerly, capture next time
    if (net->graph_exec) cudaGraphExecDestroy(net->graph_exec);
    net->graph_exec = nullptr;
    net->graph_key = key;
    return loss_grad_body(net, pde, interior, forcing, Ni, boundary, g_boundary, Nb, initial, g_initial, N0, Ni_global,
                          Nbi_global, out, st, false);
  }
  const int64_t l0 = net->launches;
  const bool dirty0 = net->derived_dirty;
  net->body_refreshed = false;
  HR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const hrkan_status sb = loss_grad_body(net, pde, interior, forcing, Ni, boundary, g_boundary, Nb, initial, g_initial,
                                         N0, Ni_global, Nbi_global, out, st, true);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(st, &graph);
  net->graph_launches = net->launches - l0;
  net->launches = l0;
  net->graph_refreshes = net->body_refreshed;
  net->derived_dirty = dirty0;        // capture records launches without running them
  if (sb != HRKAN_OK || ec != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    std::memset(&net->graph_key, 0, sizeof(GraphKey));
    if (sb != HRKAN_OK) return sb;
    return fail(HRKAN_ECUDA, std::string("graph capture failed: ") + cudaGetErrorString(ec));
  }
  const cudaError_t ei = cudaGraphInstantiate(&net->graph_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    net->graph_exec = nullptr;
    std::memset(&net->graph_key, 0, sizeof(GraphKey));
    return fail(HRKAN_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
  }
  net->graph_key.ws_gen = workspace_generation();   // capture itself never reallocates
  HR_CUDA(cudaGraphLaunch(net->graph_exec, st));
  net->launches += net->graph_launches;
  if (net->graph_refreshes) net->derived_dirty = false;
  return HRKAN_OK;
}

hrkan_status hrkan_set_graph_mode(hrkan_net_t net, int32_t enable) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  net->graph_mode = enable != 0;
  if (!net->graph_mode && net->graph_exec) {
    cudaGraphExecDestroy(net->graph_exec);
    net->graph_exec = nullptr;
  }
  std::memset(&net->graph_key, 0, sizeof(GraphKey));
  return HRKAN_OK;
}

hrkan_status hrkan_adam_step(hrkan_net_t net, const float* grad, float lr, float beta1, float beta2, float eps,
                             void* stream) {
  if (!net || !grad) return fail(HRKAN_EINVAL, "NULL argument");
  if (!std::isfinite(lr) || !std::isfinite(eps) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f))
    return fail(HRKAN_EINVAL, "invalid Adam hyper-parameters");
  DeviceGuard dg(net->device);
  cudaStream_t st = (cudaStream_t)stream;
  const float* dg_ptr;
  HR_TRY(stage_in(grad, net->pub_n_params, net->st_out, st, &dg_ptr));
  const int64_t n = net->pub_n_params;
  HR_LAUNCH(HRKAN_K_ADAM, "k_adam",
            k_adam<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(net->pub_params, net->adam_m, net->adam_v, dg_ptr, n, lr, beta1,
                                                                beta2, eps, net->adam_t));
  net->derived_dirty = true;
  return HRKAN_OK;
}

hrkan_status hrkan_profile_enable(hrkan_net_t net, int32_t enable) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  net->prof_on = enable != 0;
  return HRKAN_OK;
}

hrkan_status hrkan_profile_read(hrkan_net_t net, double* ms, int64_t* n) {
  if (!net) return fail(HRKAN_EINVAL, "net is NULL");
  DeviceGuard dg(net->device);
  double acc[HRKAN_K_NUM_CLASSES] = {0};
  int64_t cnt[HRKAN_K_NUM_CLASSES] = {0};
  for (size_t i = 0; i < net->prof_used; ++i) {
    const auto& ev = net->prof_pool[i];
    HR_CUDA(cudaEventSynchronize(ev.b));
    float t = 0.f;
    HR_CUDA(cudaEventElapsedTime(&t, ev.a, ev.b));
    acc[ev.cls] += t;
    cnt[ev.cls] += 1;
  }
  net->prof_used = 0;
  for (int c = 0; c < HRKAN_K_NUM_CLASSES; ++c) {
    if (ms) ms[c] = acc[c];
    if (n) n[c] = cnt[c];
  }
  return HRKAN_OK;
}

void hrkan_free(hrkan_net_t net) {
  if (!net) return;
  DeviceGuard dg(net->device);
  cudaDeviceSynchronize();
  if (net->graph_exec) cudaGraphExecDestroy(net->graph_exec);
  for (auto& ev : net->prof_pool) {
    cudaEventDestroy(ev.a);
    cudaEventDestroy(ev.b);
  }
  if (net->pub_params != net->params) cudaFree(net->pub_params);
  cudaFree(net->params);
  cudaFree(net->adam_m);
  cudaFree(net->adam_v);
  cudaFree(net->adam_t);
  for (float* p : net->wt) cudaFree(p);
  DevBuf* bufs[] = {&net->jets, &net->adj_a, &net->adj_b, &net->loss_part, &net->w_part, &net->b_part, &net->last_part, &net->first_part,
                    &net->st_int, &net->st_f, &net->st_bnd, &net->st_gb, &net->st_ini, &net->st_gi,
                    &net->st_out, &net->st_pts, &net->st_u, &net->st_du, &net->st_d2u, &net->tc_ws,
                    &net->tc_yw, &net->tc_yd, &net->tiny_cnt, &net->pad_grad, &net->tc_bias_part};
  for (DevBuf* b : bufs) b->release();
  tc_free(net);
  delete net;
}

}  // extern "C"
