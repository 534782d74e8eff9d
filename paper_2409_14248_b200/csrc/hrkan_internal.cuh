// hrkan_internal.cuh -- the network object and the host helpers shared by the translation units of
// libhrkan.so (hrkan_abi.cu: the C ABI; pass_m<M>.cu: the chunked loss+gradient scheduler
// instantiated for HR order M, compiled in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/hrkan.h"
#include "hr_basis.cuh"

using namespace hrkan;

namespace hrkan {

// Records the thread-local error message returned by hrkan_last_error() (hrkan_abi.cu).
hrkan_status fail(hrkan_status s, const std::string& msg);
void clear_error();

#define HR_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(HRKAN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

#define HR_TRY(...)                     \
  do {                                  \
    hrkan_status s_ = (__VA_ARGS__);    \
    if (s_ != HRKAN_OK) return s_;      \
  } while (0)

template <int V>
using IC = std::integral_constant<int, V>;

// RAII current-device switch (the caller's current device is restored).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline bool is_device_ptr(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Process-wide count of workspace reallocations.  A captured CUDA graph bakes in raw workspace
// pointers, so the graph key of hrkan_pinn_loss_grad carries this generation and any reallocation
// (e.g. a larger hrkan_forward_jet between training steps) forces a re-capture.
uint64_t workspace_generation();
void bump_workspace_generation();

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    bump_workspace_generation();
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  float* f() const { return static_cast<float*>(p); }
};

// Per-layer state of the tensor-core engine (tc_kernels.cuh).
struct TcLayerState {
  uint16_t* w_fwd = nullptr;   // pre-tiled, bf16 hi/lo-split W for the forward kernel
  uint16_t* w_dgr = nullptr;   // pre-tiled, bf16 hi/lo-split W^T for the dgrad kernel
  int nkb = 0;              // forward K-blocks
  int ntile_dgr = 0;        // dgrad M-tiles
};

}  // namespace hrkan

using namespace hrkan;

// Argument signature of a captured hrkan_pinn_loss_grad call (CUDA-graph replay).
struct GraphKey {
  const void* ptrs[8];
  int64_t n[6];
  uint64_t ws_gen;                     // workspace_generation() when the signature was recorded
  float f[11];
  int32_t kind, engine;
};

struct hrkan_net {
  int device = 0;
  int L = 0, D = 0, G = 0, k = 0, m = 0, B = 0;
  float lo = -1.f, hi = 1.f;
  std::vector<int> widths;
  std::vector<int64_t> w_off, b_off;   // offsets into the flat parameter vector
  int64_t n_params = 0;
  int64_t max_layer_w = 0;
  int max_width = 0;                   // max over widths[1..L]
  BasisCfg bc{};
  float* params = nullptr;             // flat, owned (the layout the kernels run on: `widths`)
  // Width padding (hrkan_create): hidden widths in (32, 256] that the tensor-core kernels do not take
  // (they need 64, 128 or 256 neurons) are zero-padded up to the next such width.  `widths`, `w_off`,
  // `b_off`, `n_params` and `params` then describe the padded net the kernels run on; the public
  // parameter / gradient vectors keep the caller's compact layout (`pub_*`), which is also the Adam
  // master copy.  Padded neurons have zero weights and bias, so they emit an all-zero jet and receive a
  // zero adjoint: the compact entries of every result are unchanged.  Not padded: pub_params == params.
  bool padded = false;
  std::vector<int> pub_widths;
  std::vector<int64_t> pub_w_off, pub_b_off;
  int64_t pub_n_params = 0;
  float* pub_params = nullptr;
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  int* adam_t = nullptr;               // device [t, finished-block counter]: k_adam increments t on the
                                       // device, so a captured Adam step keeps its bias correction live
  std::vector<float*> wt;              // derived: W_l transposed to [I][B][O]
  bool derived_dirty = true;
  int64_t chunk = 0;                   // 0 = auto
  int engine = 0;
  int64_t launches = 0;
  int num_sms = 148;
  // workspace
  DevBuf jets, adj_a, adj_b, loss_part, w_part, b_part, last_part, first_part;
  DevBuf st_int, st_f, st_bnd, st_gb, st_ini, st_gi, st_out, st_pts, st_u, st_du, st_d2u;
  DevBuf tc_ws;                         // tensor-core path scratch
  DevBuf tiny_cnt;                      // k_tiny_step's finished-block counter (reset by the last block)
  DevBuf tc_yw, tc_yd;                  // pre-split bf16 hi/lo Ybar operands of the reverse kernels
  DevBuf pad_grad;                      // [n_params + 4] gradient of the padded net (gathered into the caller's compact vector)
  DevBuf tc_bias_part;                  // bias-gradient partials emitted by the fused output layer (k_last_v3 SPLIT)
  std::vector<TcLayerState> tc_layers;
  int tc_seg = 96;                      // K-blocks per forward TMEM segment, double-buffered accumulators (C3/C4: one segment;
                                        // the drains run on the generator warps: C4 fwd 3.79 -> 3.11 ms, u 1.2e-5 -> 1.7e-5)
  int tc_seg_single = 160;              // ... single accumulator (the drain stalls the MMA): C5 -> 2 segments
  int tc_wseg = 256;                    // wgrad stages per TMEM drain into the fp32 master
  bool fuse_split = true;               // output layer emits the last hidden layer's pre-split operands (HRKAN_FUSE_SPLIT)
  int tc_dbg = 0;                       // timing-experiment switches (HRKAN_TC_DBG; 0 in production)
  // CUDA-graph replay of hrkan_pinn_loss_grad (hrkan_set_graph_mode)
  bool graph_mode = false;
  GraphKey graph_key{};
  cudaGraphExec_t graph_exec = nullptr;
  int64_t graph_launches = 0;
  bool graph_refreshes = false;         // the captured body re-tiles the derived weight copies
  bool body_refreshed = false;          // set by refresh_derived (capture bookkeeping)
  // device-time profiling (hrkan_profile_enable / hrkan_profile_read)
  struct ProfEv { cudaEvent_t a, b; int cls; };
  bool prof_on = false;
  std::vector<ProfEv> prof_pool;
  size_t prof_used = 0;
};

namespace hrkan {

constexpr int NZ_MAX = 64;

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
using PFN_tmapEncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                         const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                         CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PFN_tmapEncodeTiled tmap_encoder() {
  static PFN_tmapEncodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmapEncodeTiled>(f);
    else
      cudaGetLastError();
  }
  return fn;
}

// fp32 3-D tensor map over a row-major [d2][d1][d0] array (d0 innermost), box b0 x b1 x b2, no swizzle,
// zero fill out of bounds.  Requires 16-B aligned base and d0*4, d0*d1*4 multiples of 16.
inline hrkan_status make_tmap_f32_3d(CUtensorMap* m, const float* base, uint64_t d0, uint64_t d1, uint64_t d2,
                                     uint32_t b0, uint32_t b1, uint32_t b2) {
  PFN_tmapEncodeTiled enc = tmap_encoder();
  if (!enc) return fail(HRKAN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HRKAN_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return HRKAN_OK;
}

// Opt a kernel into `dyn` bytes of dynamic shared memory whenever its static + dynamic shared memory
// exceeds the 48 KB default (the static part counts: k_wgrad_first at O = 128, D = 3 needs it).
template <class K>
inline cudaError_t smem_optin(K kfn, size_t dyn) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, (const void*)kfn);
  if (e != cudaSuccess) return e;
  if (fa.sharedSizeBytes + dyn <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute((const void*)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
}

inline int prof_pre(hrkan_net* net, cudaStream_t st) {
  if (!net->prof_on) return -1;
  if (net->prof_used == net->prof_pool.size()) {
    hrkan_net::ProfEv ev{};
    if (cudaEventCreate(&ev.a) != cudaSuccess || cudaEventCreate(&ev.b) != cudaSuccess) return -1;
    net->prof_pool.push_back(ev);
  }
  cudaEventRecord(net->prof_pool[net->prof_used].a, st);
  return (int)net->prof_used++;
}

inline hrkan_status check_launch(hrkan_net* net, const char* what, int cls = HRKAN_K_OTHER, cudaStream_t st = nullptr,
                          int prof_idx = -1) {
  net->launches++;
  cudaError_t e = cudaGetLastError();
  if (prof_idx >= 0) {
    cudaEventRecord(net->prof_pool[prof_idx].b, st);
    net->prof_pool[prof_idx].cls = cls;
  }
  if (e != cudaSuccess) return fail(HRKAN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HRKAN_OK;
}

// Launch statement bracketed by profiling events and followed by the launch-error check.
#define HR_LAUNCH(CLS, NAME, ...)                                   \
  do {                                                              \
    const int pi_ = prof_pre(net, st);                              \
    __VA_ARGS__;                                                    \
    HR_TRY(check_launch(net, NAME, CLS, st, pi_));                  \
  } while (0)

}  // namespace hrkan


namespace hrkan {

inline int64_t auto_chunk(const hrkan_net* net) {
  if (net->chunk > 0) return net->chunk;
  const int C = 1 + 2 * net->D;
  int64_t sumw = 0;
  for (int l = 1; l <= net->L; ++l) sumw += net->widths[l];
  const double bytes_per_point = 4.0 * C * (double)(sumw + 2 * net->max_width) * 1.0;
  const double budget = 12.0e9;
  int64_t c = (int64_t)(budget / bytes_per_point);
  c = std::min<int64_t>(c, 1 << 20);
  c = std::max<int64_t>(256, c / 256 * 256);
  return c;
}

// Workspace for chunks of Pc points with C channels.
inline hrkan_status ensure_workspace(hrkan_net* net, int64_t Pc, int C) {
  int64_t sumw = 0;
  for (int l = 1; l <= net->L; ++l) sumw += net->widths[l];
  HR_CUDA(net->jets.ensure(sizeof(float) * (size_t)Pc * C * sumw));
  HR_CUDA(net->adj_a.ensure(sizeof(float) * (size_t)Pc * C * net->max_width));
  HR_CUDA(net->adj_b.ensure(sizeof(float) * (size_t)Pc * C * net->max_width));
  HR_CUDA(net->loss_part.ensure(sizeof(float) * 2 * (size_t)((Pc + 255) / 256 + 1)));
  HR_CUDA(net->w_part.ensure(sizeof(float) * (size_t)NZ_MAX * net->max_layer_w));
  HR_CUDA(net->b_part.ensure(sizeof(float) * (size_t)NZ_MAX * net->max_width));
  return HRKAN_OK;
}

enum PassKind { PASS_JET = 0, PASS_INTERIOR = 1, PASS_BOUNDARY = 2 };

struct PassArgs {
  PassKind kind;
  const float* pts;        // [P][D] device
  int64_t P;
  const float* forcing;    // interior Poisson (device) or null
  const float* g;          // boundary targets (device)
  float* u; float* du; float* d2u;   // PASS_JET outputs (device)
  float* grad;             // flat gradient (device)
  float* out_loss;         // device scalar slot
  float* out_flag;
  const hrkan_pde* pde;
  float inv_n;             // 1/N_int_global or 1/N_bi_global
  float* jet_out;          // PASS_JET of a generic jet spec: [P][C] output jet (device)
};

// Generic jet specs (jet_kernels.cuh)
enum JetSpecId { JSPEC_TAYLOR5 = 0, JSPEC_HESS2 = 1, JSPEC_HESS3 = 2 };

// Forward + (optional) loss/seeds + reverse over one point set, chunk by chunk.

// Arguments of the one-launch tiny-net step (tiny_kernels.cuh); device pointers.
struct TinyArgs {
  const hrkan_pde* pde;
  const float *interior, *forcing, *boundary, *g_boundary, *initial, *g_initial;
  int64_t Ni, Nb, N0;
  float inv_int, inv_bi;
  float* out;
};

// One scheduler per HR order m (pass_m<m>.cu).
#define HRKAN_DECLARE_DISPATCH(MM) \
  hrkan_status dispatch_pass_m##MM(hrkan_net* net, int nf, int ns, const PassArgs& a, cudaStream_t st); \
  hrkan_status tiny_step_m##MM(hrkan_net* net, const TinyArgs& t, cudaStream_t st); \
  hrkan_status dispatch_spec_m##MM(hrkan_net* net, int spec, const PassArgs& a, cudaStream_t st);
HRKAN_DECLARE_DISPATCH(2)
HRKAN_DECLARE_DISPATCH(3)
HRKAN_DECLARE_DISPATCH(4)
HRKAN_DECLARE_DISPATCH(5)
HRKAN_DECLARE_DISPATCH(6)
HRKAN_DECLARE_DISPATCH(7)
HRKAN_DECLARE_DISPATCH(8)

}  // namespace hrkan
