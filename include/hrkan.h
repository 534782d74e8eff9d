/*
 * hrkan.h -- C ABI of libhrkan.so, the B200 (sm_100a) hot path of HRKAN physics-informed training
 * (Higher-order-ReLU KANs, arXiv 2409.14248).
 *
 * Citations: P:n = PAPER.md line n (/root/reference, Sec./Eq. given), SURVEY §8 = the builder's
 * hot-path table in SURVEY.md, whose readings of silent/garbled points are listed in DESIGN.md.
 *
 * What the library computes:
 *   basis      v_{m,n}(x) = ReLU(e_n - x)^m ReLU(x - s_n)^m c_m, c_m = (2/(e_n-s_n))^{2m}
 *              (Eq. 2) with s_n = lo + (n-k)h, e_n = s_n + (k+1)h, h = (hi-lo)/G,
 *              n = 0..G+k-1 ("same support as the B-splines").
 *   layer      y_j = b_j + sum_{i,n} W[j,i,n] v_n(x_i)   (KAN layer as a matrix product),
 *              evaluated on a second-order jet (value, d/dxi_a, diagonal d^2/dxi_a^2).
 *   loss       L = alpha L_pde + L_bi (Eq. 4, Eq. 8) with the Poisson residual
 *              r = sum_a u_aa - f, f = -D pi^2 prod_a sin(pi xi_a) (Eq. 3) or the viscous
 *              Burgers residual r = u_t + adv u u_x - visc u_xx (Eq. 5; Eq. 7 is adv=1/4,
 *              visc=nu/16), L_pde = (1/N_int) sum r^2, L_bi = (1/N_bi) sum (u - g)^2 pooled over
 *              boundary and initial points.
 *   gradient   dL/dtheta by a hand-written reverse pass through the jet.
 *   optimiser  bias-corrected Adam ("Adam optimizer").
 *
 * Conventions for every call:
 *   - All tensors are fp32, row-major, contiguous.  Pointers may be DEVICE pointers (the fast
 *     path) or HOST pointers (pinned or pageable): host buffers are detected with
 *     cudaPointerGetAttributes and staged through library-owned device buffers with
 *     cudaMemcpyAsync on `stream`; a host `out`/`u`/... is written back asynchronously, so the
 *     caller must synchronise `stream` before reading it.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *     asynchronous and stream-ordered; the library never synchronises except in create/free
 *     and when it must read back a host-staged result.  Calls on one net must be issued on one
 *     stream (the net owns one workspace); distinct nets may run concurrently.
 *   - The library never calls NCCL: the data-parallel allreduce of the `out` buffer of
 *     hrkan_pinn_loss_grad is the caller's (torch.distributed over NCCL).
 *   - Errors are returned as hrkan_status; hrkan_last_error() gives a thread-local message.
 *     The library never aborts the process.
 *
 * Flat parameter layout (params, gradient, Adam m and v):
 *   for l = 0..L-1:  W_l[O_l][I_l][G+k] row-major, then b_l[O_l];  I_l = widths[l], O_l = widths[l+1].
 *   The bias acts on the value channel only (SURVEY §8(c) reading 3).
 */
#ifndef HRKAN_H_
#define HRKAN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hrkan_net* hrkan_net_t;

typedef enum {
  HRKAN_OK = 0,
  HRKAN_EINVAL = 1,        /* invalid argument (see each call)                              */
  HRKAN_EUNSUPPORTED = 2,  /* device is not sm_100 (B200) or the config exceeds a kernel limit */
  HRKAN_ENOMEM = 3,        /* device allocation failed                                       */
  HRKAN_ECUDA = 4,         /* a CUDA launch / runtime error (message from cudaGetErrorString) */
  HRKAN_ENONFINITE = 5     /* reserved: non-finite values are reported through out[] flag     */
} hrkan_status;

typedef enum {
  HRKAN_POISSON = 0,   /* r = sum_a u_aa - f (Eq. 3)                                           */
  HRKAN_BURGERS = 1,   /* r = u_t + adv u u_x - visc u_xx (Eq. 5; Eq. 7), D = 2 (x, t)     */
  HRKAN_KAWAHARA = 2,  /* r = u_t + adv u u_x + disp3 u_xxx - disp5 u_xxxxx, D = 2 (x, t): a PDE with a
                          fifth derivative ("u_xxxxx ... pick m to be larger, like 6"); m >= 3
                          (v^(5) is non-zero for 2m >= 5 and continuous for m >= 6)                   */
  HRKAN_ANISO = 3      /* r = sum_{a<=b} aniso[q(a,b)] u_ab - f with mixed second derivatives (full
                          Hessian); q runs over the upper triangle row-major:
                          D=2 (xx, xy, yy), D=3 (xx, xy, xz, yy, yz, zz); forcing f required          */
} hrkan_pde_kind;

typedef struct {
  int32_t kind;   /* hrkan_pde_kind                                                         */
  float alpha;    /* weight of L_pde (paper: 0.05, P:142 / P:239)                            */
  float adv;      /* Burgers: r = u_t + adv*u*u_x - visc*u_xx  (coordinates (x, t))         */
  float visc;     /*   BASELINE.json: adv = 1, visc = 0.01/pi;  paper Eq. 7: 1/4, 0.001/16   */
  float disp3;    /* Kawahara: coefficient of u_xxx                                         */
  float disp5;    /* Kawahara: coefficient of -u_xxxxx                                      */
  float aniso[6]; /* HRKAN_ANISO: coefficients of u_ab over the upper triangle (a <= b)     */
} hrkan_pde;

/* Jet kinds of hrkan_forward_jet_ex (higher-order and mixed jets). */
typedef enum {
  HRKAN_JET_TAYLOR5 = 1,  /* D = 2 (x, t): C = 7 channels [u, u_x, u_xx, u_xxx, u_xxxx, u_xxxxx, u_t]        */
  HRKAN_JET_HESSIAN = 2   /* D = 2 or 3: C = 1 + D + D(D+1)/2 channels [u, u_a (a < D), u_ab (a <= b, upper
                             triangle row-major)] -- the full Hessian, mixed terms included                 */
} hrkan_jet_kind;

/* Create a network.  widths[0..n_widths-1] (host) = [D, hidden..., 1]; basis G (grid
 * intervals), k (B-spline order giving G+k supports), m (HR order, Eq. 2), [grid_lo, grid_hi]
 * the basis grid range.  Parameters are initialised on `device` with
 * W ~ N(0, 1/(I_l (G+k))) (variance), b = 0 from a counter-based Philox4x32-10 stream keyed by
 * `seed` (SURVEY §8(c) reading 5).  Adam state is zeroed (t = 0).
 * Execution detail that never shows at this boundary: with at least two hidden layers, every hidden width
 * in (32, 256] and G+k >= 8, hidden widths other than 64 / 128 / 256 are zero-padded internally to the next
 * of those so that every hidden->hidden contraction (P:45 / P:87) runs on the tensor-core kernels; padded
 * neurons have zero weights and bias, emit an all-zero jet and receive a zero adjoint, and every vector
 * exchanged through this API (parameters, gradient, Adam state) keeps the caller's compact layout for the
 * widths given here.  Environment HRKAN_PAD_WIDTHS=0 (read at create) disables the padding.
 * EINVAL: n_widths < 2, any width < 1, widths[0] not in {1,2,3}, widths[n-1] != 1, G < 1, k < 1,
 *         m < 2 or m > 8, grid_lo >= grid_hi or non-finite, out == NULL.
 * EUNSUPPORTED: the device is not compute capability 10.0 (sm_100a code only).
 * Ownership: the returned net owns its device memory; release it with hrkan_free. */
hrkan_status hrkan_create(const int32_t* widths, int32_t n_widths, int32_t G, int32_t k, int32_t m,
                          float grid_lo, float grid_hi, uint64_t seed, int32_t device,
                          hrkan_net_t* out);

/* The widths the kernels of a net created with these arguments run on (host-only query, no device
 * needed): `out[0..n_widths-1]` (host) receives `widths` with the hidden entries zero-padded as
 * hrkan_create's "execution detail" describes (equal to `widths` when no padding applies or
 * HRKAN_PAD_WIDTHS=0).  The public vectors never use these widths; the query exists so that callers
 * and tests can see which nets take the tensor-core path.  EINVAL: NULL pointers, n_widths < 2,
 * a width < 1, G < 1 or k < 1. */
hrkan_status hrkan_execution_widths(const int32_t* widths, int32_t n_widths, int32_t G, int32_t k, int32_t* out);

/* Number of parameters = sum_l O_l*I_l*(G+k) + O_l.  Returns -1 for a NULL net. */
int64_t hrkan_num_params(hrkan_net_t net);

/* Copy the flat parameter vector out / in (device or host pointer of num_params floats).
 * set_params also invalidates the kernels' derived weight copies. */
hrkan_status hrkan_get_params(hrkan_net_t net, float* dst, void* stream);
hrkan_status hrkan_set_params(hrkan_net_t net, const float* src, void* stream);

/* Re-initialise the parameters (same rule as hrkan_create) and zero the Adam state. */
hrkan_status hrkan_init_params(hrkan_net_t net, uint64_t seed, void* stream);

/* Evaluate the network jet at P points pts[P, D]:  u[P] = u(xi),  du[P, D] = du/dxi_a,
 * d2u[P, D] = d^2u/dxi_a^2 (diagonal of the Hessian).  Any of u/du/d2u may be NULL (not
 * written).  P = 0 is a no-op.  EINVAL: P < 0, pts == NULL with P > 0. */
hrkan_status hrkan_forward_jet(hrkan_net_t net, const float* pts, int64_t P,
                               float* u, float* du, float* d2u, void* stream);

/* Higher-order / mixed jet of the network at P points pts[P, D]: jet[P][C] with the
 * channels of `kind` (see hrkan_jet_kind), all exact derivatives of the network function u(xi).  The
 * layers compose the jet channel by channel: Faa di Bruno's formula with the partial Bell polynomials for
 * the x-orders (TAYLOR5), the second-order chain rule z_ab = phi'' h_a h_b + phi' h_ab (HESSIAN).
 * EINVAL: P < 0, NULL pointers with P > 0, unknown kind, TAYLOR5 with D != 2 or m < 3, HESSIAN with D = 1.
 * EUNSUPPORTED: a width above 256.  P = 0 is a no-op. */
hrkan_status hrkan_forward_jet_ex(hrkan_net_t net, int32_t kind, const float* pts, int64_t P, float* jet, void* stream);

/* One PINN loss + gradient evaluation.
 *   interior[Ni, D]  collocation points; forcing[Ni] = f (Poisson) or NULL for the built-in
 *                    f = -D pi^2 prod sin(pi xi_a); ignored for Burgers and Kawahara; required for ANISO.
 *   boundary[Nb, D], g_boundary[Nb]  boundary points and targets;
 *   initial[N0, D],  g_initial[N0]   initial-condition points and targets (may be NULL if N0=0).
 *   Ni_global, Nbi_global: the normalisers N_int and N_bi = Nb + N0 of the WHOLE job.  Pass the
 *   local counts when unsharded; in data parallel every rank passes the global counts so that the
 *   sum over ranks of `out` is the global loss and gradient.
 *   out[num_params + 4]: out[0..np-1] = dL/dtheta (OVERWRITTEN, flat layout), out[np] = alpha*L_pde
 *   part, out[np+1] = L_bi part, out[np+2] = non-finite flag (count of non-finite residuals /
 *   boundary errors; summed by an allreduce so any rank's flag shows), out[np+3] = 0 (pad).
 * Burgers and Kawahara require D = 2 (coordinates (x, t)); Kawahara m >= 3; ANISO D = 2 or 3 and a forcing.
 * The interior pass of KAWAHARA / ANISO runs the generic jet engine (band-limited FFMA kernels on the
 * TAYLOR5 / HESSIAN jets); boundary and initial points always run the value-only kernels.
 * EINVAL: negative counts, NULL pointer with non-zero count, Ni_global < Ni, Nbi_global < Nb+N0,
 *         Burgers/Kawahara with D != 2, Kawahara with m < 3, ANISO with D = 1 or no forcing, unknown pde
 *         kind, out == NULL. */
hrkan_status hrkan_pinn_loss_grad(hrkan_net_t net, const hrkan_pde* pde,
                                  const float* interior, const float* forcing, int64_t Ni,
                                  const float* boundary, const float* g_boundary, int64_t Nb,
                                  const float* initial, const float* g_initial, int64_t N0,
                                  int64_t Ni_global, int64_t Nbi_global,
                                  float* out, void* stream);

/* One bias-corrected Adam step on the net's parameters with gradient grad[num_params]
 * (t += 1 first; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; theta -= lr mhat/(sqrt(vhat)+eps),
 * mhat = m/(1-b1^t), vhat = v/(1-b2^t); "Adam optimizer").  The step count t lives in
 * device memory and is advanced by the kernel itself, so a caller's CUDA-graph capture of a whole
 * training step (loss+grad, allreduce, Adam) replays with a live bias correction.  hrkan_init_params
 * resets t to 0.  EINVAL: grad == NULL, lr/eps not finite, beta outside [0,1). */
hrkan_status hrkan_adam_step(hrkan_net_t net, const float* grad, float lr, float beta1, float beta2,
                             float eps, void* stream);

/* Upper bound on collocation points processed per internal chunk (bounds the saved-jet
 * workspace, SURVEY §7 hard part (f)).  0 = default.  EINVAL: chunk < 0. */
hrkan_status hrkan_set_chunk_points(hrkan_net_t net, int64_t chunk);

/* Select the engine (a change re-derives every kernel-private weight copy before the next call): 0 = auto (one-launch fused kernel for tiny nets -- every width <= 8, <= 4 layers,
 * <= 2048 parameters, k <= 7; its last block reduces the gradient -- else tcgen05 tensor cores where a
 * hidden layer is wide (O in {64,128,256}, I % 8 == 0, G+k >= 8) and SIMT FFMA elsewhere), 1 = force the
 * layered SIMT FFMA kernels, 2 = force tcgen05 where supported (layered).
 * EINVAL: unknown mode. */
hrkan_status hrkan_set_engine(hrkan_net_t net, int32_t mode);

/* CUDA-graph replay of hrkan_pinn_loss_grad (enable != 0).  When enabled, and the call uses only
 * device buffers on a non-legacy stream that is not already being captured, and per-launch profiling
 * is off: the first call with a given argument signature (all pointers, counts, pde fields, stream,
 * chunk size, engine) runs eagerly, the second captures the whole call into a CUDA graph (weight
 * re-tiling included) and later calls replay it with one cudaGraphLaunch -- the launch-latency
 * bound small configs (C1, C2) become one graph launch per step.  Results are bitwise identical to
 * eager calls.  Changing any argument re-captures, and so does any growth of the library's workspace
 * (e.g. an hrkan_forward_jet on more points than the training chunk between two steps): the graph's
 * baked-in workspace pointers are never replayed after a reallocation.  A caller's own stream capture (e.g. of a whole
 * training step with the NCCL allreduce) simply records the eager launches.  EINVAL: net == NULL. */
hrkan_status hrkan_set_graph_mode(hrkan_net_t net, int32_t enable);

/* Number of kernels the library launched on this net since creation (for bench accounting). */
int64_t hrkan_launch_count(hrkan_net_t net);

/* Kernel classes timed by the profiling hooks below. */
typedef enum {
  HRKAN_K_FWD_FIRST = 0, HRKAN_K_FWD_HIDDEN = 1, HRKAN_K_FWD_LAST = 2, HRKAN_K_LOSS = 3,
  HRKAN_K_WGRAD_FIRST = 4, HRKAN_K_WGRAD_HIDDEN = 5, HRKAN_K_WGRAD_LAST = 6,
  HRKAN_K_DGRAD_HIDDEN = 7, HRKAN_K_DGRAD_LAST = 8, HRKAN_K_REDUCE = 9, HRKAN_K_ADAM = 10,
  HRKAN_K_OTHER = 11, HRKAN_K_FUSED_STEP = 12 /* one-launch tiny-net loss+grad (all layers) */,
  HRKAN_K_NUM_CLASSES = 13
} hrkan_kernel_class;

/* Device-time profiling: while enabled, every launch is bracketed by CUDA events recorded on the
 * launching stream.  hrkan_profile_read synchronises those events, writes per-class total
 * milliseconds ms[HRKAN_K_NUM_CLASSES] and launch counts n[HRKAN_K_NUM_CLASSES] (host arrays,
 * either may be NULL), and resets the accumulators.  EINVAL: net == NULL. */
hrkan_status hrkan_profile_enable(hrkan_net_t net, int32_t enable);
hrkan_status hrkan_profile_read(hrkan_net_t net, double* ms, int64_t* n);

/* Free the net and all its device memory (synchronises its device).  NULL is a no-op. */
void hrkan_free(hrkan_net_t net);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* hrkan_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HRKAN_H_ */
