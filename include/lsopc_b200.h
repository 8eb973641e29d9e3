/*
 * lsopc_b200.h -- C ABI of the B200-native DSO level-set ILT hot path.
 *
 * The reference (`lsopc` 0.1.0, /root/reference/pkg/src/lsopc) is a Python
 * package whose "plugin interface" is its module-level function API; every
 * entry point below replaces one of those functions and cites it.  Plain
 * pointers and sizes only: arrays are row-major [y][x] (fields.py:3-4), real
 * fields float64, binary grids uint8, kernels complex128 interleaved (re, im).
 *
 * Pointer residency: arguments named *_dev are device pointers (caller-owned,
 * e.g. torch tensors); *_host are host pointers.  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Calls are asynchronous on `stream` unless
 * they return a host scalar.
 *
 * Errors: every call returns an lsopc_status; on failure
 * lsopc_last_error() gives a thread-local message.  The host mirror maps
 * LSOPC_EINVAL -> ValueError, LSOPC_EDEGENERATE -> DegenerateInputError,
 * LSOPC_ENUMERIC -> NumericalError (errors.py:4-13), LSOPC_ECUDA -> RuntimeError.
 */
#ifndef LSOPC_B200_H
#define LSOPC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LSOPC_OK = 0,
  LSOPC_EINVAL = 1,
  LSOPC_EDEGENERATE = 2,
  LSOPC_ENUMERIC = 3,
  LSOPC_ECUDA = 4
} lsopc_status;

typedef enum { LSOPC_FP32 = 0, LSOPC_FP64 = 1 } lsopc_precision;

typedef struct lsopc_plan lsopc_plan;    /* workspace for one (H, W, precision) */
typedef struct lsopc_kset lsopc_kset;    /* device spectra of one KernelSet     */
typedef struct lsopc_session lsopc_session; /* one optimize() run on device     */

const char* lsopc_last_error(void);
int lsopc_abi_version(void);

/* Workspace for H x W grids (powers of two, 4..8192; fields.py:1-6 contract,
 * SPEC.md:51).  precision: transforms in complex64 (FP32) or complex128.
 * FP64 takes sides up to 4096, plus 8192 x W with 256 <= W <= 1024 (the
 * split plan); LSOPC_EINVAL otherwise. */
int lsopc_plan_create(int H, int W, int precision, lsopc_plan** out);
int lsopc_plan_destroy(lsopc_plan* plan);

/* KernelSet.stacked_ffts (litho.py:71-82) + embed_kernel (fields.py:61-74):
 * spectra of n_k K x K kernels on the plan's grid, built once on device.
 * coeffs_host: n_k*K*K complex128 interleaved; weights_host: n_k float64. */
int lsopc_kset_create(lsopc_plan* plan, int n_k, int K, const double* coeffs_host,
                      const double* weights_host, void* stream, lsopc_kset** out);
int lsopc_kset_destroy(lsopc_kset* ks);
/* Download the set's spectra as complex128 n_k x [H][W] (KernelSet.stacked_ffts). */
int lsopc_kset_download(const lsopc_kset* ks, double* out_c128_dev, void* stream);

/* aerial_intensity (litho.py:114-126): out = max(dose * sum_k w_k |M (*) h_k|^2, 0) */
int lsopc_aerial_intensity(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev,
                           double dose, double* out_dev, void* stream);

/* print_corners (litho.py:141-154): nominal (focus, 1.0), outer (focus, 1.02),
 * inner (defocus, 0.98).  binarize != 0: outputs uint8 hard prints
 * (litho.py:129-131), else float64 sigmoid prints (litho.py:134-138). */
int lsopc_print_corners(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus,
                        const double* mask_dev, double i_th, double sigma_z, int binarize,
                        void* nominal_dev, void* inner_dev, void* outer_dev, void* stream);

/* _socs_gradient (optimizer.py:99-111):
 * out = 4 sigma_z dose Re sum_k w_k [((z - z_t) z (1 - z) conj(A_k)) (*) h_k(-.)] */
int lsopc_socs_gradient(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev,
                        const double* z_dev, const double* zt_dev, double sigma_z, double dose,
                        double* out_dev, void* stream);

/* convolve (fields.py:77-87) with the set's first kernel: circular
 * convolution, complex128 output [H][W] interleaved. */
int lsopc_convolve(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev, double* out_c128_dev,
                   void* stream);

/* geometry_gradient (levelset.py:109-119) and GeometryGradient.magnitude
 * (levelset.py:60-62).  Any output may be NULL. */
int lsopc_geometry_gradient(int H, int W, const double* phi_dev, double* gx, double* gy,
                            double* gxx, double* gyy, double* gxy, double* mag, void* stream);

/* curvature (levelset.py:126-139); m_dev may be NULL */
int lsopc_curvature(int H, int W, const double* phi_dev, const double* m_dev, double weight,
                    double* out_dev, void* stream);

/* tsdf_from_mask (levelset.py:86-101).  Returns LSOPC_EDEGENERATE on uniform masks. */
int lsopc_tsdf(int H, int W, const uint8_t* mask_dev, double d_upper, double d_lower,
               double* phi_dev, void* stream);

/* Elementwise operators on n values (a, b device arrays; see lsopc_ew_op). */
typedef enum {
  LSOPC_EW_MASK = 1,      /* out8 = a <= 0           mask_from_phi   levelset.py:104-106 */
  LSOPC_EW_HEAVISIDE = 2, /* out8 = a >= 0           heaviside       levelset.py:142-144 */
  LSOPC_EW_AXPBY = 3,     /* out = p0 a + p1 b       velocity        optimizer.py:132-134 */
  LSOPC_EW_SIGMOID = 4,   /* out = 1/(1+exp(-p0 (a - p1)))  resist_sigmoid litho.py:134-138 */
  LSOPC_EW_HARD = 5,      /* out8 = a >= p0          resist_hard     litho.py:129-131 */
  LSOPC_EW_NEG = 6,       /* out = -a                cg_direction restart optimizer.py:154-169 */
  LSOPC_EW_CG = 7,        /* out = -a + p0 b         cg_direction    optimizer.py:169 */
  LSOPC_EW_MOTION = 8,    /* out = -a * b            motion_term     optimizer.py:137-140 */
  LSOPC_EW_EVOLVE = 9,    /* out = clip(a + p0 b, p1, p2)  evolve_step levelset.py:154-166 */
  LSOPC_EW_AHF = 10,      /* out = (1 + (2/pi) atan(a/p0))/2  ahf    levelset.py:147-151 */
  LSOPC_EW_HYPOT = 11     /* out = hypot(a, b) (glibc-exact) GeometryGradient.magnitude levelset.py:60-62 */
} lsopc_ew_op;
int lsopc_elementwise(int op, size_t n, const double* a_dev, const double* b_dev, double p0,
                      double p1, double p2, double* out_dev, uint8_t* out8_dev, void* stream);

/* Deterministic reductions to a host scalar (fixed-order tree, no float atomics). */
typedef enum {
  LSOPC_RD_SUMSQDIFF = 1, /* sum (a-b)^2        ilt_loss / pvb_loss  optimizer.py:88-96 */
  LSOPC_RD_DOT = 2,       /* sum a b            cg_direction denom   optimizer.py:162     */
  LSOPC_RD_DOTDIFF = 3,   /* sum a (a-b)        cg_direction numer   optimizer.py:165     */
  LSOPC_RD_MAXABS = 4,    /* max |a|            cfl_timestep         optimizer.py:143-151 */
  LSOPC_RD_COUNTNEQ8 = 5, /* #(a8 != b8)        l2_error / pvband    metrics.py:39-52     */
  LSOPC_RD_NONFINITE = 6, /* n - (first index with a non-finite) or 0 (check_finite)      */
  LSOPC_RD_COUNTNEQ = 7   /* #(a != b) on float64 l2_error/pvband on non-uint8 grids       */
} lsopc_rd_op;
int lsopc_reduce(int op, size_t n, const double* a_dev, const double* b_dev, const uint8_t* a8_dev,
                 const uint8_t* b8_dev, double* out_host, void* stream);

/* OptConfig (optimizer.py:38-64) */
typedef struct {
  double alpha, beta, curvature_weight, sigma_z, i_th, eta, d_upper, d_lower;
  int max_iters;
  double stop_rel_tol;
  int stop_patience;
  int use_curvature;
  int cg_restart_every;
  /* 0: optimize's update phi + dt*(-v_total*|grad phi|) (optimizer.py:262-268);
   * 1: modulation_search's phi - (dt*v_total)*|grad phi| (optimizer.py:328-331).
   * The two orders round differently; each mode reproduces its caller. */
  int update_form;
  /* 1: skip the uniform-target check (a strip of a larger tile may be uniform;
   * the caller checks the whole tile, optimizer.py:197-201) */
  int skip_target_check;
  /* Opt-in extensions (not in the reference; 0 = the reference's behaviour):
   * grad_scheme 1: Godunov upwind |grad phi| in the update term instead of the
   * central one (levelset.py:60-62); reinit_every N > 0: after every N-th
   * completed iteration phi <- TSDF(mask_from_phi(phi)) (levelset.py:86-101),
   * whole-grid sessions only. */
  int grad_scheme;
  int reinit_every;
} lsopc_config;

typedef struct {
  int iters;          /* len(loss_history) */
  int l2;             /* metrics.py:39-44 on the best iterate's hard prints */
  int pvband;         /* metrics.py:47-52 */
  int nonfinite_iter; /* -1, or the iteration whose loss was non-finite (optimizer.py:240-241) */
} lsopc_result;

/* optimize (optimizer.py:204-284) minus shot counting: the full DSO loop on
 * device.  target_dev uint8 [H][W]; phi0_dev / mod_dev may be NULL (TSDF of
 * the target / all-ones gate).  Outputs: best_phi_dev (f64), final_mask_dev
 * (u8), history_host (max_iters x 7 f64: l_ilt, l_pvb, l_dso, dt, max_v,
 * max_step, max_grad_mag).  Synchronises `stream`. */
int lsopc_optimize(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus,
                   const uint8_t* target_dev, const double* phi0_dev, const double* mod_dev,
                   const lsopc_config* cfg, double* best_phi_dev, uint8_t* final_mask_dev,
                   double* history_host, lsopc_result* result, void* stream);

/* Split form of lsopc_optimize for pipelined / timed use: create, enqueue
 * iterations without host synchronisation, query, finish. */
int lsopc_session_create(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus,
                         const uint8_t* target_dev, const double* phi0_dev, const double* mod_dev,
                         const lsopc_config* cfg, void* stream, lsopc_session** out);
/* Enqueue up to n more iterations (bounded by max_iters); never blocks. */
int lsopc_session_enqueue(lsopc_session* s, int n);
/* Blocks until the enqueued work is done; *stopped = stop rule fired. */
int lsopc_session_poll(lsopc_session* s, int* stopped, int* iters_enqueued);
/* Final hard prints + metrics; writes outputs like lsopc_optimize. */
int lsopc_session_finish(lsopc_session* s, double* best_phi_dev, uint8_t* final_mask_dev,
                         double* history_host, lsopc_result* result);
int lsopc_session_destroy(lsopc_session* s);
/* Current (not best) phi of the session, f64 [H][W]; used by
 * modulation_search (optimizer.py:317-336), which scores the last iterate. */
int lsopc_session_phi(lsopc_session* s, double* phi_dev);
/* L_ilt, L_pvb and L_DSO = alpha L_ilt + beta L_pvb of the session's current
 * phi: _forward_losses(mask_from_phi(phi)) (optimizer.py:172-177), computed
 * on the device whether or not the loop has stopped (modulation_search's
 * candidate score, optimizer.py:334-336).  Synchronises the session stream;
 * any output pointer may be NULL. */
int lsopc_session_losses(lsopc_session* s, double* l_ilt, double* l_pvb, double* l_dso);
/* Number of kernel launches one DSO iteration enqueues (bench accounting). */
int lsopc_session_launches_per_iter(const lsopc_session* s);

/* DevelSet-Net front end -> DSO initial state in one pass (configs[3];
 * PAPER.md:553-635, boundary optimizer.py:215-228): phi0 = clip(phi_raw,
 * d_lower, d_upper) and m = AHF_epsilon(m_raw) = (1 + (2/pi) atan(m_raw/eps))/2
 * (levelset.py:147-151); float32 network outputs, float64 results. */
int lsopc_dsn_init(size_t n, const float* phi_raw_dev, const float* m_raw_dev, double d_lower, double d_upper,
                   double epsilon, double* phi0_dev, double* m_dev, void* stream);

/* Oversized tile split across ranks into full-height strips (BASELINE
 * configs[4]).  The session's grid is this rank's window: its
 * interior columns [ix0, ix1) plus halo columns refreshed from the
 * neighbouring ranks each iteration; [xlo, xhi) bounds the x-neighbours of
 * the phi stencil (replicate padding at the global tile edge).  After
 * set_tile the iteration is driven phase by phase: each phase leaves this
 * rank's partial scalars in lsopc_session_scalars() (8 doubles on the
 * device: [0..1] losses (sum), [2..3] Polak-Ribiere dots (sum), [4..5]
 * max |v_total|, max |grad phi| (max), [6] max step (max)), which the caller
 * combines across ranks before the next phase; after phase 4 the caller
 * refreshes the halo columns of lsopc_session_phi_ptr().  Forward phases
 * threshold phi directly, so only phi needs exchanging.
 * Phase 1 = phase 6 (stop rule, best iterate) then phase 5 (adjoint, dot
 * partials).  Several strips sharing one plan's work fields in one process
 * run 0, 5 per strip back to back (the adjoint reads only the forward's
 * fields, never the stop decision's outputs), combine losses and dots
 * together, then 6, 2, 3, 4 per strip. */
int lsopc_session_set_tile(lsopc_session* s, int ix0, int ix1, int xlo, int xhi);
/* The general strip window: interior [iy0, iy1) x [ix0, ix1), stencil
 * neighbours bounded by [ylo, yhi) x [xlo, xhi).  Full-width strips (rows
 * of the tile, iy-ranges) keep the long 8192-point axis on the rows, whose
 * transforms stream by TMA; set_tile is the full-height special case. */
int lsopc_session_set_window(lsopc_session* s, int ix0, int ix1, int xlo, int xhi, int iy0, int iy1, int ylo,
                             int yhi);
int lsopc_session_phase(lsopc_session* s, int phase);
double* lsopc_session_scalars(lsopc_session* s);
double* lsopc_session_phi_ptr(lsopc_session* s);
/* device pointer to the session's stop flag (int; non-zero once the stop rule fired) */
int* lsopc_session_state_flag(lsopc_session* s);

/* Measurement hook: run `reps` more iterations of the session, recording CUDA
 * events on the session stream at the pass boundaries, and write the mean
 * per-iteration milliseconds of each pass to ms_out[8]:
 * 0 mask FFT (2 launches), 1 F1 forward columns, 2 F2 forward rows + intensity,
 * 3 resist/loss/best (3 launches), 4 A1 adjoint rows, 5 A2 adjoint columns,
 * 6 A3 adjoint finish + CG dots, 7 level-set step (5 launches).  Synchronises. */
int lsopc_session_time_passes(lsopc_session* s, int reps, double* ms_out);

/* fracture / shot_count (metrics.py:55-108): greedy largest all-ones
 * rectangle (ties topmost, then leftmost), host code.  rects_host may be NULL;
 * returns the count via *count. */
int lsopc_fracture(int H, int W, const uint8_t* mask_host, int32_t* rects_host, size_t rects_cap,
                   size_t* count);

/* EXTENSION (no reference implementation; parity UNPINNED):
 * edge placement error of a printed image against its target, both uint8
 * DEVICE grids [H][W] (non-zero = lit).  Samples on the target's edges at a
 * lattice (horizontal edges at columns x = offset mod spacing, vertical edges
 * at rows y = offset mod spacing); EPE = signed displacement of the printed
 * edge along the outward normal, saturating at max_search; a violation when
 * |EPE| > threshold.  out_host[4] = samples, violations, sum |EPE|,
 * max |EPE|.  Synchronises `stream`. */
int lsopc_epe(int H, int W, const uint8_t* print_dev, const uint8_t* target_dev, int spacing, int offset,
              int threshold, int max_search, double* out_host, void* stream);

/* The same greedy fracture of a DEVICE mask (uint8 [H][W], non-zero = lit)
 * on the GPU: one thread-block cluster runs the whole greedy loop with the
 * lit bounding box's column heights in distributed shared memory; boxes too
 * large for it finish on the host algorithm above.  Rectangles (x, y, w, h)
 * go to host memory (rects_host may be NULL: count only).  Synchronises
 * `stream`. */
int lsopc_fracture_dev(int H, int W, const uint8_t* mask_dev, int32_t* rects_host, size_t rects_cap,
                       size_t* count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSOPC_B200_H */
