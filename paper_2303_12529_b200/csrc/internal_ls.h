// Level-set / loop-control launchers and the device-resident loop state.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace lsb {

// Device-resident state of the DSO loop (optimizer.py:230-269).  Every kernel
// of an iteration reads `stopped` first, so the host can enqueue iterations
// without waiting for the stop rule.
struct DevState {
  double best, l_ilt, l_pvb, l_dso;
  double beta;
  double vmax, gmax, dt;
  int stopped, improved, use_beta, streak, nhist, nonfinite_it;
  int it;  // index of the iteration in flight (advanced by the update's control kernel)
  // hard-print L2 / PVBand counts (metrics.py:39-52) of the best iterate,
  // recorded by the forward that found it: the result's metrics without a
  // final forward pass (optimizer.py:271-277 recomputes the same prints)
  double best_l2, best_pvb;
  int have_counts;
  unsigned ticket[4];  // last-block tickets of the fused control tails (control.cuh), zero between launches
};

// Window of a strip of an oversized tile run on one rank (window
// coordinates): [iy0, iy1) x [ix0, ix1) is the interior this rank owns
// (losses, dots, maxima, updates), [ylo, yhi) x [xlo, xhi) bounds the
// neighbours of the phi stencil (replicate padding at the global tile edge,
// halo data elsewhere).  Strips are full-width (rows) or full-height
// (columns); the row fields default to the whole grid (kAll is clamped to H).
constexpr int kAll = 1 << 30;
struct Tile {
  int ix0, ix1, xlo, xhi;
  int iy0 = 0, iy1 = kAll, ylo = 0, yhi = kAll;
};
inline Tile full_tile(int W) { return Tile{0, W, 0, W}; }

struct LoopCfg {
  double alpha, beta, stop_rel_tol;
  int stop_patience;
};

// Fused control tail of a producing kernel (control.cuh): its last block runs
// the control body on the partials the kernel just wrote.  st == nullptr: none.
struct LoopTail {
  DevState* st;
  double* hist;
  LoopCfg c;
  double eta;
  int restart_every;
};

enum EwOp { EW_MASK = 1, EW_HEAVISIDE, EW_AXPBY, EW_SIGMOID, EW_HARD, EW_NEG, EW_CG, EW_MOTION, EW_EVOLVE, EW_AHF, EW_HYPOT };
enum RdOp { RD_SUMSQDIFF = 1, RD_DOT, RD_DOTDIFF, RD_MAXABS, RD_COUNTNEQ8, RD_NONFINITE, RD_COUNTNEQ };

int ls_blocks();
void launch_geometry(int H, int W, const double* phi, double* gx, double* gy, double* gxx, double* gyy,
                     double* gxy, double* mag, cudaStream_t s);
void launch_curvature(int H, int W, const double* phi, const double* m, double weight, double* out,
                      cudaStream_t s);
// tail (nullable): run the CFL control (after_velocity) / the history record
// (after_update) in the kernel's last block instead of a separate launch
void launch_ls_velocity(int H, int W, const double* phi, const double* v, const double* dprev, const double* m,
                        double weight, int use_curv, DevState* st, double* d, double* u, double* gm,
                        double* partials, Tile t, cudaStream_t s, const LoopTail* tail = nullptr,
                        int upwind = 0);
void launch_ls_update(int H, int W, double* phi, const double* u, const double* gm, double lo, double hi,
                      DevState* st, uint8_t* mask, double* partials, Tile t, cudaStream_t s,
                      const LoopTail* tail = nullptr);
void launch_dsn_init(size_t n, const float* phi_raw, const float* m_raw, double lo, double hi, double eps,
                     double* phi0, double* m, cudaStream_t s);
// fixed-order reduction of nb blocks of nv partials (sum or max) into out[0..nv)
void launch_reduce_partials(const double* part, int nb, int nv, int is_max, double* out, cudaStream_t s);
void launch_copy_best(size_t n, const double* phi, double* best, const DevState* st, cudaStream_t s);
void launch_after_forward(const double* part, int nb, LoopCfg c, DevState* st, double* hist, cudaStream_t s);
// restart_every: Polak-Ribiere restart period (optimizer.py:253); iteration 0 always restarts
void launch_after_grad(const double* dots, int nb, int restart_every, DevState* st, cudaStream_t s);
void launch_after_velocity(const double* part, int nb, double eta, DevState* st, double* hist, cudaStream_t s);
void launch_after_update(const double* part, int nb, DevState* st, double* hist, cudaStream_t s);
void launch_elementwise(int op, size_t n, const double* a, const double* b, double p0, double p1, double p2,
                        double* out, uint8_t* out8, cudaStream_t s);
// out: device scalar.  W > 0 restricts RD_COUNTNEQ8 to columns [ix0, ix1) x rows [iy0, iy1) of rows of width W.
void launch_reduce(int op, size_t n, const double* a, const double* b, const uint8_t* a8, const uint8_t* b8,
                   double* partials, double* out, cudaStream_t s, int W = 0, int ix0 = 0, int ix1 = 0,
                   int iy0 = 0, int iy1 = kAll);

// p[i] = p[i] != 0 (uint8, in place; 16-byte aligned p)
void launch_binarize_u8(size_t n, uint8_t* p, cudaStream_t s);

// exact EDT -> truncated signed distance (levelset.py:86-101)
// skip (nullable, device): every kernel returns at entry when *skip != 0
void launch_tsdf(int H, int W, const uint8_t* mask, double d_upper, double d_lower, double* phi,
                 int* scratch_i32, double* scratch_f64, cudaStream_t s, const int* skip = nullptr);
// Opt-in periodic reinitialisation of the DSO loop (extension): after the
// update of iteration it, *skip = 0 iff the loop runs, (it + 1) % every == 0
// and the mask (lit count *lit of n) is not uniform; phi is then replaced by
// the exact TSDF of its own mask.
void launch_reinit_gate(const DevState* st, const double* lit, double n, int every, int* skip, cudaStream_t s);
size_t tsdf_scratch_i32(int H, int W);
size_t tsdf_scratch_f64(int H, int W);

}  // namespace lsb
