// Internal launcher declarations shared between the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace lsb {

enum Prec { F32 = 0, F64 = 1 };

// ---- FFT geometry for one plan ------------------------------------------------
struct Grid {
  int H, W, lgH, lgW;
  int prec;             // Prec
  const void* tw;       // twiddle table exp(-2 pi i j / nmax), j < nmax, element C
  const void* tw64;     // the same table in double precision (spectra builds)
  int lgnmax;           // log2 table length
  // Tall-grid split (H = 8192): each column's transform runs as four
  // 2048-point transforms on the decimated "planes" (frequency row 4 f2 + c
  // -> plane c row f2, stored at row c * 2048 + f2), the column passes on the
  // virtual 2048 x 4W grid those planes form in memory, and the radix-4
  // combine across the planes folded into the row passes (spectral.cuh).
  int vsplit = 0;
  // F1 as a tap contraction on the tensor cores (f1_tc.cu; fp32 tier)
  int tcf1 = 0;
  size_t n() const { return (size_t)H * W; }
  size_t csize() const { return prec == F64 ? 16 : 8; }
  size_t rsize() const { return prec == F64 ? 8 : 4; }
};

// Optional device flag: when non-null and *stop != 0 every CTA exits at once
// (the device-side stop rule of the optimisation loop).
using StopFlag = const int*;

inline int ilog2i(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// One SOCS kernel set as seen by the spectral passes (spectral.cu).  All
// complex fields are column-tiled (engine.cuh) in the plan's precision.
struct SpecSet {
  int nk;
  const double* w;   // host weights (sigma_k), nk
  const void* spec;  // nk spectra
  void* T;           // nk column-tiled work fields: T_k after F1, U_k after A1
  void* A;           // nk row-major fields A_k (F2 -> A1)
  void* I;           // real intensity sum_k w_k |A_k|^2, row-major (element R)
  const void* gate;  // real gate, row-major (element R)
  void* V;           // complex adjoint accumulator (column-tiled)
  // kernel groups (small grids): per-group partials of I and V, and the
  // tickets of the last-arriving group item (null: no groups)
  void* Ipart;       // 8 groups x 2 sets x H*W elements R
  void* Vpart;       // 8 groups x 2 sets x H*W complex
  unsigned* tick;    // 2 passes x 2 sets x max(H, W) tickets, zero between launches
  // tensor-core F1 (f1_tc.cu): the taps' row DFT G_k(i, v) / W, [W][K][nk]
  // complex64 (null: this set runs the FFT F1), and the kernel side K
  const void* G;
  int K;
};

// K0: spectra of nk K x K kernels (float64 transform, stored in plan precision)
// coeffs_dev: nk x K x K interleaved complex128; scratch, scratch2: >= H*W*16 bytes
void launch_kernel_spectra(const Grid& g, int nk, int K, const double* coeffs_dev, void* spec,
                           void* scratch, void* scratch2, cudaStream_t s);
// one spectrum (plan precision, column-tiled) -> complex128 row-major
void launch_spec_to_c128(const Grid& g, const void* field, double* out, cudaStream_t s);

// M^ = FFT2(mask); exactly one of mask_u8 / mask_f64 / phi (mask = phi <= 0) is non-null.
// scratch >= H*W complex elements.
// cols = false: the row pass only (M~ in scratch, for the tensor-core F1)
void launch_mask_fft(const Grid& g, const uint8_t* mask_u8, const double* mask_f64, const double* phi,
                     void* mhat, void* scratch, StopFlag stop, cudaStream_t s, bool cols = true);

// forward of nsets (1 or 2) sets: T_k = IFFT_y(M^ H_k)/(HW), I = sum_k w_k |IFFT_x T_k|^2.
// a0_c128 (nullable): the first set's first field A_0 as complex128 row-major.
void launch_forward(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, double* a0_c128,
                    StopFlag stop, cudaStream_t s);

// the two halves of launch_forward / launch_adjoint (per-pass timing).
// launch_f1 runs the tensor-core F1 on mtilde (the mask's row transform, the
// mask pass's scratch) when use_tc_f1(), else the FFT F1 on mhat.
void launch_f1(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s,
               const void* mtilde = nullptr);

// tensor-core F1 (f1_tc.cu)
bool tcf1_plan_ok(int H, int W, int prec, int vsplit);
bool tcf1_kset_ok(int nk, int K);
bool use_tc_f1(const Grid& g, const SpecSet* sets, int nsets);
void launch_tap_rows(const Grid& g, int nk, int K, const double* coeffs_dev, void* G, cudaStream_t s);
void launch_f1_tc(const Grid& g, const void* mtilde, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
void launch_f2(const Grid& g, const SpecSet* sets, int nsets, double* a0_c128, StopFlag stop, cudaStream_t s);
void launch_a1(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
void launch_a2(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);

// adjoint of nsets sets: U_k = FFT_x(gate IFFT_x T_k) (in place),
// V = IFFT_y(sum_k w_k conj(H_k) FFT_y U_k)
void launch_adjoint(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);

// out = scale * Re IFFT_x(V0 [+ V1]) (f64 row-major); with v_prev, per-CTA CG dot
// partials dots[blk*2 + {0,1}] = {sum v (v - vp), sum vp^2}.  Returns the
// number of partial blocks written (0 without v_prev).
struct LoopTail;  // internal_ls.h
// tail (nullable): the Polak-Ribiere control (after_grad) in the last CTA
int launch_adjoint_finish(const Grid& g, const void* V0, const void* V1, double scale, double* out,
                          const double* v_prev, double* dots, StopFlag stop, cudaStream_t s, int ix0 = 0,
                          int ix1 = 0,  // dots over columns [ix0, ix1) (0, 0: all)
                          const LoopTail* tail = nullptr, int iy0 = 0, int iy1 = 1 << 30);  // ... rows [iy0, iy1)
int finish_max_blocks();

// ---- elementwise / reductions ---------------------------------------------------
int reduce_blocks();   // number of partial slots used by grid-stride reducers

struct ResistParams {
  double i_th, sigma_z, alpha, beta;
};
// Z corners from intensities (R), partials[blk*4+{0..3}] = L_ilt, L_pvb and the
// hard-print L2 / PVB counts (with a target), gates wf/wd
// (R, nullable), Z outputs (f64, nullable), hard prints (u8, nullable).
void launch_resist(const Grid& g, const void* If, const void* Id, const uint8_t* target_u8,
                   const double* target_f64, ResistParams p, void* wf, void* wd,
                   double* z_nom, double* z_in, double* z_out, uint8_t* h_nom,
                   uint8_t* h_in, uint8_t* h_out, double* partials, StopFlag stop,
                   cudaStream_t s, int ix0 = 0, int ix1 = 0,  // losses over columns [ix0, ix1) (0, 0: all)
                   const LoopTail* tail = nullptr,   // after_forward fused into the DSO loop form
                   int iy0 = 0, int iy1 = 1 << 30);   // ... and rows [iy0, iy1)
// single-corner intensity output: out = max(dose * I, 0) (f64)
void launch_scale_intensity(const Grid& g, const void* I, double dose, double* out, cudaStream_t s);
// gate for a user-supplied print: w = scale * (z - zt) z (1 - z)   (element R)
void launch_gate(const Grid& g, const double* z, const double* zt, double scale, void* w,
                 cudaStream_t s);

}  // namespace lsb
