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
  size_t n() const { return (size_t)H * W; }
  size_t csize() const { return prec == F64 ? 16 : 8; }
  size_t rsize() const { return prec == F64 ? 8 : 4; }
};

// Optional device flag: when non-null and *stop != 0 every CTA exits at once
// (the device-side stop rule of the optimisation loop).
using StopFlag = const int*;

// spectrum of one kernel set: nk x [H][W] complex (element C of the grid)
// coeffs_dev: nk x K x K interleaved complex128; scratch: >= H*W*16 bytes
void launch_kernel_spectra(const Grid& g, int nk, int K, const double* coeffs_dev,
                           void* spec, void* scratch, cudaStream_t s);

// M^ = FFT2(mask) ; mask is u8 (mask_u8 != null) or f64
void launch_mask_fft(const Grid& g, const uint8_t* mask_u8, const double* mask_f64,
                     void* mhat, void* scratch, StopFlag stop, cudaStream_t s);

// forward for one kernel set: for each k, A_k = IFFT2(M^ H_k); I = sum_k w_k |A_k|^2
// A (nullable) receives nk fields; I is element R.
void launch_forward_set(const Grid& g, int nk, const void* mhat, const void* spec,
                        const double* weights_host, void* A, void* I, void* scratch,
                        StopFlag stop, cudaStream_t s);

// adjoint for one kernel set, accumulated into G (first==true overwrites):
// G += sum_k w_k conj(H_k) FFT2(gate * A_k)
void launch_adjoint_set(const Grid& g, int nk, const void* A, const void* gate,
                        const void* spec, const double* weights_host, void* G, bool first,
                        void* scratch, StopFlag stop, cudaStream_t s);

// out = scale * Re IFFT2_unnormalised(G)  (f64 out); optional CG dot partials
// with v_prev: dots[blk*2 + {0,1}] = {sum v (v - vp), sum vp^2} over the block.
// Returns the number of dot partial blocks written (0 when v_prev is null).
int launch_adjoint_finish(const Grid& g, const void* G, double scale, double* out,
                          const double* v_prev, double* dots, void* scratch,
                          StopFlag stop, cudaStream_t s);

// ---- elementwise / reductions ---------------------------------------------------
int reduce_blocks();   // number of partial slots used by grid-stride reducers

struct ResistParams {
  double i_th, sigma_z, alpha, beta;
};
// Z corners from intensities (R), losses into partials[blk*2+{0,1}], gates wf/wd
// (R, nullable), Z outputs (f64, nullable), hard prints (u8, nullable).
void launch_resist(const Grid& g, const void* If, const void* Id, const uint8_t* target_u8,
                   const double* target_f64, ResistParams p, void* wf, void* wd,
                   double* z_nom, double* z_in, double* z_out, uint8_t* h_nom,
                   uint8_t* h_in, uint8_t* h_out, double* partials, StopFlag stop,
                   cudaStream_t s);
// single-corner intensity output: out = max(dose * I, 0) (f64)
void launch_scale_intensity(const Grid& g, const void* I, double dose, double* out, cudaStream_t s);
// gate for a user-supplied print: w = scale * (z - zt) z (1 - z)   (element R)
void launch_gate(const Grid& g, const double* z, const double* zt, double scale, void* w,
                 cudaStream_t s);

// copy the first field of A (element C) to complex128
void launch_to_c128(const Grid& g, const void* A, double* out, cudaStream_t s);

// one launch of a single spectral pass for measurement:
// 0 forward COLS, 1 forward ROWS, 2 adjoint ROWS, 3 adjoint COLS
void launch_bench_pass(const Grid& g, int which, const void* spec, void* mhat, void* A, void* I, void* gate,
                       void* G, void* scratch, cudaStream_t s);

}  // namespace lsb
