// C++ launchers of the spectral passes (internal.h) and the one-time kernel
// spectra build (K0).  The pass templates live in spectral.cuh.
#include "spectral.cuh"

namespace lsb {
namespace spec {
extern template void mask_fft_impl<float>(const Grid& g, const void* src, int kind, void* mhat, void* scratch, StopFlag stop,
                   cudaStream_t s);
extern template void f1_impl<float>(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template void f2_impl<float>(const Grid& g, const SpecSet* sets, int nsets, double2* a0_out, StopFlag stop, cudaStream_t s);
extern template void a1_impl<float>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template void a2_impl<float>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template int finish_impl<float>(const Grid& g, const void* V0, const void* V1, double scale, double* out, const double* vp,
                double* dots, StopFlag stop, cudaStream_t s, int ix0, int ix1, const LoopTail* tail, int iy0,
                int iy1);
extern template void mask_fft_impl<double>(const Grid& g, const void* src, int kind, void* mhat, void* scratch, StopFlag stop,
                   cudaStream_t s);
extern template void f1_impl<double>(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template void f2_impl<double>(const Grid& g, const SpecSet* sets, int nsets, double2* a0_out, StopFlag stop, cudaStream_t s);
extern template void a1_impl<double>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template void a2_impl<double>(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s);
extern template int finish_impl<double>(const Grid& g, const void* V0, const void* V1, double scale, double* out, const double* vp,
                double* dots, StopFlag stop, cudaStream_t s, int ix0, int ix1, const LoopTail* tail, int iy0,
                int iy1);
}  // namespace spec

using namespace spec;

namespace {
template <typename RC>
__global__ void k_embed(int K, int H, int W, const double2* __restrict__ coeffs, typename CT<RC>::C* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * K) return;
  int i = t / K, j = t % K;
  int y = ((i - K / 2) % H + H) % H;
  int x = ((j - K / 2) % W + W) % W;
  out[(size_t)y * W + x] = cmk((RC)coeffs[t].x, (RC)coeffs[t].y);
}

// K0 of a split plan (H = 8192): the direct separable DFT of the K x K taps in
// float64, G(i, v) = sum_j h(i, j) e^(-2 pi i v tc_j / W), then
// H(u, v) = sum_i G(i, v) e^(-2 pi i u tr_i / H), with tc_j = (j - K/2) mod W,
// tr_i = (i - K/2) mod H (fields.py:61-74 embedding) -- K multiply-adds per
// output, no 8192-point transform -- stored in the plan precision,
// column-tiled, rows in split order (u = 4 f2 + c at row c * H/4 + f2).
__global__ void k_dft_rows(int K, int W, int lgnmax, const double2* __restrict__ h, const double2* __restrict__ tw,
                           double2* G) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (v >= W) return;
  const int step = (1 << lgnmax) / W;
  double2 acc = make_double2(0.0, 0.0);
  for (int j = 0; j < K; ++j) {
    const int tc = ((j - K / 2) % W + W) % W;
    const double2 w = tw[(int)(((long long)v * tc) % W) * step];
    acc = acc + cmul(h[i * K + j], w);
  }
  G[(size_t)i * W + v] = acc;
}
template <typename C>
__global__ void k_dft_cols_split(int K, int H, int W, int lgT, int lgnmax, const double2* __restrict__ G,
                                 const double2* __restrict__ tw, C* out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x, u = blockIdx.y;
  if (v >= W) return;
  const int step = (1 << lgnmax) / H;
  double2 acc = make_double2(0.0, 0.0);
  for (int i = 0; i < K; ++i) {
    const int tr = ((i - K / 2) % H + H) % H;
    const double2 w = tw[(int)(((long long)u * tr) % H) * step];
    acc = acc + cmul(G[(size_t)i * W + v], w);
  }
  const int yd = (u & 3) * (H >> 2) + (u >> 2);
  out[(((size_t)(v >> lgT) * H + yd) << lgT) | (v & ((1 << lgT) - 1))] = cmk((decltype(C{}.x))acc.x,
                                                                           (decltype(C{}.x))acc.y);
}
}  // namespace

// ============================================================================

int finish_max_blocks() { return 148 * 2; }

void launch_mask_fft(const Grid& g, const uint8_t* mu8, const double* mf, const double* phi, void* mhat,
                     void* scratch, StopFlag stop, cudaStream_t s, bool cols) {
  const void* src = mu8 ? (const void*)mu8 : mf ? (const void*)mf : (const void*)phi;
  const int kind = mu8 ? SRC_U8 : mf ? SRC_F64 : SRC_PHI;
  void* out = cols ? mhat : nullptr;  // null: the row pass only
  if (g.prec == F64) mask_fft_impl<double>(g, src, kind, out, scratch, stop, s);
  else mask_fft_impl<float>(g, src, kind, out, scratch, stop, s);
}

void launch_f1(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s,
               const void* mtilde) {
  if (mtilde && use_tc_f1(g, sets, nsets)) {
    launch_f1_tc(g, mtilde, sets, nsets, stop, s);
    return;
  }
  if (g.prec == F64) f1_impl<double>(g, mhat, sets, nsets, stop, s);
  else f1_impl<float>(g, mhat, sets, nsets, stop, s);
}
void launch_f2(const Grid& g, const SpecSet* sets, int nsets, double* a0_c128, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) f2_impl<double>(g, sets, nsets, reinterpret_cast<double2*>(a0_c128), stop, s);
  else f2_impl<float>(g, sets, nsets, reinterpret_cast<double2*>(a0_c128), stop, s);
}
void launch_a1(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) a1_impl<double>(g, sets, nsets, stop, s);
  else a1_impl<float>(g, sets, nsets, stop, s);
}
void launch_a2(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) a2_impl<double>(g, sets, nsets, stop, s);
  else a2_impl<float>(g, sets, nsets, stop, s);
}
void launch_forward(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, double* a0_c128,
                    StopFlag stop, cudaStream_t s) {
  launch_f1(g, mhat, sets, nsets, stop, s);
  launch_f2(g, sets, nsets, a0_c128, stop, s);
}
void launch_adjoint(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  launch_a1(g, sets, nsets, stop, s);
  launch_a2(g, sets, nsets, stop, s);
}

int launch_adjoint_finish(const Grid& g, const void* V0, const void* V1, double scale, double* out,
                          const double* vp, double* dots, StopFlag stop, cudaStream_t s, int ix0, int ix1,
                          const LoopTail* tail, int iy0, int iy1) {
  if (g.prec == F64) return finish_impl<double>(g, V0, V1, scale, out, vp, dots, stop, s, ix0, ix1, tail, iy0, iy1);
  return finish_impl<float>(g, V0, V1, scale, out, vp, dots, stop, s, ix0, ix1, tail, iy0, iy1);
}

// K0: spectra, row pass then column pass, stored column-tiled in the plan's
// precision.  The transforms run in float64 (then round to complex64 for the
// FP32 tier) up to 4096-point sides; an FP32 plan with a larger side (the
// 8192^2 tile of configs[4]) transforms in float32, since one CTA holds at
// most a 4096-point complex128 sequence (relative error ~1e-7, far inside the
// FP32 tier's 1e-4).  scratch, scratch2: >= H*W*16 bytes each.
template <typename RC>
void spectra_impl(const Grid& g, int nk, int K, const double* coeffs_dev, void* spec, void* scratch, void* scratch2,
                  cudaStream_t s) {
  using CC = typename CT<RC>::C;
  Grid gc = g;
  gc.prec = sizeof(RC) == 8 ? F64 : F32;
  gc.tw = sizeof(RC) == 8 ? g.tw64 : g.tw;
  Shape<RC> sh = shape_of<RC>(gc);
  const size_t n = g.n();
  const int lgT_out = g.prec == F64 ? shape_of<double>(g).lgT : shape_of<float>(g).lgT;
  for (int k = 0; k < nk; ++k) {
    cudaMemsetAsync(scratch, 0, n * sizeof(CC), s);
    const int nt = K * K;
    k_embed<RC><<<(nt + 255) / 256, 256, 0, s>>>(K, g.H, g.W, reinterpret_cast<const double2*>(coeffs_dev) + (size_t)k * nt,
                                                static_cast<CC*>(scratch));
    RowsOp<RC, false> rr;
    rr.sh = sh;
    rr.in = static_cast<const CC*>(scratch);
    rr.Lin = sh.rm();
    rr.Lout = sh.ct();
    rr.out = static_cast<CC*>(scratch2);
    rr.tw = static_cast<const CC*>(gc.tw);
    rr.bufE = row_bufE(sh);
    rr.nitems = g.H >> sh.lgR;
    launch_op<RC>(rr, row_threads(sh), 0, nullptr, s);
    if (g.prec == F64) {
      ColsOp<RC, double, false> cc;
      cc.sh = sh;
      cc.in = static_cast<const CC*>(scratch2);
      cc.Lin = sh.ct();
      cc.Lout = Lay{g.H, lgT_out};
      cc.out = static_cast<double2*>(spec) + (size_t)k * n;
      cc.scale = (RC)1;
      cc.tw = static_cast<const CC*>(gc.tw);
      cc.bufE = col_bufE(sh);
      cc.nitems = g.W >> sh.lgS;
      launch_op<RC>(cc, col_threads(sh), 0, nullptr, s);
    } else {
      ColsOp<RC, float, false> cc;
      cc.sh = sh;
      cc.in = static_cast<const CC*>(scratch2);
      cc.Lin = sh.ct();
      cc.Lout = Lay{g.H, lgT_out};
      cc.out = static_cast<float2*>(spec) + (size_t)k * n;
      cc.scale = (RC)1;
      cc.tw = static_cast<const CC*>(gc.tw);
      cc.bufE = col_bufE(sh);
      cc.nitems = g.W >> sh.lgS;
      launch_op<RC>(cc, col_threads(sh), 0, nullptr, s);
    }
  }
}

void launch_kernel_spectra(const Grid& g, int nk, int K, const double* coeffs_dev, void* spec, void* scratch,
                           void* scratch2, cudaStream_t s) {
  if (g.vsplit) {
    double2* G = static_cast<double2*>(scratch);
    const double2* tw = static_cast<const double2*>(g.tw64);
    const int lgT = g.prec == F64 ? shape_of<double>(g).lgT : shape_of<float>(g).lgT;
    for (int k = 0; k < nk; ++k) {
      const double2* h = reinterpret_cast<const double2*>(coeffs_dev) + (size_t)k * K * K;
      k_dft_rows<<<dim3((g.W + 127) / 128, K), 128, 0, s>>>(K, g.W, g.lgnmax, h, tw, G);
      if (g.prec == F64)
        k_dft_cols_split<double2><<<dim3((g.W + 127) / 128, g.H), 128, 0, s>>>(
            K, g.H, g.W, lgT, g.lgnmax, G, tw, static_cast<double2*>(spec) + (size_t)k * g.n());
      else
        k_dft_cols_split<float2><<<dim3((g.W + 127) / 128, g.H), 128, 0, s>>>(
            K, g.H, g.W, lgT, g.lgnmax, G, tw, static_cast<float2*>(spec) + (size_t)k * g.n());
    }
    return;
  }
  if (g.prec == F32 && std::max(g.H, g.W) > 4096) spectra_impl<float>(g, nk, K, coeffs_dev, spec, scratch, scratch2, s);
  else spectra_impl<double>(g, nk, K, coeffs_dev, spec, scratch, scratch2, s);
}

// spectrum field (plan precision, column-tiled) -> complex128 row-major
void launch_spec_to_c128(const Grid& g, const void* field, double* out, cudaStream_t s) {
  const int lgq = g.vsplit ? g.lgH - 2 : -1;  // split plans store rows in split order
  if (g.prec == F64) {
    Lay L{g.H, shape_of<double>(g).lgT};
    k_ct_to_c128<double><<<148 * 4, 256, 0, s>>>(g.n(), L, g.W, static_cast<const double2*>(field),
                                                   reinterpret_cast<double2*>(out), lgq);
  } else {
    Lay L{g.H, shape_of<float>(g).lgT};
    k_ct_to_c128<float><<<148 * 4, 256, 0, s>>>(g.n(), L, g.W, static_cast<const float2*>(field),
                                                  reinterpret_cast<double2*>(out), lgq);
  }
}

}  // namespace lsb
