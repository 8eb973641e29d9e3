// SOCS forward model and its adjoint on the shared-memory FFT engine.
//
// Replaces (reference, /root/reference/pkg/src/lsopc):
//   KernelSet.stacked_ffts + embed_kernel      litho.py:71-82, fields.py:61-74   (K0)
//   aerial_intensity / print_corners           litho.py:114-154                  (K1, K2)
//   resist_sigmoid / resist_hard, losses       litho.py:129-138, optimizer.py:88-96 (K3)
//   _socs_gradient / ilt_ / pvb_gradient       optimizer.py:99-129               (K4)
//
// Frequency-domain layout is natural [fy][fx].  A 2-D transform is a ROWS pass
// (length W, along x) and a COLS pass (length H, along y); every pointwise
// operation that precedes or follows a transform is fused into the pass's
// load/store functor.  The adjoint uses conj(t) = IFFT2(FFT2(gate A) conj(H))
// (equal real part to the reference's IFFT2(FFT2(gate conj A) H(-f))), so the
// forward and adjoint read the same spectrum at the same frequency.
#include "common.cuh"
#include "fft.cuh"
#include "internal.h"

#include <algorithm>
#include <stdexcept>

namespace lsb {

namespace {

template <typename R> constexpr int elems_per_cta() { return sizeof(R) == 4 ? 8192 : 4096; }

template <bool ROWS> struct Pos {
  int W = 0, nb = 0, tile = 0;
  LS_D size_t pos(int seq, int idx) const {
    if constexpr (ROWS) return (size_t)(tile * nb + seq) * W + idx;
    else return (size_t)idx * W + (size_t)(tile * nb + seq);
  }
  LS_D void finish(double*) {}
};

// plain copy / precision conversion
template <typename RI, typename RO, bool ROWS> struct FCopy : Pos<ROWS> {
  using CI = typename CT<RI>::C;
  using CO = typename CT<RO>::C;
  const CI* x;
  CO* y;
  LS_D CI load(int s, int i) const { return x[this->pos(s, i)]; }
  LS_D void store(int s, int i, CI v) { y[this->pos(s, i)] = cmk((RO)v.x, (RO)v.y); }
};

// mask -> complex (threshold already applied by the producer of mask_u8)
template <typename R> struct FMaskRows : Pos<true> {
  using C = typename CT<R>::C;
  const uint8_t* mu8;
  const double* mf;
  C* y;
  LS_D C load(int s, int i) const {
    size_t p = pos(s, i);
    R m = mu8 ? (R)mu8[p] : (R)mf[p];
    return cmk(m, (R)0);
  }
  LS_D void store(int s, int i, C v) { y[pos(s, i)] = v; }
};

// forward COLS: (M^ * H_k * scale) -> inverse along y
template <typename R> struct FFwdCol : Pos<false> {
  using C = typename CT<R>::C;
  const C* mhat;
  const C* spec;
  R scale;
  C* y;
  LS_D C load(int s, int i) const {
    size_t p = pos(s, i);
    return cmul(mhat[p], __ldg(&spec[p])) * scale;
  }
  LS_D void store(int s, int i, C v) { y[pos(s, i)] = v; }
};

// forward ROWS: inverse along x -> A_k (stored) and I += w |A_k|^2
template <typename R> struct FFwdRow : Pos<true> {
  using C = typename CT<R>::C;
  const C* x;
  C* a;
  R* I;
  R w;
  int first;
  LS_D C load(int s, int i) const { return x[pos(s, i)]; }
  LS_D void store(int s, int i, C v) {
    size_t p = pos(s, i);
    if (a) a[p] = v;
    R e = w * (v.x * v.x + v.y * v.y);
    I[p] = first ? e : I[p] + e;
  }
};

// adjoint ROWS: gate * A_k -> forward along x
template <typename R> struct FAdjRow : Pos<true> {
  using C = typename CT<R>::C;
  const C* a;
  const R* gate;
  C* y;
  LS_D C load(int s, int i) const {
    size_t p = pos(s, i);
    return a[p] * gate[p];
  }
  LS_D void store(int s, int i, C v) { y[pos(s, i)] = v; }
};

// adjoint COLS: forward along y -> G += w conj(H_k) * v
template <typename R> struct FAdjCol : Pos<false> {
  using C = typename CT<R>::C;
  const C* x;
  const C* spec;
  R w;
  C* G;
  int first;
  LS_D C load(int s, int i) const { return x[pos(s, i)]; }
  LS_D void store(int s, int i, C v) {
    size_t p = pos(s, i);
    C t = cmulc(v, __ldg(&spec[p])) * w;
    G[p] = first ? t : G[p] + t;
  }
};

// final ROWS of the adjoint: inverse along x, keep scale * Re, CG dot partials
template <typename R> struct FFinish : Pos<true> {
  using C = typename CT<R>::C;
  const C* x;
  double scale;
  double* out;
  const double* vp;
  double* dots;
  double acc[2] = {0.0, 0.0};
  LS_D C load(int s, int i) const { return x[pos(s, i)]; }
  LS_D void store(int s, int i, C v) {
    size_t p = pos(s, i);
    double val = scale * (double)v.x;
    out[p] = val;
    if (vp) {
      double q = vp[p];
      acc[0] += val * (val - q);
      acc[1] += q * q;
    }
  }
  LS_D void finish(double* red) {
    if (!vp) return;
    __syncthreads();
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
      dots[2 * tile + 0] = acc[0];
      dots[2 * tile + 1] = acc[1];
    }
  }
};

template <typename R, bool SEQ_FAST, bool INV, class F>
__global__ void __launch_bounds__(512, 2) k_fft(F f, fft::Geo geo, const typename CT<R>::C* __restrict__ tw,
                                             StopFlag stop) {
  using C = typename CT<R>::C;
  if (stop && *stop) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* sm = reinterpret_cast<C*>(smraw);
  f.tile = blockIdx.x;
  fft::run<SEQ_FAST, INV>(geo, sm, tw, f);
  f.finish(reinterpret_cast<double*>(smraw));
}

inline int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// Launch one pass.  ROWS: sequences are the H rows (length W); else the W
// columns (length H).  Returns the grid size (number of CTAs).
template <typename R, bool ROWS, bool INV, class F>
int launch_pass(const Grid& g, F f, const void* tw, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const int lgn = ROWS ? g.lgW : g.lgH;
  const int nseq = ROWS ? g.H : g.W;
  const int n = 1 << lgn;
  const int E = std::max(elems_per_cta<R>(), n);
  const int nb = std::min(E / n, nseq);
  const int threads = nb * n / fft::P_of<C>();
  if (threads < 1) throw std::runtime_error("grid too small for the FFT engine (need H*W >= 16)");
  fft::Geo geo{lgn, nb, ilog2(nb), g.lgnmax - lgn};
  const size_t smem = std::max(fft::smem_bytes<C>(n, nb), (size_t)(64 * sizeof(double)));
  auto kern = k_fft<R, !ROWS, INV, F>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_set = true;
  }
  f.W = g.W;
  f.nb = nb;
  const int grid = nseq / nb;
  kern<<<grid, threads, smem, s>>>(f, geo, static_cast<const C*>(tw), stop);
  return grid;
}

__global__ void k_embed(int K, int H, int W, const double2* __restrict__ coeffs, double2* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * K) return;
  int i = t / K, j = t % K;
  int y = ((i - K / 2) % H + H) % H;
  int x = ((j - K / 2) % W + W) % W;
  out[(size_t)y * W + x] = coeffs[t];
}

template <typename R>
void forward_set_impl(const Grid& g, int nk, const void* mhat, const void* spec, const double* wts,
                      void* A, void* I, void* scratch, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const size_t n = g.n();
  const R inv_n = (R)(1.0 / (double)n);
  for (int k = 0; k < nk; ++k) {
    FFwdCol<R> fc;
    fc.mhat = static_cast<const C*>(mhat);
    fc.spec = static_cast<const C*>(spec) + (size_t)k * n;
    fc.scale = inv_n;
    fc.y = static_cast<C*>(scratch);
    launch_pass<R, false, true>(g, fc, g.tw, stop, s);
    FFwdRow<R> fr;
    fr.x = static_cast<const C*>(scratch);
    fr.a = A ? static_cast<C*>(A) + (size_t)k * n : nullptr;
    fr.I = static_cast<R*>(I);
    fr.w = (R)wts[k];
    fr.first = (k == 0);
    launch_pass<R, true, true>(g, fr, g.tw, stop, s);
  }
}

template <typename R>
void adjoint_set_impl(const Grid& g, int nk, const void* A, const void* gate, const void* spec,
                      const double* wts, void* G, bool first, void* scratch, StopFlag stop,
                      cudaStream_t s) {
  using C = typename CT<R>::C;
  const size_t n = g.n();
  for (int k = 0; k < nk; ++k) {
    FAdjRow<R> fr;
    fr.a = static_cast<const C*>(A) + (size_t)k * n;
    fr.gate = static_cast<const R*>(gate);
    fr.y = static_cast<C*>(scratch);
    launch_pass<R, true, false>(g, fr, g.tw, stop, s);
    FAdjCol<R> fc;
    fc.x = static_cast<const C*>(scratch);
    fc.spec = static_cast<const C*>(spec) + (size_t)k * n;
    fc.w = (R)wts[k];
    fc.G = static_cast<C*>(G);
    fc.first = first && (k == 0);
    launch_pass<R, false, false>(g, fc, g.tw, stop, s);
  }
}

template <typename R>
int adjoint_finish_impl(const Grid& g, const void* G, double scale, double* out, const double* vp,
                        double* dots, void* scratch, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  FCopy<R, R, false> fc;
  fc.x = static_cast<const C*>(G);
  fc.y = static_cast<C*>(scratch);
  launch_pass<R, false, true>(g, fc, g.tw, stop, s);
  FFinish<R> ff;
  ff.x = static_cast<const C*>(scratch);
  ff.scale = scale;
  ff.out = out;
  ff.vp = vp;
  ff.dots = dots;
  int grid = launch_pass<R, true, true>(g, ff, g.tw, stop, s);
  return vp ? grid : 0;
}

template <typename R>
void mask_fft_impl(const Grid& g, const uint8_t* mu8, const double* mf, void* mhat, void* scratch,
                   StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  FMaskRows<R> fm;
  fm.mu8 = mu8;
  fm.mf = mf;
  fm.y = static_cast<C*>(scratch);
  launch_pass<R, true, false>(g, fm, g.tw, stop, s);
  FCopy<R, R, false> fc;
  fc.x = static_cast<const C*>(scratch);
  fc.y = static_cast<C*>(mhat);
  launch_pass<R, false, false>(g, fc, g.tw, stop, s);
}

// ---- resist / losses / gates -------------------------------------------------

constexpr int kRedBlocks = 148 * 4;
constexpr int kRedThreads = 256;

LS_D double sigmoid(double i, double i_th, double sz) { return 1.0 / (1.0 + exp(-sz * (i - i_th))); }

template <typename R>
__global__ void __launch_bounds__(kRedThreads)
k_resist(size_t n, const R* __restrict__ If, const R* __restrict__ Id, const uint8_t* __restrict__ tu8,
         const double* __restrict__ tf, ResistParams p, R* wf, R* wd, double* z_nom, double* z_in,
         double* z_out, uint8_t* h_nom, uint8_t* h_in, uint8_t* h_out, double* partials,
         StopFlag stop) {
  __shared__ double red[64];
  if (stop && *stop) return;
  double acc[2] = {0.0, 0.0};
  const bool have_t = tu8 || tf;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    // litho.py:125-126: I = max(dose * sum, 0); corners: litho.py:147-149
    double sf = (double)If[i];
    double i_nom = fmax(1.0 * sf, 0.0);
    double i_out = fmax(1.02 * sf, 0.0);
    double i_in = Id ? fmax(0.98 * (double)Id[i], 0.0) : 0.0;
    if (h_nom) {  // litho.py:129-131 (inclusive threshold)
      h_nom[i] = i_nom >= p.i_th;
      h_out[i] = i_out >= p.i_th;
      if (h_in) h_in[i] = i_in >= p.i_th;
    }
    if (!z_nom && !wf && !partials) continue;
    double zn = sigmoid(i_nom, p.i_th, p.sigma_z);
    double zo = sigmoid(i_out, p.i_th, p.sigma_z);
    double zi = sigmoid(i_in, p.i_th, p.sigma_z);
    if (z_nom) {
      z_nom[i] = zn;
      z_out[i] = zo;
      if (z_in) z_in[i] = zi;
    }
    if (have_t) {
      double zt = tu8 ? (double)tu8[i] : tf[i];
      double dn = zn - zt, di = zi - zt, dout = zo - zt;
      acc[0] += dn * dn;               // optimizer.py:88-90
      acc[1] += di * di + dout * dout;  // optimizer.py:93-96
      if (wf) {
        // optimizer.py:109 gate, 114-134 doses and alpha/beta folded per kernel set
        double gn = dn * zn * (1.0 - zn);
        double go = dout * zo * (1.0 - zo);
        double gi = di * zi * (1.0 - zi);
        wf[i] = (R)(p.alpha * gn + p.beta * 1.02 * go);
        wd[i] = (R)(p.beta * 0.98 * gi);
      }
    }
  }
  if (partials) {
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
      partials[2 * blockIdx.x] = acc[0];
      partials[2 * blockIdx.x + 1] = acc[1];
    }
  }
}

template <typename R>
__global__ void k_scale_intensity(size_t n, const R* __restrict__ I, double dose, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = fmax(dose * (double)I[i], 0.0);
}

template <typename R>
__global__ void k_gate(size_t n, const double* __restrict__ z, const double* __restrict__ zt, double scale,
                       R* w) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double zz = z[i];
    w[i] = (R)(scale * ((zz - zt[i]) * zz * (1.0 - zz)));
  }
}

template <typename R>
__global__ void k_to_c128(size_t n, const typename CT<R>::C* __restrict__ a, double2* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = make_double2((double)a[i].x, (double)a[i].y);
}

}  // namespace

void launch_to_c128(const Grid& g, const void* A, double* out, cudaStream_t s) {
  if (g.prec == F64) k_to_c128<double><<<kRedBlocks, 256, 0, s>>>(g.n(), static_cast<const double2*>(A), reinterpret_cast<double2*>(out));
  else k_to_c128<float><<<kRedBlocks, 256, 0, s>>>(g.n(), static_cast<const float2*>(A), reinterpret_cast<double2*>(out));
}

int reduce_blocks() { return kRedBlocks; }

namespace {
template <typename R>
void bench_pass_impl(const Grid& g, int which, const void* spec, void* mhat, void* A, void* I, void* gate,
                     void* G, void* scratch, cudaStream_t s) {
  using C = typename CT<R>::C;
  switch (which) {
    case 0: {
      FFwdCol<R> f;
      f.mhat = static_cast<const C*>(mhat);
      f.spec = static_cast<const C*>(spec);
      f.scale = (R)1;
      f.y = static_cast<C*>(scratch);
      launch_pass<R, false, true>(g, f, g.tw, nullptr, s);
    } break;
    case 1: {
      FFwdRow<R> f;
      f.x = static_cast<const C*>(scratch);
      f.a = static_cast<C*>(A);
      f.I = static_cast<R*>(I);
      f.w = (R)1;
      f.first = 0;
      launch_pass<R, true, true>(g, f, g.tw, nullptr, s);
    } break;
    case 2: {
      FAdjRow<R> f;
      f.a = static_cast<const C*>(A);
      f.gate = static_cast<const R*>(gate);
      f.y = static_cast<C*>(scratch);
      launch_pass<R, true, false>(g, f, g.tw, nullptr, s);
    } break;
    default: {
      FAdjCol<R> f;
      f.x = static_cast<const C*>(scratch);
      f.spec = static_cast<const C*>(spec);
      f.w = (R)1;
      f.G = static_cast<C*>(G);
      f.first = 0;
      launch_pass<R, false, false>(g, f, g.tw, nullptr, s);
    } break;
  }
}
}  // namespace

void launch_bench_pass(const Grid& g, int which, const void* spec, void* mhat, void* A, void* I, void* gate,
                       void* G, void* scratch, cudaStream_t s) {
  if (g.prec == F64) bench_pass_impl<double>(g, which, spec, mhat, A, I, gate, G, scratch, s);
  else bench_pass_impl<float>(g, which, spec, mhat, A, I, gate, G, scratch, s);
}

void launch_kernel_spectra(const Grid& g, int nk, int K, const double* coeffs_dev, void* spec,
                           void* scratch, cudaStream_t s) {
  const size_t n = g.n();
  Grid g64 = g;
  g64.prec = F64;
  g64.tw = g.tw64;
  for (int k = 0; k < nk; ++k) {
    cudaMemsetAsync(scratch, 0, n * sizeof(double2), s);
    int nt = K * K;
    k_embed<<<(nt + 255) / 256, 256, 0, s>>>(K, g.H, g.W, reinterpret_cast<const double2*>(coeffs_dev) + (size_t)k * nt,
                                            static_cast<double2*>(scratch));
    FCopy<double, double, true> fr;
    fr.x = static_cast<const double2*>(scratch);
    fr.y = static_cast<double2*>(scratch);
    launch_pass<double, true, false>(g64, fr, g.tw64, nullptr, s);
    if (g.prec == F64) {
      FCopy<double, double, false> fc;
      fc.x = static_cast<const double2*>(scratch);
      fc.y = static_cast<double2*>(spec) + (size_t)k * n;
      launch_pass<double, false, false>(g64, fc, g.tw64, nullptr, s);
    } else {
      FCopy<double, float, false> fc;
      fc.x = static_cast<const double2*>(scratch);
      fc.y = static_cast<float2*>(spec) + (size_t)k * n;
      launch_pass<double, false, false>(g64, fc, g.tw64, nullptr, s);
    }
  }
}

void launch_mask_fft(const Grid& g, const uint8_t* mu8, const double* mf, void* mhat, void* scratch,
                     StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) mask_fft_impl<double>(g, mu8, mf, mhat, scratch, stop, s);
  else mask_fft_impl<float>(g, mu8, mf, mhat, scratch, stop, s);
}

void launch_forward_set(const Grid& g, int nk, const void* mhat, const void* spec, const double* wts,
                        void* A, void* I, void* scratch, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) forward_set_impl<double>(g, nk, mhat, spec, wts, A, I, scratch, stop, s);
  else forward_set_impl<float>(g, nk, mhat, spec, wts, A, I, scratch, stop, s);
}

void launch_adjoint_set(const Grid& g, int nk, const void* A, const void* gate, const void* spec,
                        const double* wts, void* G, bool first, void* scratch, StopFlag stop,
                        cudaStream_t s) {
  if (g.prec == F64) adjoint_set_impl<double>(g, nk, A, gate, spec, wts, G, first, scratch, stop, s);
  else adjoint_set_impl<float>(g, nk, A, gate, spec, wts, G, first, scratch, stop, s);
}

int launch_adjoint_finish(const Grid& g, const void* G, double scale, double* out, const double* vp,
                          double* dots, void* scratch, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) return adjoint_finish_impl<double>(g, G, scale, out, vp, dots, scratch, stop, s);
  return adjoint_finish_impl<float>(g, G, scale, out, vp, dots, scratch, stop, s);
}

void launch_resist(const Grid& g, const void* If, const void* Id, const uint8_t* tu8, const double* tf,
                   ResistParams p, void* wf, void* wd, double* z_nom, double* z_in, double* z_out,
                   uint8_t* h_nom, uint8_t* h_in, uint8_t* h_out, double* partials, StopFlag stop,
                   cudaStream_t s) {
  if (g.prec == F64)
    k_resist<double><<<kRedBlocks, kRedThreads, 0, s>>>(
        g.n(), static_cast<const double*>(If), static_cast<const double*>(Id), tu8, tf, p,
        static_cast<double*>(wf), static_cast<double*>(wd), z_nom, z_in, z_out, h_nom, h_in, h_out, partials, stop);
  else
    k_resist<float><<<kRedBlocks, kRedThreads, 0, s>>>(
        g.n(), static_cast<const float*>(If), static_cast<const float*>(Id), tu8, tf, p,
        static_cast<float*>(wf), static_cast<float*>(wd), z_nom, z_in, z_out, h_nom, h_in, h_out, partials, stop);
}

void launch_scale_intensity(const Grid& g, const void* I, double dose, double* out, cudaStream_t s) {
  if (g.prec == F64) k_scale_intensity<double><<<kRedBlocks, 256, 0, s>>>(g.n(), static_cast<const double*>(I), dose, out);
  else k_scale_intensity<float><<<kRedBlocks, 256, 0, s>>>(g.n(), static_cast<const float*>(I), dose, out);
}

void launch_gate(const Grid& g, const double* z, const double* zt, double scale, void* w, cudaStream_t s) {
  if (g.prec == F64) k_gate<double><<<kRedBlocks, 256, 0, s>>>(g.n(), z, zt, scale, static_cast<double*>(w));
  else k_gate<float><<<kRedBlocks, 256, 0, s>>>(g.n(), z, zt, scale, static_cast<float*>(w));
}

}  // namespace lsb
