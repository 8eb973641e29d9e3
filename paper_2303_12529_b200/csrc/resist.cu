// Resist model, losses and adjoint gates (pointwise, grid-stride).
//
// Replaces (reference, /root/reference/pkg/src/lsopc):
//   resist_sigmoid / resist_hard               litho.py:129-138
//   corner doses (nominal / outer / inner)     litho.py:98-100,147-149
//   ilt_loss / pvb_loss                        optimizer.py:88-96
//   the adjoint gate (Z - Z_t) Z (1 - Z)       optimizer.py:109, 114-134
#include <stdexcept>

#include "common.cuh"
#include "control.cuh"
#include "internal.h"
#include "internal_ls.h"

namespace lsb {

namespace {

// ---- resist / losses / gates -------------------------------------------------

constexpr int kRedBlocks = 148 * 4;
constexpr int kRedThreads = 256;

LS_D double sigmoid(double i, double i_th, double sz) { return 1.0 / (1.0 + exp(-sz * (i - i_th))); }

template <typename R>
__global__ void __launch_bounds__(kRedThreads)
k_resist(size_t n, const R* __restrict__ If, const R* __restrict__ Id, const uint8_t* __restrict__ tu8,
         const double* __restrict__ tf, ResistParams p, R* wf, R* wd, double* z_nom, double* z_in,
         double* z_out, uint8_t* h_nom, uint8_t* h_in, uint8_t* h_out, double* partials,
         StopFlag stop, int W, int ix0, int ix1, int iy0, int iy1) {
  __shared__ double red[128];
  if (stop && *stop) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const bool have_t = tu8 || tf;
  const RowSplit rs = row_split(W);
  const bool whole = ix0 <= 0 && ix1 >= W && iy0 <= 0 && iy1 >= (int)(n / (size_t)W);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    // litho.py:125-126: I = max(dose * sum, 0); corners: litho.py:147-149
    double sf = (double)If[i];
    double i_nom = nmax(1.0 * sf, 0.0);
    double i_out = nmax(1.02 * sf, 0.0);
    double i_in = Id ? nmax(0.98 * (double)Id[i], 0.0) : 0.0;
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
      const int x = whole ? ix0 : (int)col_of(rs, i), y = whole ? iy0 : (int)row_of(rs, i);
      if (x >= ix0 && x < ix1 && y >= iy0 && y < iy1) {  // strip interior (the whole grid by default)
        acc[0] += dn * dn;               // optimizer.py:88-90
        acc[1] += di * di + dout * dout;  // optimizer.py:93-96
        // hard prints (litho.py:129-131): L2 vs the target, PVB inner vs outer (metrics.py:39-52)
        acc[2] += ((i_nom >= p.i_th) != (zt != 0.0)) ? 1.0 : 0.0;
        acc[3] += ((i_in >= p.i_th) != (i_out >= p.i_th)) ? 1.0 : 0.0;
      }
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
    block_sum<4>(acc, red);
    if (threadIdx.x == 0)
      for (int j = 0; j < 4; ++j) partials[4 * blockIdx.x + j] = acc[j];
  }
}

// The DSO loop's form of k_resist (losses + gates, no Z / print outputs),
// four consecutive pixels per thread with 16 B loads and stores: the
// pointwise pass is latency-bound unless each thread keeps several vector
// loads in flight.  Arithmetic per pixel is exactly k_resist's.
LS_D void ld4(const float* p, size_t i, float (&o)[4]) {
  const float4 t = *reinterpret_cast<const float4*>(p + i);
  o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
}
LS_D void ld4(const double* p, size_t i, double (&o)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p + i), b = *reinterpret_cast<const double2*>(p + i + 2);
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
LS_D void st4(float* p, size_t i, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p + i) = make_float4(v[0], v[1], v[2], v[3]);
}
LS_D void st4(double* p, size_t i, const double (&v)[4]) {
  *reinterpret_cast<double2*>(p + i) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + i + 2) = make_double2(v[2], v[3]);
}

template <typename R>
__global__ void __launch_bounds__(kRedThreads)
k_resist_loop(size_t n4, const R* __restrict__ If, const R* __restrict__ Id, const uint8_t* __restrict__ tu8,
              const double* __restrict__ tf, ResistParams p, R* wf, R* wd, double* partials, StopFlag stop, int W,
              int ix0, int ix1, int iy0, int iy1, LoopTail tail) {
  __shared__ double red[128];
  if (stop && *stop) return;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const RowSplit rs = row_split(W);
  const bool whole = ix0 <= 0 && ix1 >= W && iy0 <= 0 && iy1 >= (int)(4 * n4 / (size_t)W);
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < n4; g += (size_t)gridDim.x * blockDim.x) {
    const size_t i = 4 * g;
    R sf[4], sd[4] = {(R)0, (R)0, (R)0, (R)0};
    double zt[4];
    ld4(If, i, sf);
    if (Id) ld4(Id, i, sd);
    if (tu8) {  // binary targets: a select, not an int->float conversion
      const uchar4 t = *reinterpret_cast<const uchar4*>(tu8 + i);
      const unsigned char tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) zt[e] = (double)tv[e];
    } else {
      ld4(tf, i, zt);
    }
    const int x0 = whole ? ix0 : (int)col_of(rs, i);
    const bool row_in = whole || ((int)row_of(rs, i) >= iy0 && (int)row_of(rs, i) < iy1);
    R gf[4], gd[4];
    // float64 sigmoid and gates in both tiers: the loop's losses agree with the
    // API path (print_corners / ilt_loss) on the same intensities
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double i_nom = nmax(1.0 * (double)sf[e], 0.0);
      const double i_out = nmax(1.02 * (double)sf[e], 0.0);
      const double i_in = Id ? nmax(0.98 * (double)sd[e], 0.0) : 0.0;
      const double zn = sigmoid(i_nom, p.i_th, p.sigma_z), zo = sigmoid(i_out, p.i_th, p.sigma_z),
                   zi = sigmoid(i_in, p.i_th, p.sigma_z);
      const double dn = zn - zt[e], di = zi - zt[e], dout = zo - zt[e];
      if (whole || (row_in && x0 + e >= ix0 && x0 + e < ix1)) {
        acc[0] += dn * dn;
        acc[1] += di * di + dout * dout;
        acc[2] += ((i_nom >= p.i_th) != (zt[e] != 0.0)) ? 1.0 : 0.0;
        acc[3] += ((i_in >= p.i_th) != (i_out >= p.i_th)) ? 1.0 : 0.0;
      }
      gf[e] = (R)(p.alpha * (dn * zn * (1.0 - zn)) + p.beta * 1.02 * (dout * zo * (1.0 - zo)));
      gd[e] = (R)(p.beta * 0.98 * (di * zi * (1.0 - zi)));
    }
    if (wf) {
      st4(wf, i, gf);
      st4(wd, i, gd);
    }
  }
  block_sum<4>(acc, red);
  if (threadIdx.x == 0)
    for (int j = 0; j < 4; ++j) partials[4 * blockIdx.x + j] = acc[j];
  if (tail.st && last_block(&tail.st->ticket[0], red)) {
    after_forward_body(partials, gridDim.x, tail.c, tail.st, tail.hist, red);
    release_ticket(&tail.st->ticket[0]);
  }
}

template <typename R>
__global__ void k_scale_intensity(size_t n, const R* __restrict__ I, double dose, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = nmax(dose * (double)I[i], 0.0);
}

template <typename R>
__global__ void k_gate(size_t n, const double* __restrict__ z, const double* __restrict__ zt, double scale,
                       R* w) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double zz = z[i];
    w[i] = (R)(scale * ((zz - zt[i]) * zz * (1.0 - zz)));
  }
}

}  // namespace

int reduce_blocks() { return kRedBlocks; }

void launch_resist(const Grid& g, const void* If, const void* Id, const uint8_t* tu8, const double* tf,
                   ResistParams p, void* wf, void* wd, double* z_nom, double* z_in, double* z_out,
                   uint8_t* h_nom, uint8_t* h_in, uint8_t* h_out, double* partials, StopFlag stop,
                   cudaStream_t s, int ix0, int ix1, const LoopTail* tail, int iy0, int iy1) {
  if (ix1 <= 0) ix1 = g.W;
  if (iy1 > g.H) iy1 = g.H;
  const LoopTail tl = tail ? *tail : LoopTail{};
  const bool loop_form = !z_nom && !h_nom && (tu8 || tf) && partials && g.n() % 4 == 0 && g.W % 4 == 0;
  if (loop_form) {
    if (g.prec == F64)
      k_resist_loop<double><<<kRedBlocks, kRedThreads, 0, s>>>(
          g.n() / 4, static_cast<const double*>(If), static_cast<const double*>(Id), tu8, tf, p,
          static_cast<double*>(wf), static_cast<double*>(wd), partials, stop, g.W, ix0, ix1, iy0, iy1, tl);
    else
      k_resist_loop<float><<<kRedBlocks, kRedThreads, 0, s>>>(
          g.n() / 4, static_cast<const float*>(If), static_cast<const float*>(Id), tu8, tf, p,
          static_cast<float*>(wf), static_cast<float*>(wd), partials, stop, g.W, ix0, ix1, iy0, iy1, tl);
    return;
  }
  if (tail) throw std::invalid_argument("fused loop control needs the DSO loop form of the resist pass");
  if (g.prec == F64)
    k_resist<double><<<kRedBlocks, kRedThreads, 0, s>>>(
        g.n(), static_cast<const double*>(If), static_cast<const double*>(Id), tu8, tf, p,
        static_cast<double*>(wf), static_cast<double*>(wd), z_nom, z_in, z_out, h_nom, h_in, h_out, partials, stop,
        g.W, ix0, ix1, iy0, iy1);
  else
    k_resist<float><<<kRedBlocks, kRedThreads, 0, s>>>(
        g.n(), static_cast<const float*>(If), static_cast<const float*>(Id), tu8, tf, p,
        static_cast<float*>(wf), static_cast<float*>(wd), z_nom, z_in, z_out, h_nom, h_in, h_out, partials, stop,
        g.W, ix0, ix1, iy0, iy1);
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
