// Level-set stencils, CG direction, CFL step and the clamped update, plus the
// small deterministic reductions and elementwise operators on the path.
//
// Replaces (reference, /root/reference/pkg/src/lsopc):
//   mask_from_phi / heaviside              levelset.py:104-106,142-144   (a7)
//   geometry_gradient / .magnitude         levelset.py:109-119,60-62     (a16)
//   curvature                              levelset.py:126-139           (a17)
//   velocity / cg_direction / cfl_timestep optimizer.py:132-169          (a14,a15,a19)
//   _step_fields, update + record          optimizer.py:180-194,257-269  (a18,a20)
//   evolve_step / motion_term              levelset.py:154-166, optimizer.py:137-140
//   l2_error / pvband                      metrics.py:39-52              (a24)
//
// All level-set arithmetic is float64 and written with explicit
// round-to-nearest intrinsics in the reference's evaluation order, so no FMA
// contraction changes a bit: the stencil results are bit-identical to numpy.
// |grad phi| reproduces glibc's hypot (the kernel numpy.hypot calls).
#include "common.cuh"
#include "internal_ls.h"

namespace lsb {

namespace {

LS_D double mul(double a, double b) { return __dmul_rn(a, b); }
LS_D double add(double a, double b) { return __dadd_rn(a, b); }
LS_D double sub(double a, double b) { return __dsub_rn(a, b); }
LS_D double dvd(double a, double b) { return __ddiv_rn(a, b); }

// glibc (>= 2.35) __ieee754_hypot, non-FMA kernel: sysdeps/ieee754/dbl-64/e_hypot.c
LS_D double glibc_hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(add(mul(ax, ax), mul(ay, ay)));
  double t1, t2;
  if (h <= mul(2.0, ay)) {
    double delta = sub(h, ay);
    t1 = mul(ax, sub(mul(2.0, delta), ax));
    t2 = mul(sub(delta, mul(2.0, sub(ax, ay))), delta);
  } else {
    double delta = sub(h, ax);
    t1 = mul(mul(2.0, delta), sub(ax, mul(2.0, ay)));
    t2 = add(mul(sub(mul(4.0, delta), ay), ay), mul(delta, delta));
  }
  return sub(h, dvd(add(t1, t2), mul(2.0, h)));
}

LS_D double np_hypot(double x, double y) {
  if (isinf(x) || isinf(y)) return CUDART_INF;
  if (isnan(x) || isnan(y)) return x + y;
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  if (ax > LARGE) {
    if (ay <= mul(ax, EPS)) return add(ax, ay);
    return dvd(glibc_hypot_kernel(mul(ax, SCALE), mul(ay, SCALE)), SCALE);
  }
  if (ay < TINY) {
    if (ax >= dvd(ay, EPS)) return add(ax, ay);
    return mul(glibc_hypot_kernel(dvd(ax, SCALE), dvd(ay, SCALE)), SCALE);
  }
  if (ay <= mul(ax, EPS)) return add(ax, ay);
  return glibc_hypot_kernel(ax, ay);
}

struct Geom {
  double gx, gy, gxx, gyy, gxy;
};

// levelset.py:112-118, replicate ("edge") padding; x-neighbours clamped to
// [xlo, xhi) (the whole row unless the grid is a strip of a larger tile)
LS_D Geom geometry_at(const double* __restrict__ phi, int H, int W, int y, int x, int xlo = 0, int xhi = -1) {
  if (xhi < 0) xhi = W;
  const int xe = x + 1 < xhi ? x + 1 : xhi - 1, xw = x > xlo ? x - 1 : xlo;
  const int ys = y + 1 < H ? y + 1 : H - 1, yn = y > 0 ? y - 1 : 0;
  const double* r = phi + (size_t)y * W;
  const double* rs = phi + (size_t)ys * W;
  const double* rn = phi + (size_t)yn * W;
  const double c = r[x], e = r[xe], w = r[xw], s = rs[x], n = rn[x];
  Geom g;
  g.gx = mul(0.5, sub(e, w));
  g.gy = mul(0.5, sub(s, n));
  g.gxx = sub(add(e, w), mul(2.0, c));
  g.gyy = sub(add(s, n), mul(2.0, c));
  g.gxy = mul(0.25, sub(sub(rs[xe], rs[xw]), sub(rn[xe], rn[xw])));
  return g;
}

// levelset.py:135-136 (weight * num / den), EPS_DEN = 1e-8
LS_D double curvature_of(const Geom& g, double weight) {
  double gy2 = mul(g.gy, g.gy), gx2 = mul(g.gx, g.gx);
  double num = add(sub(mul(g.gxx, gy2), mul(mul(mul(2.0, g.gy), g.gx), g.gxy)), mul(g.gyy, gx2));
  return dvd(mul(weight, num), add(add(gx2, gy2), 1e-8));
}

constexpr int kBlocks = 148 * 4;
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
k_geometry(int H, int W, const double* __restrict__ phi, double* gx, double* gy, double* gxx, double* gyy,
           double* gxy, double* mag) {
  const size_t n = (size_t)H * W;
  const RowSplit rs = row_split(W);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)row_of(rs, i), x = (int)col_of(rs, i);
    Geom g = geometry_at(phi, H, W, y, x);
    if (gx) { gx[i] = g.gx; gy[i] = g.gy; gxx[i] = g.gxx; gyy[i] = g.gyy; gxy[i] = g.gxy; }
    if (mag) mag[i] = np_hypot(g.gx, g.gy);
  }
}

__global__ void __launch_bounds__(kThreads)
k_curvature(int H, int W, const double* __restrict__ phi, const double* __restrict__ m, double weight,
            double* out) {
  const size_t n = (size_t)H * W;
  const RowSplit rs = row_split(W);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)row_of(rs, i), x = (int)col_of(rs, i);
    double k = curvature_of(geometry_at(phi, H, W, y, x), weight);
    out[i] = m ? mul(k, m[i]) : k;
  }
}

// ---- loop kernels -------------------------------------------------------------

// _step_fields (optimizer.py:180-194) + the update field of optimizer.py:262:
//   d = -v (+ beta d_prev); v_total = d - kappa/(|grad phi| + 1e-8); u = -v_total |grad phi|
__global__ void __launch_bounds__(kThreads)
k_ls_velocity(int H, int W, const double* __restrict__ phi, const double* __restrict__ v,
              const double* __restrict__ dprev, const double* __restrict__ m, double weight, int use_curv,
              const DevState* st, double* d_out, double* u_out, double* gm_out, double* partials, Tile tl) {
  __shared__ double red[64];
  if (st->stopped) return;
  const int use_beta = st->use_beta;
  const double beta = st->beta;
  const size_t n = (size_t)H * W;
  double mx[2] = {0.0, 0.0};  // max |v_total|, max |grad phi|
  const RowSplit rs = row_split(W);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)row_of(rs, i), x = (int)col_of(rs, i);
    Geom g = geometry_at(phi, H, W, y, x, tl.xlo, tl.xhi);
    double gm = np_hypot(g.gx, g.gy);
    double d = -v[i];
    if (use_beta) d = add(d, mul(beta, dprev[i]));
    double vt = d;
    if (use_curv) {
      double k = curvature_of(g, weight);
      if (m) k = mul(k, m[i]);
      vt = sub(d, dvd(k, add(gm, 1e-8)));
    }
    d_out[i] = d;
    if (gm_out) {  // modulation_search form: keep v_total and |grad phi| apart
      u_out[i] = vt;
      gm_out[i] = gm;
    } else {
      u_out[i] = mul(-vt, gm);
    }
    if (x >= tl.ix0 && x < tl.ix1) {
      mx[0] = fmax(mx[0], fabs(vt));
      mx[1] = fmax(mx[1], gm);
    }
  }
  block_max<2>(mx, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = mx[0];
    partials[2 * blockIdx.x + 1] = mx[1];
  }
}

// optimizer.py:266-268: phi <- clip(phi + dt * u, D_l, D_u); next mask = [phi <= 0]
__global__ void __launch_bounds__(kThreads)
k_ls_update(int H, int W, double* phi, const double* __restrict__ u, const double* __restrict__ gm, double lo,
            double hi, const DevState* st, uint8_t* mask, double* partials, Tile tl) {
  __shared__ double red[32];
  if (st->stopped) return;
  const double dt = st->dt;
  const size_t n = (size_t)H * W;
  double mx[1] = {0.0};
  const RowSplit rs = row_split(W);
  const bool whole = tl.ix0 <= 0 && tl.ix1 >= W;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = whole ? 0 : (int)col_of(rs, i);
    if (x < tl.ix0 || x >= tl.ix1) continue;  // strip halo: owned by a neighbour rank
    double step, p;
    if (gm) {  // optimizer.py:329: phi - dt * v_total * grad_mag
      step = mul(mul(dt, u[i]), gm[i]);
      p = fmin(fmax(sub(phi[i], step), lo), hi);
    } else {   // optimizer.py:262,266: phi + dt * (-v_total * grad_mag)
      step = mul(dt, u[i]);
      p = fmin(fmax(add(phi[i], step), lo), hi);
    }
    phi[i] = p;
    mask[i] = p <= 0.0;
    mx[0] = fmax(mx[0], fabs(step));
  }
  block_max<1>(mx, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = mx[0];
}

__global__ void k_copy_best(size_t n, const double* __restrict__ phi, double* best, const DevState* st) {
  if (!st->improved) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    best[i] = phi[i];
}

// fixed-order reduction of nb partial pairs by one block
template <int NV, bool MAX>
LS_D void reduce_partials(const double* part, int nb, double (&out)[NV], double* red) {
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
#pragma unroll
    for (int j = 0; j < NV; ++j) acc[j] = MAX ? fmax(acc[j], part[NV * b + j]) : acc[j] + part[NV * b + j];
  }
  if (MAX) block_max<NV>(acc, red);
  else block_sum<NV>(acc, red);
#pragma unroll
  for (int j = 0; j < NV; ++j) out[j] = acc[j];
}

// optimizer.py:238-251: loss, best iterate, patience
__global__ void k_after_forward(const double* part, int nb, LoopCfg c, DevState* st, double* hist) {
  __shared__ double red[64];
  if (st->stopped) return;
  double l[2];
  reduce_partials<2, false>(part, nb, l, red);
  if (threadIdx.x != 0) return;
  const double l_ilt = l[0], l_pvb = l[1];
  const double l_dso = c.alpha * l_ilt + c.beta * l_pvb;
  st->l_ilt = l_ilt;
  st->l_pvb = l_pvb;
  st->l_dso = l_dso;
  st->improved = 0;
  if (!isfinite(l_dso)) {
    st->nonfinite_it = st->it;
    st->stopped = 1;
    return;
  }
  double rel;
  if (l_dso < st->best) {
    rel = isfinite(st->best) ? (st->best - l_dso) / st->best : CUDART_INF;
    st->best = l_dso;
    st->improved = 1;
  } else {
    rel = 0.0;
  }
  st->streak = rel < c.stop_rel_tol ? st->streak + 1 : 0;
  if (st->streak >= c.stop_patience) {
    double* h = hist + 7 * st->nhist;
    h[0] = l_ilt; h[1] = l_pvb; h[2] = l_dso; h[3] = 0.0; h[4] = 0.0; h[5] = 0.0; h[6] = 0.0;
    st->nhist += 1;
    st->stopped = 1;
  }
}

// optimizer.py:154-169,253: Polak-Ribiere beta with restart
__global__ void k_after_grad(const double* dots, int nb, int restart_every, DevState* st) {
  __shared__ double red[64];
  if (st->stopped) return;
  const int restart = st->it == 0 || st->it % restart_every == 0;
  double s[2] = {0.0, 0.0};
  if (!restart) reduce_partials<2, false>(dots, nb, s, red);
  if (threadIdx.x != 0) return;
  st->use_beta = 0;
  st->beta = 0.0;
  if (restart || s[1] == 0.0) return;
  double b = s[0] / s[1];
  if (b <= 0.0) return;
  st->beta = b;
  st->use_beta = 1;
}

// optimizer.py:143-151,257-261: dt = eta / max|v_total|
__global__ void k_after_velocity(const double* part, int nb, double eta, DevState* st, double* hist) {
  __shared__ double red[64];
  if (st->stopped) return;
  double m[2];
  reduce_partials<2, true>(part, nb, m, red);
  if (threadIdx.x != 0) return;
  st->vmax = m[0];
  st->gmax = m[1];
  if (m[0] == 0.0) {
    double* h = hist + 7 * st->nhist;
    h[0] = st->l_ilt; h[1] = st->l_pvb; h[2] = st->l_dso; h[3] = 0.0; h[4] = 0.0; h[5] = 0.0; h[6] = m[1];
    st->nhist += 1;
    st->stopped = 1;
    return;
  }
  st->dt = eta / m[0];
}

// optimizer.py:262-265: history record of a completed step
__global__ void k_after_update(const double* part, int nb, DevState* st, double* hist) {
  __shared__ double red[32];
  if (st->stopped) return;
  double m[1];
  reduce_partials<1, true>(part, nb, m, red);
  if (threadIdx.x != 0) return;
  double* h = hist + 7 * st->nhist;
  h[0] = st->l_ilt; h[1] = st->l_pvb; h[2] = st->l_dso; h[3] = st->dt; h[4] = st->vmax; h[5] = m[0];
  h[6] = st->gmax;
  st->nhist += 1;
  st->it += 1;
}

// ---- elementwise API operators -------------------------------------------------

__global__ void k_elementwise(int op, size_t n, const double* __restrict__ a, const double* __restrict__ b,
                              double p0, double p1, double p2, double* out, uint8_t* out8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    switch (op) {
      case EW_MASK: out8[i] = a[i] <= 0.0; break;                   // levelset.py:106
      case EW_HEAVISIDE: out8[i] = a[i] >= 0.0; break;              // levelset.py:144
      case EW_AXPBY: out[i] = add(mul(p0, a[i]), mul(p1, b[i])); break;  // optimizer.py:134
      case EW_SIGMOID:                                              // litho.py:138
        out[i] = dvd(1.0, add(1.0, exp(mul(-p0, sub(a[i], p1))))); break;
      case EW_HARD: out8[i] = a[i] >= p0; break;                    // litho.py:131
      case EW_NEG: out[i] = -a[i]; break;                           // optimizer.py:328
      case EW_CG: out[i] = add(-a[i], mul(p0, b[i])); break;        // optimizer.py:335
      case EW_MOTION: out[i] = mul(-a[i], b[i]); break;             // optimizer.py:140 (-v |grad phi|)
      case EW_EVOLVE:                                                // levelset.py:165
        out[i] = fmin(fmax(add(a[i], mul(p0, b[i])), p1), p2); break;
      case EW_AHF:                                                   // levelset.py:151
        out[i] = mul(0.5, add(1.0, mul(2.0 / CUDART_PI, atan(dvd(a[i], p0))))); break;
      case EW_HYPOT: out[i] = np_hypot(a[i], b[i]); break;          // levelset.py:62
      default: break;
    }
  }
}

// DevelSet-Net outputs -> DSO inputs in one pass (boundary
// optimizer.py:215-228): phi0 = clip(phi_raw, D_l, D_u), m = AHF_eps(m_raw)
// (levelset.py:147-151), float32 network outputs widened to float64.
__global__ void k_dsn_init(size_t n, const float* __restrict__ phi_raw, const float* __restrict__ m_raw,
                           double lo, double hi, double eps, double* phi0, double* m) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    phi0[i] = fmin(fmax((double)phi_raw[i], lo), hi);
    m[i] = mul(0.5, add(1.0, mul(2.0 / CUDART_PI, atan(dvd((double)m_raw[i], eps)))));
  }
}

__global__ void __launch_bounds__(kThreads)
k_reduce(int op, size_t n, const double* __restrict__ a, const double* __restrict__ b,
         const uint8_t* __restrict__ a8, const uint8_t* __restrict__ b8, double* partials, int W, int ix0, int ix1) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    switch (op) {
      case RD_SUMSQDIFF: { double t = a[i] - b[i]; acc[0] += t * t; } break;
      case RD_DOT: acc[0] += a[i] * b[i]; break;
      case RD_DOTDIFF: acc[0] += a[i] * (a[i] - b[i]); break;
      case RD_MAXABS: acc[0] = fmax(acc[0], fabs(a[i])); break;
      case RD_COUNTNEQ8:  // b8 null: vs 0; W > 0: columns [ix0, ix1) only
        if (W > 0) {
          const int x = (int)col_of(row_split(W), i);
          if (x < ix0 || x >= ix1) break;
        }
        acc[0] += (a8[i] != (b8 ? b8[i] : 0)) ? 1.0 : 0.0;
        break;
      case RD_COUNTNEQ: acc[0] += (a[i] != b[i]) ? 1.0 : 0.0; break;
      case RD_NONFINITE: if (!isfinite(a[i])) acc[0] = fmax(acc[0], (double)(n - i)); break;
      default: break;
    }
  }
  if (op == RD_MAXABS || op == RD_NONFINITE) block_max<1>(acc, red);
  else block_sum<1>(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
}

template <int NV, bool MAX>
__global__ void k_reduce_partials(const double* part, int nb, double* out) {
  __shared__ double red[64];
  double r[NV];
  reduce_partials<NV, MAX>(part, nb, r, red);
  if (threadIdx.x == 0)
    for (int j = 0; j < NV; ++j) out[j] = r[j];
}

__global__ void k_reduce_final(int op, const double* part, int nb, double* out) {
  __shared__ double red[32];
  double r[1];
  if (op == RD_MAXABS || op == RD_NONFINITE) reduce_partials<1, true>(part, nb, r, red);
  else reduce_partials<1, false>(part, nb, r, red);
  if (threadIdx.x == 0) *out = r[0];
}

}  // namespace

int ls_blocks() { return kBlocks; }

void launch_geometry(int H, int W, const double* phi, double* gx, double* gy, double* gxx, double* gyy,
                     double* gxy, double* mag, cudaStream_t s) {
  k_geometry<<<kBlocks, kThreads, 0, s>>>(H, W, phi, gx, gy, gxx, gyy, gxy, mag);
}
void launch_curvature(int H, int W, const double* phi, const double* m, double weight, double* out,
                      cudaStream_t s) {
  k_curvature<<<kBlocks, kThreads, 0, s>>>(H, W, phi, m, weight, out);
}
void launch_ls_velocity(int H, int W, const double* phi, const double* v, const double* dprev, const double* m,
                        double weight, int use_curv, const DevState* st, double* d, double* u, double* gm,
                        double* partials, Tile t, cudaStream_t s) {
  k_ls_velocity<<<kBlocks, kThreads, 0, s>>>(H, W, phi, v, dprev, m, weight, use_curv, st, d, u, gm, partials, t);
}
void launch_ls_update(int H, int W, double* phi, const double* u, const double* gm, double lo, double hi,
                      const DevState* st, uint8_t* mask, double* partials, Tile t, cudaStream_t s) {
  k_ls_update<<<kBlocks, kThreads, 0, s>>>(H, W, phi, u, gm, lo, hi, st, mask, partials, t);
}
void launch_copy_best(size_t n, const double* phi, double* best, const DevState* st, cudaStream_t s) {
  k_copy_best<<<kBlocks, kThreads, 0, s>>>(n, phi, best, st);
}
void launch_after_forward(const double* part, int nb, LoopCfg c, DevState* st, double* hist, cudaStream_t s) {
  k_after_forward<<<1, 256, 0, s>>>(part, nb, c, st, hist);
}
void launch_after_grad(const double* dots, int nb, int restart_every, DevState* st, cudaStream_t s) {
  k_after_grad<<<1, 256, 0, s>>>(dots, nb, restart_every, st);
}
void launch_after_velocity(const double* part, int nb, double eta, DevState* st, double* hist, cudaStream_t s) {
  k_after_velocity<<<1, 256, 0, s>>>(part, nb, eta, st, hist);
}
void launch_after_update(const double* part, int nb, DevState* st, double* hist, cudaStream_t s) {
  k_after_update<<<1, 256, 0, s>>>(part, nb, st, hist);
}
void launch_dsn_init(size_t n, const float* phi_raw, const float* m_raw, double lo, double hi, double eps,
                     double* phi0, double* m, cudaStream_t s) {
  k_dsn_init<<<kBlocks, kThreads, 0, s>>>(n, phi_raw, m_raw, lo, hi, eps, phi0, m);
}
void launch_reduce_partials(const double* part, int nb, int nv, int is_max, double* out, cudaStream_t s) {
  if (nv == 1) {
    if (is_max) k_reduce_partials<1, true><<<1, 256, 0, s>>>(part, nb, out);
    else k_reduce_partials<1, false><<<1, 256, 0, s>>>(part, nb, out);
  } else {
    if (is_max) k_reduce_partials<2, true><<<1, 256, 0, s>>>(part, nb, out);
    else k_reduce_partials<2, false><<<1, 256, 0, s>>>(part, nb, out);
  }
}
void launch_elementwise(int op, size_t n, const double* a, const double* b, double p0, double p1, double p2,
                        double* out, uint8_t* out8, cudaStream_t s) {
  k_elementwise<<<kBlocks, kThreads, 0, s>>>(op, n, a, b, p0, p1, p2, out, out8);
}
void launch_reduce(int op, size_t n, const double* a, const double* b, const uint8_t* a8, const uint8_t* b8,
                   double* partials, double* out, cudaStream_t s, int W, int ix0, int ix1) {
  k_reduce<<<kBlocks, kThreads, 0, s>>>(op, n, a, b, a8, b8, partials, W, ix0, ix1);
  k_reduce_final<<<1, 256, 0, s>>>(op, partials, kBlocks, out);
}

}  // namespace lsb
