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
#include <stdexcept>

#include "common.cuh"
#include "control.cuh"
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
LS_D Geom geometry_at(const double* __restrict__ phi, int H, int W, int y, int x, int xlo = 0, int xhi = -1,
                      int ylo = 0, int yhi = -1) {
  if (xhi < 0) xhi = W;
  if (yhi < 0 || yhi > H) yhi = H;
  const int xe = x + 1 < xhi ? x + 1 : xhi - 1, xw = x > xlo ? x - 1 : xlo;
  const int ys = y + 1 < yhi ? y + 1 : yhi - 1, yn = y > ylo ? y - 1 : ylo;
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

// Stencil input of one pixel (levelset.py:112-118 operands + the loop fields);
// dmx .. dpy: one-sided differences for the opt-in upwind |grad phi|
struct VelIn {
  Geom g;
  double v, dp, m;
  double dmx, dpx, dmy, dpy;
};

// Opt-in extension (not in the reference, which uses the central |grad phi|
// of levelset.py:60-62 in the update): Godunov upwind |grad phi| for
// phi_t + F |grad phi| = 0 with F = v_total (Osher & Sethian), one-sided
// differences with replicate padding, summed in the order
// max(D-x,0)^2 + min(D+x,0)^2 + max(D-y,0)^2 + min(D+y,0)^2 for F > 0 and the
// mirrored terms otherwise (oracle/lsopc_oracle.py grad_mag_upwind).
LS_D double upwind_mag(const VelIn& a, double F) {
  double tx0, tx1, ty0, ty1;
  if (F > 0.0) {
    tx0 = fmax(a.dmx, 0.0); tx1 = fmin(a.dpx, 0.0); ty0 = fmax(a.dmy, 0.0); ty1 = fmin(a.dpy, 0.0);
  } else {
    tx0 = fmin(a.dmx, 0.0); tx1 = fmax(a.dpx, 0.0); ty0 = fmin(a.dmy, 0.0); ty1 = fmax(a.dpy, 0.0);
  }
  return __dsqrt_rn(add(add(add(mul(tx0, tx0), mul(tx1, tx1)), mul(ty0, ty0)), mul(ty1, ty1)));
}

// one-sided differences at (y, x) with the stencil's clamps (slow path)
LS_D void one_sided_at(const double* __restrict__ phi, int H, int W, int y, int x, int xlo, int xhi, int ylo,
                       int yhi, VelIn& a) {
  const int xe = x + 1 < xhi ? x + 1 : xhi - 1, xw = x > xlo ? x - 1 : xlo;
  const int ys = y + 1 < yhi ? y + 1 : yhi - 1, yn = y > ylo ? y - 1 : ylo;
  const double c = phi[(size_t)y * W + x];
  a.dmx = sub(c, phi[(size_t)y * W + xw]);
  a.dpx = sub(phi[(size_t)y * W + xe], c);
  a.dmy = sub(c, phi[(size_t)yn * W + x]);
  a.dpy = sub(phi[(size_t)ys * W + x], c);
}

// _step_fields (optimizer.py:180-194) + the update field of optimizer.py:262:
//   d = -v (+ beta d_prev); v_total = d - kappa/(|grad phi| + 1e-8); u = -v_total |grad phi|
LS_D double vel_emit(const VelIn& a, int use_beta, double beta, int use_curv, bool have_m, double weight,
                     double& gm_out, double& d_out, double& gu_out, int upwind) {
  const double gm = np_hypot(a.g.gx, a.g.gy);
  double d = -a.v;
  if (use_beta) d = add(d, mul(beta, a.dp));
  double vt = d;
  if (use_curv) {
    double k = curvature_of(a.g, weight);
    if (have_m) k = mul(k, a.m);
    vt = sub(d, dvd(k, add(gm, 1e-8)));
  }
  gm_out = gm;
  d_out = d;
  gu_out = upwind ? upwind_mag(a, vt) : gm;  // |grad phi| of the update term
  return vt;
}

// Two horizontally adjacent pixels (x even) per trip: the three stencil rows
// are read as a 4-wide window (16 B loads for the centre pair), the loop
// fields as double2, so each thread keeps enough bytes in flight; pairs that
// touch a clamped column fall back to the per-pixel stencil.
constexpr int kVelThreads = 192;  // 80 registers: four 6-warp blocks per SM keep kBlocks one wave
template <bool UPWIND>
__global__ void __launch_bounds__(kVelThreads, kBlocks / 148)
k_ls_velocity(int H, int W, const double* __restrict__ phi, const double* __restrict__ v,
              const double* __restrict__ dprev, const double* __restrict__ m, double weight, int use_curv,
              DevState* st, double* d_out, double* u_out, double* gm_out, double* partials, Tile tl,
              LoopTail tail) {
  constexpr int upwind = UPWIND;
  __shared__ double red[64];
  if (st->stopped) return;
  const int use_beta = st->use_beta;
  const double beta = st->beta;
  const size_t n2 = (size_t)H * W / 2;
  double mx[2] = {0.0, 0.0};  // max |v_total|, max |grad phi|
  const RowSplit rs = row_split(W);
  const int yhi = tl.yhi < H ? tl.yhi : H, ylo = tl.ylo;
  const int iy1 = tl.iy1 < H ? tl.iy1 : H;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n2; q += (size_t)gridDim.x * blockDim.x) {
    const size_t i = 2 * q;
    const int y = (int)row_of(rs, i), x = (int)col_of(rs, i);
    VelIn a[2];
    if (x - 1 >= tl.xlo && x + 2 < tl.xhi) {
      const int ys = y + 1 < yhi ? y + 1 : yhi - 1, yn = y > ylo ? y - 1 : ylo;
      const double* r = phi + (size_t)y * W + x;
      const double* rS = phi + (size_t)ys * W + x;
      const double* rN = phi + (size_t)yn * W + x;
      const double2 c0 = *reinterpret_cast<const double2*>(r), s0 = *reinterpret_cast<const double2*>(rS),
                    n0 = *reinterpret_cast<const double2*>(rN);
      const double cw = r[-1], ce = r[2], sw = rS[-1], se = rS[2], nw = rN[-1], ne = rN[2];
      // window columns x-1, x, x+1, x+2 of rows y, y+1 (s), y-1 (n)
      const double R0[4] = {cw, c0.x, c0.y, ce}, S0[4] = {sw, s0.x, s0.y, se}, N0[4] = {nw, n0.x, n0.y, ne};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        Geom& g = a[e].g;
        const double c = R0[1 + e], ee = R0[2 + e], w = R0[e], s = S0[1 + e], nn = N0[1 + e];
        g.gx = mul(0.5, sub(ee, w));
        g.gy = mul(0.5, sub(s, nn));
        g.gxx = sub(add(ee, w), mul(2.0, c));
        g.gyy = sub(add(s, nn), mul(2.0, c));
        g.gxy = mul(0.25, sub(sub(S0[2 + e], S0[e]), sub(N0[2 + e], N0[e])));
        if (upwind) {
          a[e].dmx = sub(c, w);
          a[e].dpx = sub(ee, c);
          a[e].dmy = sub(c, nn);
          a[e].dpy = sub(s, c);
        }
      }
    } else {
      a[0].g = geometry_at(phi, H, W, y, x, tl.xlo, tl.xhi, ylo, yhi);
      a[1].g = geometry_at(phi, H, W, y, x + 1, tl.xlo, tl.xhi, ylo, yhi);
      if (upwind) {
        one_sided_at(phi, H, W, y, x, tl.xlo, tl.xhi, ylo, yhi, a[0]);
        one_sided_at(phi, H, W, y, x + 1, tl.xlo, tl.xhi, ylo, yhi, a[1]);
      }
    }
    const double2 vv = *reinterpret_cast<const double2*>(v + i);
    a[0].v = vv.x;
    a[1].v = vv.y;
    if (use_beta) {
      const double2 t = *reinterpret_cast<const double2*>(dprev + i);
      a[0].dp = t.x;
      a[1].dp = t.y;
    } else {
      a[0].dp = a[1].dp = 0.0;
    }
    if (m) {
      const double2 t = *reinterpret_cast<const double2*>(m + i);
      a[0].m = t.x;
      a[1].m = t.y;
    } else {
      a[0].m = a[1].m = 1.0;
    }
    double vt[2], gm[2], d[2], gu[2];
#pragma unroll
    for (int e = 0; e < 2; ++e)
      vt[e] = vel_emit(a[e], use_beta, beta, use_curv, m != nullptr, weight, gm[e], d[e], gu[e], upwind);
    *reinterpret_cast<double2*>(d_out + i) = make_double2(d[0], d[1]);
    if (gm_out) {  // modulation_search form: keep v_total and |grad phi| apart
      *reinterpret_cast<double2*>(u_out + i) = make_double2(vt[0], vt[1]);
      *reinterpret_cast<double2*>(gm_out + i) = make_double2(gu[0], gu[1]);
    } else {
      *reinterpret_cast<double2*>(u_out + i) = make_double2(mul(-vt[0], gu[0]), mul(-vt[1], gu[1]));
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (x + e >= tl.ix0 && x + e < tl.ix1 && y >= tl.iy0 && y < iy1) {
        mx[0] = nmax(mx[0], fabs(vt[e]));
        mx[1] = nmax(mx[1], gm[e]);
      }
    }
  }
  block_max<2>(mx, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = mx[0];
    partials[2 * blockIdx.x + 1] = mx[1];
  }
  if (tail.st && last_block(&tail.st->ticket[2], red)) {
    after_velocity_body(partials, gridDim.x, tail.eta, tail.st, tail.hist, red);
    release_ticket(&tail.st->ticket[2]);
  }
}

// optimizer.py:266-268: phi <- clip(phi + dt * u, D_l, D_u); next mask = [phi <= 0].
// Four pixels per trip (16 B loads); a group that straddles the strip
// interior's edge takes the per-pixel path (halo pixels are left untouched).
__global__ void __launch_bounds__(kThreads)
k_ls_update(int H, int W, double* phi, const double* __restrict__ u, const double* __restrict__ gm, double lo,
            double hi, DevState* st, uint8_t* mask, double* partials, Tile tl, LoopTail tail) {
  __shared__ double red[32];
  if (st->stopped) return;
  const double dt = st->dt;
  const size_t n4 = (size_t)H * W / 4;
  double mx[1] = {0.0};
  const RowSplit rs = row_split(W);
  const bool all_rows = tl.iy0 <= 0 && tl.iy1 >= H;
  const bool whole = tl.ix0 <= 0 && tl.ix1 >= W && all_rows;
  auto one = [&](double ph, double uu, double gg, double& step) {
    if (gm) {  // optimizer.py:329: phi - dt * v_total * grad_mag
      step = mul(mul(dt, uu), gg);
      return nclip(sub(ph, step), lo, hi);
    }
    step = mul(dt, uu);  // optimizer.py:262,266: phi + dt * (-v_total * grad_mag)
    return nclip(add(ph, step), lo, hi);
  };
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x) {
    const size_t i = 4 * q;
    const int x = whole ? 0 : (int)col_of(rs, i);
    const bool row_in = all_rows || ((int)row_of(rs, i) >= tl.iy0 && (int)row_of(rs, i) < tl.iy1);
    if (whole || (row_in && x >= tl.ix0 && x + 4 <= tl.ix1)) {
      const double2 p0 = *reinterpret_cast<const double2*>(phi + i), p1 = *reinterpret_cast<const double2*>(phi + i + 2);
      const double2 u0 = *reinterpret_cast<const double2*>(u + i), u1 = *reinterpret_cast<const double2*>(u + i + 2);
      double2 g0 = make_double2(0.0, 0.0), g1 = g0;
      if (gm) {
        g0 = *reinterpret_cast<const double2*>(gm + i);
        g1 = *reinterpret_cast<const double2*>(gm + i + 2);
      }
      double s0, s1, s2, s3;
      const double q0 = one(p0.x, u0.x, g0.x, s0), q1 = one(p0.y, u0.y, g0.y, s1), q2 = one(p1.x, u1.x, g1.x, s2),
                   q3 = one(p1.y, u1.y, g1.y, s3);
      *reinterpret_cast<double2*>(phi + i) = make_double2(q0, q1);
      *reinterpret_cast<double2*>(phi + i + 2) = make_double2(q2, q3);
      *reinterpret_cast<uchar4*>(mask + i) = make_uchar4(q0 <= 0.0, q1 <= 0.0, q2 <= 0.0, q3 <= 0.0);
      mx[0] = nmax(nmax(nmax(mx[0], fabs(s0)), nmax(fabs(s1), fabs(s2))), fabs(s3));
    } else {
      for (int e = 0; e < 4; ++e) {
        if (!row_in || x + e < tl.ix0 || x + e >= tl.ix1) continue;  // strip halo: owned by a neighbour rank
        double step;
        const double p = one(phi[i + e], u[i + e], gm ? gm[i + e] : 0.0, step);
        phi[i + e] = p;
        mask[i + e] = p <= 0.0;
        mx[0] = nmax(mx[0], fabs(step));
      }
    }
  }
  block_max<1>(mx, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = mx[0];
  if (tail.st && last_block(&tail.st->ticket[3], red)) {
    after_update_body(partials, gridDim.x, tail.st, tail.hist, red);
    release_ticket(&tail.st->ticket[3]);
  }
}

__global__ void k_copy_best(size_t n, const double* __restrict__ phi, double* best, const DevState* st) {
  if (!st->improved) return;
  const size_t n2 = n / 2;  // 16 B copies, odd tail below
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<double2*>(best)[i] = reinterpret_cast<const double2*>(phi)[i];
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) best[n - 1] = phi[n - 1];
}

// ---- loop control: single-block kernels (strip phases, API); the DSO graph
// runs the same bodies as fused tails of their producers (control.cuh)

__global__ void k_after_forward(const double* part, int nb, LoopCfg c, DevState* st, double* hist) {
  __shared__ double red[128];
  after_forward_body(part, nb, c, st, hist, red);
}
__global__ void k_after_grad(const double* dots, int nb, int restart_every, DevState* st) {
  __shared__ double red[64];
  after_grad_body(dots, nb, restart_every, st, red);
}
__global__ void k_after_velocity(const double* part, int nb, double eta, DevState* st, double* hist) {
  __shared__ double red[64];
  after_velocity_body(part, nb, eta, st, hist, red);
}
__global__ void k_after_update(const double* part, int nb, DevState* st, double* hist) {
  __shared__ double red[32];
  after_update_body(part, nb, st, hist, red);
}

// opt-in reinitialisation gate (internal_ls.h launch_reinit_gate)
__global__ void k_reinit_gate(const DevState* st, const double* lit, double n, int every, int* skip) {
  const double c = *lit;
  *skip = (st->stopped || every <= 0 || st->it % every != 0 || c == 0.0 || c == n) ? 1 : 0;
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
        out[i] = nclip(add(a[i], mul(p0, b[i])), p1, p2); break;
      case EW_AHF:                                                   // levelset.py:151
        out[i] = mul(0.5, add(1.0, mul(2.0 / CUDART_PI, atan(dvd(a[i], p0))))); break;
      case EW_HYPOT: out[i] = np_hypot(a[i], b[i]); break;          // levelset.py:62
      default: break;
    }
  }
}

// target != 0 -> 0 / 1 bytes in place (optimizer.py:197: np.asarray(target) != 0),
// 16 bytes per thread step
__global__ void k_binarize_u8(size_t n, uint8_t* p) {
  const size_t n16 = n / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = reinterpret_cast<uint4*>(p)[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // per byte: 1 if non-zero
      const uint32_t x = w[k];
      const uint32_t nz = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
      w[k] = (nz >> 7) & 0x01010101u;
    }
    reinterpret_cast<uint4*>(p)[i] = v;
  }
  for (size_t i = n16 * 16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = p[i] != 0;
}

// DevelSet-Net outputs -> DSO inputs in one pass (boundary
// optimizer.py:215-228): phi0 = clip(phi_raw, D_l, D_u), m = AHF_eps(m_raw)
// (levelset.py:147-151), float32 network outputs widened to float64.
__global__ void k_dsn_init(size_t n, const float* __restrict__ phi_raw, const float* __restrict__ m_raw,
                           double lo, double hi, double eps, double* phi0, double* m) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    phi0[i] = nclip((double)phi_raw[i], lo, hi);
    m[i] = mul(0.5, add(1.0, mul(2.0 / CUDART_PI, atan(dvd((double)m_raw[i], eps)))));
  }
}

__global__ void __launch_bounds__(kThreads)
k_reduce(int op, size_t n, const double* __restrict__ a, const double* __restrict__ b,
         const uint8_t* __restrict__ a8, const uint8_t* __restrict__ b8, double* partials, int W, int ix0, int ix1,
         int iy0, int iy1) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    switch (op) {
      case RD_SUMSQDIFF: { double t = a[i] - b[i]; acc[0] += t * t; } break;
      case RD_DOT: acc[0] += a[i] * b[i]; break;
      case RD_DOTDIFF: acc[0] += a[i] * (a[i] - b[i]); break;
      case RD_MAXABS: acc[0] = nmax(acc[0], fabs(a[i])); break;
      case RD_COUNTNEQ8:  // b8 null: vs 0; W > 0: columns [ix0, ix1) x rows [iy0, iy1) only
        if (W > 0) {
          const int x = (int)col_of(row_split(W), i), y = (int)row_of(row_split(W), i);
          if (x < ix0 || x >= ix1 || y < iy0 || y >= iy1) break;
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
  __shared__ double red[32 * NV];
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
                        double weight, int use_curv, DevState* st, double* d, double* u, double* gm,
                        double* partials, Tile t, cudaStream_t s, const LoopTail* tail, int upwind) {
  if (W % 4) throw std::invalid_argument("level-set loop kernels need a width divisible by 4");
  if (upwind)
    k_ls_velocity<true><<<kBlocks, kVelThreads, 0, s>>>(H, W, phi, v, dprev, m, weight, use_curv, st, d, u, gm,
                                                        partials, t, tail ? *tail : LoopTail{});
  else
    k_ls_velocity<false><<<kBlocks, kVelThreads, 0, s>>>(H, W, phi, v, dprev, m, weight, use_curv, st, d, u, gm,
                                                         partials, t, tail ? *tail : LoopTail{});
}
void launch_ls_update(int H, int W, double* phi, const double* u, const double* gm, double lo, double hi,
                      DevState* st, uint8_t* mask, double* partials, Tile t, cudaStream_t s, const LoopTail* tail) {
  if (W % 4) throw std::invalid_argument("level-set loop kernels need a width divisible by 4");
  k_ls_update<<<kBlocks, kThreads, 0, s>>>(H, W, phi, u, gm, lo, hi, st, mask, partials, t,
                                           tail ? *tail : LoopTail{});
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
  if (nv == 4) {
    k_reduce_partials<4, false><<<1, 256, 0, s>>>(part, nb, out);
  } else if (nv == 1) {
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
void launch_reinit_gate(const DevState* st, const double* lit, double n, int every, int* skip, cudaStream_t s) {
  k_reinit_gate<<<1, 1, 0, s>>>(st, lit, n, every, skip);
}
void launch_binarize_u8(size_t n, uint8_t* p, cudaStream_t s) {
  k_binarize_u8<<<kBlocks, kThreads, 0, s>>>(n, p);
}
void launch_reduce(int op, size_t n, const double* a, const double* b, const uint8_t* a8, const uint8_t* b8,
                   double* partials, double* out, cudaStream_t s, int W, int ix0, int ix1, int iy0, int iy1) {
  k_reduce<<<kBlocks, kThreads, 0, s>>>(op, n, a, b, a8, b8, partials, W, ix0, ix1, iy0, iy1);
  k_reduce_final<<<1, 256, 0, s>>>(op, partials, kBlocks, out);
}

}  // namespace lsb
