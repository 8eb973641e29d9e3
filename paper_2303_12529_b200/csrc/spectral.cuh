// SOCS forward model and adjoint as persistent, pipelined spectral passes
// (templates; instantiated per precision in spec_*.cu, launched from spectral.cu).
//
// Replaces (reference, /root/reference/pkg/src/lsopc):
//   KernelSet.stacked_ffts + embed_kernel      litho.py:71-82, fields.py:61-74   (K0)
//   np.fft.fft2(mask)                          litho.py:124, optimizer.py:108    (K1)
//   aerial_intensity / print_corners           litho.py:114-154                  (K2)
//   _socs_gradient / ilt_ / pvb_gradient       optimizer.py:99-129               (K4)
//
// One DSO iteration is five spectral passes over all 2*N_k kernels instead
// of the reference's 294 full 2-D transforms:
//
//   mask:  M^ = FFT_y FFT_x [phi <= 0]                      rows + cols, once
//   F1  (cols, item = column tile x set, loop over kernels):
//        T_k = IFFT_y(M^ . H_k) / (HW)             M^ tile stays in smem
//   F2  (rows, item = row block x set, loop over kernels):
//        A_k = IFFT_x T_k  (in place),  I_set = sum_k w_k |A_k|^2 in registers
//   A1  (rows, item = row block x set, loop over kernels):
//        U_k = FFT_x(gate_set . A_k)              U_k overwrites A_k
//   A2  (cols, item = column tile x set, loop over kernels):
//        V_set = IFFT_y( sum_k w_k conj(H_k) . FFT_y U_k )   accumulated in registers
//   A3  (rows): g = scale . Re IFFT_x(V_f + V_d)  (+ CG dot partials)
//
// The adjoint uses conj(t) = IFFT2(FFT2(gate A) conj(H)) (equal real part to
// the reference's IFFT2(FFT2(gate conj A) H(-f))), so forward and adjoint read
// the same spectrum at the same frequency.  One complex field per kernel
// (T_k -> A_k -> U_k, overwritten in place) lives in HBM: it carries the 2-D
// transforms' transposes and the fields the gate needs.  The intensity and
// adjoint-spectrum accumulators stay on chip.
#pragma once
#include "common.cuh"
#include "control.cuh"
#include "engine.cuh"
#include "internal.h"
#include "internal_ls.h"
#include "tma.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace lsb {
namespace spec {

using eng::Geo;
using eng::Lay;

constexpr int kMaxK = 64;  // kernels per set carried in a launch
// Tile widths of the column-tiled layouts (scripts/mb_layout.cu measured on
// B200: whole-tile column items stream at 6.2 TB/s; a 4-row item reads 128 B
// chunks of a 4-wide tiling at 73% of that and 256 B chunks of an 8-wide
// tiling at full speed, while a 4-column item of an 8-wide tiling runs at 91%).
// U_k, V, M^, spectra: 32 B tile rows, so a column item (4 x c64 or 2 x c128) is a whole tile
template <typename C> constexpr int lg_tile() { return sizeof(C) == 8 ? 2 : 1; }
// tall grids split four ways (k_f1_split): natural row y of T_k / U_k / V is
// stored at row (y mod 4) * H/4 + y / 4
LS_HD int split_row(int y, int lgq) { return ((y & 3) << lgq) | (y >> 2); }
constexpr int kLgTileT = 3;  // T_k: read by the F2 row pass as 256 B chunks

// ---- Tall-grid split (Grid::vsplit, H = 8192 = 4 x 2048) -------------------
// With y = n2 + 2048 m and frequency f = 4 f2 + c (n2, f2 < 2048; m, c < 4):
//   X[4 f2 + c] = FFT_2048( z_c )[f2],  z_c[n2] = tw[c n2] sum_m (-i)^(c m) x[n2 + 2048 m]
//   x[n2 + 2048 m] = sum_c i^(c m) conj(tw[c n2]) IFFT_2048( X[4 . + c] )[n2]
// so the radix-4 step runs inside the row passes and every column transform
// is a 2048-point one.  Plane c (frequency rows 4 f2 + c) is stored at rows
// c * 2048 + f2; in a column-tiled layout of tile width w this makes the
// spectral fields exactly the column-tiled layout of a virtual 2048 x 4W
// grid (virtual column ((x / w) * 4 + c) * w + x mod w), so the column
// passes run unchanged on that grid.  A split row item holds R = 4Q rows:
// buffer row m * Q + q is natural row n2_0 + q + 2048 m, or -- before the
// inverse / after the forward combine -- plane row c * Q + q.
constexpr int kVsM = 2048, kLgVsM = 11;
LS_HD int vs_row(int seq, int lgq, int n20) { return n20 + (seq & ((1 << lgq) - 1)) + ((seq >> lgq) << kLgVsM); }
LS_HD int vs_plane_row(int seq, int lgq, int n20) {  // storage row of plane row seq = c * Q + q
  return ((seq >> lgq) << kLgVsM) + n20 + (seq & ((1 << lgq) - 1));
}
template <typename C> LS_D C mul_pi(C z) { return cmk(-z.y, z.x); }  // +i z (mul_mi: -i z)
// forward combine in place: natural rows m * Q + q -> plane rows c * Q + q
template <typename C>
LS_D void vs_fwd_combine(C* b, int lgW, int lgq, int n20, const C* __restrict__ tw, int tws) {
  const int cnt = 1 << (lgq + lgW);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int q = i >> lgW, x = i & ((1 << lgW) - 1), n2 = n20 + q;
    C* p = b + ((size_t)q << lgW) + x;
    const size_t st = (size_t)1 << (lgq + lgW);
    const C y0 = p[0], y1 = p[st], y2 = p[2 * st], y3 = p[3 * st];
    const C a0 = y0 + y2, a1 = y0 - y2, b0 = y1 + y3, b1 = y1 - y3;
    p[0] = a0 + b0;
    p[st] = cmul(a1 + mul_mi(b1), __ldg(&tw[n2 << tws]));
    p[2 * st] = cmul(a0 - b0, __ldg(&tw[(2 * n2) << tws]));
    p[3 * st] = cmul(a1 + mul_pi(b1), __ldg(&tw[(3 * n2) << tws]));
  }
}
// inverse combine in place: plane rows c * Q + q (+ a second accumulator
// read from global at its storage row) -> natural rows m * Q + q
template <typename C>
LS_D void vs_inv_combine(C* b, int lgW, int lgq, int n20, const C* __restrict__ tw, int tws,
                         const C* __restrict__ add = nullptr) {
  const int cnt = 1 << (lgq + lgW);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int q = i >> lgW, x = i & ((1 << lgW) - 1), n2 = n20 + q;
    C* p = b + ((size_t)q << lgW) + x;
    const size_t st = (size_t)1 << (lgq + lgW);
    C z0 = p[0], z1 = p[st], z2 = p[2 * st], z3 = p[3 * st];
    if (add) {
      const size_t W = (size_t)1 << lgW, g = (size_t)n2 * W + x, pl = (size_t)kVsM * W;
      z0 = z0 + __ldg(&add[g]);
      z1 = z1 + __ldg(&add[g + pl]);
      z2 = z2 + __ldg(&add[g + 2 * pl]);
      z3 = z3 + __ldg(&add[g + 3 * pl]);
    }
    z1 = cmulc(z1, __ldg(&tw[n2 << tws]));
    z2 = cmulc(z2, __ldg(&tw[(2 * n2) << tws]));
    z3 = cmulc(z3, __ldg(&tw[(3 * n2) << tws]));
    const C a0 = z0 + z2, a1 = z0 - z2, b0 = z1 + z3, b1 = z1 - z3;
    p[0] = a0 + b0;
    p[st] = a1 + mul_pi(b1);
    p[2 * st] = a0 - b0;
    p[3 * st] = a1 + mul_mi(b1);
  }
}
// the virtual grid of a split plan's column passes
inline Grid vs_grid(const Grid& g) {
  Grid v = g;
  v.H = kVsM;
  v.lgH = kLgVsM;
  v.W = g.W * 4;
  v.lgW = g.lgW + 2;
  v.vsplit = 0;
  return v;
}
// virtual column xv of a tile-width-2^lgt layout -> (physical column, plane)
LS_HD int vs_col(int xv, int lgt) { return ((xv >> (lgt + 2)) << lgt) | (xv & ((1 << lgt) - 1)); }
LS_HD int vs_plane(int xv, int lgt) { return (xv >> lgt) & 3; }

template <typename R> struct Shape {
  int H, W, lgH, lgW;
  int lgS, lgR;     // log2 columns per column item / rows per row item
  int lgT;          // log2 tile width of the column-tiled layout (decoupled from lgS)
  int lgTT;         // log2 tile width of the T_k fields
  int twsH, twsW;   // twiddle-table shifts for the two axes
  LS_HD Geo gcol() const { return Geo{lgH, lgS, twsH}; }
  LS_HD Geo grow() const { return Geo{lgW, lgR, twsW}; }
  LS_HD Lay ct() const { return Lay{H, lgT}; }   // column-tiled layout of spectral fields
  LS_HD Lay rm() const { return Lay{H, lgW}; }   // row-major
  // compile-time-geometry path allowed (layout tile width is the constant one)
  LS_HD bool fast() const { return lgT == lg_tile<typename CT<R>::C>() && lgTT == kLgTileT; }
  LS_HD Lay ctT() const { return Lay{H, lgTT}; }  // layout of the T_k fields
};

template <typename R> Shape<R> shape_of(const Grid& g) {
  using C = typename CT<R>::C;
  const int E = eng::cta_threads<C>() * eng::P_of<C>();
  Shape<R> s;
  s.H = g.H; s.W = g.W; s.lgH = g.lgH; s.lgW = g.lgW;
  s.lgS = std::max(0, std::min(g.lgW, ilog2i(E) - g.lgH));
  s.lgR = std::max(0, std::min(g.lgH, ilog2i(E) - g.lgW));
  s.lgT = std::min(g.lgW, lg_tile<typename CT<R>::C>());
  s.lgTT = std::min(g.lgW, kLgTileT);
  s.twsH = g.lgnmax - g.lgH;
  s.twsW = g.lgnmax - g.lgW;
  return s;
}

template <typename R>
__global__ void k_ct_to_c128(size_t n, Lay L, int W, const typename CT<R>::C* __restrict__ a, double2* out,
                             int split_lgq = -1) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i % W);
    const auto v = a[L.at(split_lgq >= 0 ? split_row(y, split_lgq) : y, x)];
    out[i] = make_double2((double)v.x, (double)v.y);
  }
}

// ---------------------------------------------------------------------------
// persistent skeleton: flattened (item, step) sequence per CTA, operands of
// step q+1 stream in (cp.async) while step q is transformed.

template <typename R, class Op>
__global__ void __launch_bounds__(eng::cta_threads<typename CT<R>::C>(), 1) k_pass(Op op, StopFlag stop) {
  using C = typename CT<R>::C;
  constexpr int NB = Op::kStages;  // ring of stage buffers: prefetch distance NB - 1
#if !defined(LSB_EXP_NOSTORE) && !defined(LSB_EXP_NOGATHER) && !defined(LSB_EXP_NOTMA)
  if (stop && *stop) return;
#endif
  extern __shared__ __align__(16) unsigned char smraw[];
  C* const base = reinterpret_cast<C*>(smraw);
  C* extra = base + NB * op.bufE;
  typename Op::State S{};
  if ((int)blockIdx.x >= op.nitems) return;
  // cursor over this CTA's flattened (item, step) sequence
  auto advance = [&](int& it, int& st) {
    if (++st == op.steps(it)) { st = 0; it += gridDim.x; }
  };
  int it = blockIdx.x, st = 0;
  int pit = it, pst = st;  // next (item, step) to prefetch
#pragma unroll
  for (int d = 0; d < NB - 1; ++d) {
#ifndef LSB_EXP_NOGATHER  // experiment switch: never fetch operands
    if (pit < op.nitems) op.prefetch(pit, op.kbase(pit) + pst, base + d * op.bufE, extra);
#endif
    eng::cp_commit();
    if (pit < op.nitems) advance(pit, pst);
  }
  int slot = 0;  // ring slot of (it, st)
  while (true) {
    const int pslot = slot == 0 ? NB - 1 : slot - 1;  // == (slot + NB - 1) % NB
#ifndef LSB_EXP_NOGATHER
    if (pit < op.nitems) op.prefetch(pit, op.kbase(pit) + pst, base + pslot * op.bufE, extra);
#endif
    eng::cp_commit();
    eng::cp_wait<NB - 1>();
    __syncthreads();
    C* const cur = base + slot * op.bufE;
    if (st == 0) op.begin(S, it, extra);
    op.step(S, it, op.kbase(it) + st, cur, extra);
    __syncthreads();
    if (st == op.steps(it) - 1) op.end(S, it, cur, extra);
    if (pit < op.nitems) advance(pit, pst);
    advance(it, st);
    if (it >= op.nitems) break;
    slot = slot == NB - 1 ? 0 : slot + 1;
  }
  op.finish(S, reinterpret_cast<double*>(smraw));
}

struct NoState {};
struct OpBase {
  static constexpr int kStages = 3;
  int bufE = 0, nitems = 0;
  // Kernel groups (small grids, too few items for the SMs): item index =
  // ((set << lgg | group) << lgt) | block; a group item runs kernels
  // [group * kpg, (group + 1) * kpg).  lgg = 0: one group per set.
  int lgg = 0, kpg = 0;
  LS_D int set_of(int it, int lgt) const { return (it >> lgt) >> lgg; }
  LS_D int grp_of(int it, int lgt) const { return (it >> lgt) & ((1 << lgg) - 1); }
  LS_D int kbase(int) const { return 0; }
  LS_D int steps(int) const { return 1; }
  template <class S, class C> LS_D void begin(S&, int, C*) const {}
  template <class S, class C> LS_D void end(S&, int, C*, C*) const {}
  template <class S> LS_D void finish(S&, double*) const {}
};

// Global stores of the transform outputs.  LSB_EXP_NOSTORE (experiment
// builds only) keeps the arithmetic but drops the writes.
template <class T> LS_D void gstore(T& dst, const T& v) {
#ifdef LSB_EXP_NOSTORE
  if (v.x == (decltype(v.x))1.2345e-30) dst = v;
#else
  dst = v;
#endif
}

// ---- address helpers: idx = j + r*STRIDE (STRIDE == 0: generic path, idx = j)

// natural (as-loaded) buffer position, column buffers [n][S]
template <int LGN, int STRIDE, typename C> LS_D int nat_col(int seq, int j, int r, int lgS) {
  if constexpr (LGN > 0) {
    constexpr int LGS = eng::lg_full<C>() - LGN;
    return (j << LGS) + seq + r * (STRIDE << LGS);
  } else {
    return (j << lgS) + seq;
  }
}
// natural buffer position, row buffers [S][n]
template <int LGN, int STRIDE> LS_D int nat_row(int seq, int j, int r, int lgn) {
  if constexpr (LGN > 0) return (seq << LGN) + j + r * STRIDE;
  else return (seq << lgn) + j;
}
// column-tiled element (y = j + r*STRIDE, x); fast path has tile width 2^kLgTile
template <int LGN, int STRIDE, typename C, int LGT = lg_tile<C>()> LS_D size_t ct_col(const Lay& L, int j, int r, int x) {
  if constexpr (LGN > 0) {
    constexpr int T = 1 << LGT;
    return (((size_t)(x >> LGT) * L.H + j) << LGT) + (x & (T - 1)) + (size_t)r * (STRIDE << LGT);
  } else {
    return L.at(j, x);
  }
}
// column-tiled element (y, x = j + r*STRIDE)
template <int LGN, int STRIDE, typename C, int LGT = lg_tile<C>()> LS_D size_t ct_row(const Lay& L, int y, int j, int r) {
  if constexpr (LGN > 0) {
    constexpr int T = 1 << LGT;
    static_assert(STRIDE % T == 0, "row stride must be a multiple of the tile width");
    return (((size_t)(j >> LGT) * L.H + y) << LGT) + (j & (T - 1)) + (size_t)r * STRIDE * L.H;
  } else {
    return L.at(y, j);
  }
}
// row-major element (y, x = j + r*STRIDE)
template <int LGN, int STRIDE> LS_D size_t rm_row(int W, int y, int j, int r) {
  return (size_t)y * W + j + (size_t)r * STRIDE;
}
// row-major element (y = j + r*STRIDE, x)
template <int LGN, int STRIDE> LS_D size_t rm_col(int W, int j, int r, int x) {
  if constexpr (LGN > 0) return (size_t)(j + r * STRIDE) * W + x;
  else return (size_t)j * W + x;
}

// ---------------------------------------------------------------------------
// mask -> M~ = FFT_x(mask) (rows).  src: u8 mask, f64 mask, or f64 phi (mask = phi <= 0)

enum MaskSrc { SRC_U8 = 0, SRC_F64 = 1, SRC_PHI = 2 };

template <typename R> struct MaskRowsOp : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  Shape<R> sh;
  const void* src;
  int kind;
  C* out;  // column-tiled
  const C* tw;
  LS_D void prefetch(int it, int, C* b, C*) const {
    const int y0 = it << sh.lgR;
    if (kind == SRC_U8) eng::gather_rect<1>(b, src, Lay{sh.H, sh.lgW}, y0, sh.lgR, 0, sh.lgW);
    else eng::gather_rect<8>(b, src, Lay{sh.H, sh.lgW}, y0, sh.lgR, 0, sh.lgW);
  }
  template <int LGN> struct F {
    const unsigned char* raw;
    int kind, y0, lgn;
    C* out;
    Lay L;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      const int p = nat_row<LGN, ST>(seq, j, r, lgn);
      R m;
      if (kind == SRC_U8) m = (R)raw[p];
      else {
        const double v = reinterpret_cast<const double*>(raw)[p];
        m = kind == SRC_PHI ? (R)(v <= 0.0) : (R)v;
      }
      return cmk(m, (R)0);
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { gstore(out[ct_row<LGN, ST, C>(L, y0 + seq, j, r)], v); }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    const Geo g = sh.grow();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{reinterpret_cast<const unsigned char*>(b), kind, it << sh.lgR, sh.lgW, out, sh.ct()};
      eng::run_fix<LGN, false, false>(g, b, tw, f);
    });
  }
};

// ---------------------------------------------------------------------------
// generic column transform: out = scale * FFT_y(in) (or IFFT_y), column-tiled in/out

template <typename R, typename RO, bool INV> struct ColsOp : OpBase {
  using C = typename CT<R>::C;
  using CO = typename CT<RO>::C;
  using State = NoState;
  Shape<R> sh;
  const C* in;
  Lay Lin, Lout;
  CO* out;
  R scale;
  const C* tw;
  LS_D void prefetch(int it, int, C* b, C*) const {
    eng::gather_rect<sizeof(C)>(b, in, Lin, 0, sh.lgH, it << sh.lgS, sh.lgS);
  }
  template <int LGN> struct F {
    const C* b;
    CO* out;
    Lay L;
    int x0, lgS;
    R scale;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const { return b[nat_col<LGN, ST, C>(seq, j, r, lgS)] * scale; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) {
      out[ct_col<LGN, ST, C>(L, j, r, x0 + seq)] = cmk((RO)v.x, (RO)v.y);
    }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    const Geo g = sh.gcol();
    eng::dispatch<C>(g, sh.fast() && Lout.lgw == lg_tile<C>(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, out, Lout, it << sh.lgS, sh.lgS, scale};
      eng::run_fix<LGN, true, INV>(g, b, tw, f);
    });
  }
};

// generic row transform of a complex field (layouts at runtime; one-time use)
template <typename R, bool INV> struct RowsOp : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  Shape<R> sh;
  const C* in;
  Lay Lin, Lout;
  C* out;
  const C* tw;
  LS_D void prefetch(int it, int, C* b, C*) const {
    eng::gather_rect<sizeof(C)>(b, in, Lin, it << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  template <int LGN> struct F {
    const C* b;
    C* out;
    Lay L;
    int y0, lgn;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const { return b[nat_row<LGN, ST>(seq, j, r, lgn)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { out[L.at(y0 + seq, j + r * ST)] = v; }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    const Geo g = sh.grow();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, out, Lout, it << sh.lgR, sh.lgW};
      eng::run_fix<LGN, false, INV>(g, b, tw, f);
    });
  }
};

// ---------------------------------------------------------------------------
// per-set parameters of the kernel-looping passes

template <typename R> struct SetArgs {
  using C = typename CT<R>::C;
  int nsets;
  int nk[2];
  const C* spec[2];      // nk x field, column-tiled
  C* T[2];               // nk x field, column-tiled: T_k, later U_k
  C* A[2];               // nk x field, row-major: A_k
  R* I[2];               // row-major intensity per set
  const R* gate[2];      // row-major gate per set
  C* V[2];               // column-tiled adjoint accumulator per set
  R w[2][kMaxK];         // kernel weights (sigma_k)
  R* Ipart;              // kernel groups: per-group partial I / V, [set][group][H*W]
  C* Vpart;
  unsigned* tick;        // [pass (F2, A2)][set][block] last-arriving tickets
  int tick_stride;       // tickets per (pass, set)
};

// Kernel groups: the item of the last group to finish a (set, block) sums the
// groups' partials in group order (deterministic whatever the arrival order)
// into the set's output and re-arms the ticket.  Called by every thread.
template <typename T>
LS_D void group_combine(const T* part, size_t pstride, T* out, size_t off, int rows, int width, int ld, int G,
                        unsigned* ticket) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == (unsigned)(G - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int cnt = rows * width;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const size_t p = off + (size_t)(i / width) * ld + (i % width);
    T acc = __ldcg(&part[p]);
    for (int g = 1; g < G; ++g) acc = acc + __ldcg(&part[(size_t)g * pstride + p]);
    out[p] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0;
}

// F1: T_k = IFFT_y(M^ . H_k) / (HW); the item's M^ values stay in registers
template <typename R> struct F1Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { C mh[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* mhat;
  R scale;
  const C* tw;
  int lgnt;
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnt)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnt) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D const C* field(int it, int k) const { return a.spec[set_of(it, lgnt)] + (size_t)k * fsz(); }  // column-tiled input
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnt), t = it & ((1 << lgnt) - 1);
    eng::gather_rect<sizeof(C)>(b, a.spec[set] + (size_t)k * fsz(), sh.ct(), 0, sh.lgH, t << sh.lgS, sh.lgS);
  }
  // the item's M^ values, pre-multiplied by the IFFT's 1/(HW) (a power of
  // two: exact), so the per-kernel product needs no extra scaling
  template <int LGN> struct LoadM {
    State& S;
    const C* mhat;
    Lay L;
    int x0;
    R scale;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      S.mh[slot] = __ldg(&mhat[ct_col<LGN, ST, C>(L, j, r, x0 + seq)]) * scale;
    }
  };
  LS_D void begin(State& S, int it, C*) const {
    const int t = it & ((1 << lgnt) - 1);
    eng::dispatch<C>(sh.gcol(), sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) eng::for_first_slots<LGN, true, C>(LoadM<LGN>{S, mhat, sh.ct(), t << sh.lgS, scale});
    });
  }
  template <int LGN> struct F {
    const C* b;
    const State& S;
    const C* mhat;  // generic path only
    C* out;
    Lay L, Lm;
    int x0, lgS;
    R scale;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      const C x = b[nat_col<LGN, ST, C>(seq, j, r, lgS)];
      if constexpr (LGN > 0) return cmul(S.mh[slot], x);
      else return cmul(mhat[Lm.at(j, x0 + seq)], x) * scale;
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) {
      gstore(out[ct_col<LGN, ST, C, kLgTileT>(L, j, r, x0 + seq)], v);
    }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnt), t = it & ((1 << lgnt) - 1);
    const Geo g = sh.gcol();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, S, mhat, a.T[set] + (size_t)k * fsz(), sh.ctT(), sh.ct(), t << sh.lgS, sh.lgS, scale};
      eng::run_fix<LGN, true, true>(g, b, tw, f);
    });
  }
};

// F2: A_k = IFFT_x T_k (row-major) and I_set = sum_k w_k |A_k|^2, accumulated
//     in registers and written once per item
template <typename R> struct F2Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { R acc[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnb)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnb) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnb), yb = it & ((1 << lgnb) - 1);
    eng::gather_rect<sizeof(C)>(b, a.T[set] + (size_t)k * fsz(), sh.ctT(), yb << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  LS_D void begin(State& S, int, C*) const {
#pragma unroll
    for (int i = 0; i < P; ++i) S.acc[i] = (R)0;
  }
  template <int LGN> struct F {
    const C* b;
    State& S;
    R w;
    C* A;  // row-major field k
    int y0, lgn, W;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const { return b[nat_row<LGN, ST>(seq, j, r, lgn)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int slot) {
      S.acc[slot] += w * (v.x * v.x + v.y * v.y);
      gstore(A[rm_row<LGN, ST>(W, y0 + seq, j, r)], v);
    }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnb), yb = it & ((1 << lgnb) - 1);
    const Geo g = sh.grow();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, S, a.w[set][k], a.A[set] + (size_t)k * fsz(), yb << sh.lgR, sh.lgW, sh.W};
      eng::run_fix<LGN, false, true>(g, b, tw, f);
    });
  }
  template <int LGN> struct WriteI {
    R* I;
    const State& S;
    int y0, W;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      I[rm_row<LGN, ST>(W, y0 + seq, j, r)] = S.acc[slot];
    }
  };
  LS_D void end(State& S, int it, C*, C*) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    const Geo g = sh.grow();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      eng::for_last_slots<LGN, false, C>(g, WriteI<LGN>{a.I[set], S, y0, sh.W});
    });
  }
};

// A1: U_k = FFT_x(gate . A_k) -> column-tiled, over T_k; the item's gate
//     values stay in registers
template <typename R> struct A1Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { R g[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnb)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnb) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnb), yb = it & ((1 << lgnb) - 1);
    eng::gather_rect<sizeof(C)>(b, a.A[set] + (size_t)k * fsz(), sh.rm(), yb << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  template <int LGN> struct LoadG {
    State& S;
    const R* gate;
    int y0, W;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      S.g[slot] = __ldg(&gate[rm_row<LGN, ST>(W, y0 + seq, j, r)]);
    }
  };
  LS_D void begin(State& S, int it, C*) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    eng::dispatch<C>(sh.grow(), sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) eng::for_first_slots<LGN, false, C>(LoadG<LGN>{S, a.gate[set], y0, sh.W});
    });
  }
  template <int LGN> struct F {
    const C* b;
    const State& S;
    const R* gate;  // generic path only
    C* out;
    Lay L;
    int y0, lgn, W;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      const C x = b[nat_row<LGN, ST>(seq, j, r, lgn)];
      if constexpr (LGN > 0) return x * S.g[slot];
      else return x * gate[(size_t)(y0 + seq) * W + j];
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { gstore(out[ct_row<LGN, ST, C>(L, y0 + seq, j, r)], v); }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnb), yb = it & ((1 << lgnb) - 1);
    const Geo g = sh.grow();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, S, a.gate[set], a.T[set] + (size_t)k * fsz(), sh.ct(), yb << sh.lgR, sh.lgW, sh.W};
      eng::run_fix<LGN, false, false>(g, b, tw, f);
    });
  }
};

// A2: V_set = IFFT_y( sum_k w_k conj(H_k) . FFT_y U_k )
template <typename R, bool VS = false> struct A2Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { C acc[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnt;
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnt)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnt) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D const C* field(int it, int k) const { return a.T[set_of(it, lgnt)] + (size_t)k * fsz(); }  // column-tiled U_k
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnt), t = it & ((1 << lgnt) - 1);
    eng::gather_rect<sizeof(C)>(b, a.T[set] + (size_t)k * fsz(), sh.ct(), 0, sh.lgH, t << sh.lgS, sh.lgS);
  }
  LS_D void begin(State& S, int, C*) const {
#pragma unroll
    for (int i = 0; i < P; ++i) S.acc[i] = cmk((R)0, (R)0);
  }
  template <int LGN> struct LoadH {
    C (&h)[P];
    const C* spec;
    Lay L;
    int x0;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      h[slot] = __ldg(&spec[ct_col<LGN, ST, C>(L, j, r, x0 + seq)]);
    }
  };
  template <int LGN> struct F {
    const C* b;
    State& S;
    const C (&h)[P];
    R w;
    int lgS;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const { return b[nat_col<LGN, ST, C>(seq, j, r, lgS)]; }
    template <int ST> LS_D void store(int, int, int, C v, int slot) { S.acc[slot] = S.acc[slot] + cmulc(v, h[slot]) * w; }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    const int set = set_of(it, lgnt), t = it & ((1 << lgnt) - 1);
    const Geo g = sh.gcol();
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      C h[P];
      eng::for_last_slots<LGN, true, C>(g, LoadH<LGN>{h, a.spec[set] + (size_t)k * fsz(), sh.ct(), t << sh.lgS});
      F<LGN> f{b, S, h, a.w[set][k], sh.lgS};
      eng::run_fix<LGN, true, false>(g, b, tw, f);
    });
  }
  template <int LGN> struct PutAcc {
    C* b;
    const State& S;
    int lgS;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      b[nat_col<LGN, ST, C>(seq, j, r, lgS)] = S.acc[slot];
    }
  };
  // V_set is written row-major (once per item), so the A3 row pass reads
  // whole contiguous row blocks
  // Split plans (VS): virtual column -> (column, plane), V stored
  // row-major with plane c's rows at c * 2048 (the A3 row pass combines them)
  int vs_lgt = -1, vs_W = 0;
  template <int LGN> struct FOut {
    const C* b;
    C* out;
    int W;
    int x0, lgS;
    int vsl, Wp;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const { return b[nat_col<LGN, ST, C>(seq, j, r, lgS)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) {
      if constexpr (VS) {
        const int xv = x0 + seq;
        out[(size_t)((vs_plane(xv, vsl) << kLgVsM) + j + r * ST) * Wp + vs_col(xv, vsl)] = v;
      } else {
        out[rm_col<LGN, ST>(W, j, r, x0 + seq)] = v;
      }
    }
  };
  LS_D void end(State& S, int it, C* b, C*) const {
    const int set = set_of(it, lgnt), t = it & ((1 << lgnt) - 1);
    const Geo g = sh.gcol();
    const size_t n = (size_t)sh.H * sh.W;
    C* dst = lgg ? a.Vpart + (size_t)((set << lgg) + grp_of(it, lgnt)) * n : a.V[set];
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      eng::for_last_slots<LGN, true, C>(g, PutAcc<LGN>{b, S, sh.lgS});
      __syncthreads();
      FOut<LGN> f{b, dst, sh.W, t << sh.lgS, sh.lgS, vs_lgt, vs_W};
      eng::run_fix<LGN, true, true>(g, b, tw, f);
    });
    __syncthreads();
    if (lgg)  // the IFFT is linear: the groups' transformed partials sum to V
      group_combine(a.Vpart + (size_t)(set << lgg) * n, n, a.V[set], (size_t)(t << sh.lgS), sh.H, 1 << sh.lgS, sh.W,
                    1 << lgg, &a.tick[(2 + set) * a.tick_stride + t]);
  }
};

// A3: out = scale * Re IFFT_x(V_0 [+ V_1]) (f64 row-major) + CG dot partials per CTA
template <typename R, bool VS = false> struct A3Op : OpBase {
  using C = typename CT<R>::C;
  struct State { double acc[2]; };
  Shape<R> sh;
  const C* V0;
  const C* V1;
  const C* tw;
  double scale;
  double* out;
  const double* vp;
  double* dots;
  int ix0, ix1;  // dots over columns [ix0, ix1) ...
  int iy0, iy1;  // ... and rows [iy0, iy1)
  int vs_lgq = -1;  // split plan: V rows in plane order, combined before the transform
  LS_D void prefetch(int it, int, C* b, C*) const {
    if constexpr (VS) {  // plane rows c * 2048 + n2_0 + q: four strips of Q rows
      for (int c = 0; c < 4; ++c)
        eng::gather_rect<sizeof(C)>(b + ((c << vs_lgq) << sh.lgW), V0, sh.rm(),
                                    vs_plane_row(c << vs_lgq, vs_lgq, it << vs_lgq), vs_lgq, 0, sh.lgW);
      return;
    }
    eng::gather_rect<sizeof(C)>(b, V0, sh.rm(), it << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  template <int LGN> struct F {
    const C* b;
    const C* v1;  // second accumulator, read directly (row-major, coalesced)
    Lay L;
    double scale;
    double* out;
    const double* vp;
    State& S;
    int y0, lgn, W, ix0, ix1, iy0, iy1;
    int lgq;  // split plan: buffer row -> natural row (v1 already folded in)
    LS_D int row(int seq) const { return VS ? vs_row(seq, lgq, y0) : y0 + seq; }
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      const C x = b[nat_row<LGN, ST>(seq, j, r, lgn)];
      if constexpr (LGN > 0) return v1 ? x + __ldg(&v1[rm_row<LGN, ST>(W, y0 + seq, j, r)]) : x;
      else return v1 ? x + __ldg(&v1[(size_t)(y0 + seq) * W + j]) : x;
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) {
      const int y = row(seq);
      const size_t p = rm_row<LGN, ST>(W, y, j, r);
      const double val = scale * (double)v.x;
      out[p] = val;
      const int x = j + r * ST;
      if (vp && x >= ix0 && x < ix1 && y >= iy0 && y < iy1) {
        const double q = vp[p];
        S.acc[0] += val * (val - q);
        S.acc[1] += q * q;
      }
    }
  };
  LS_D void step(State& S, int it, int, C* b, C*) const {
    const Geo g = sh.grow();
    if constexpr (VS) {
      vs_inv_combine(b, sh.lgW, vs_lgq, it << vs_lgq, tw, sh.twsH, V1);
      __syncthreads();
    }
    const C* v1 = VS ? nullptr : V1;
    const int y0 = VS ? it << vs_lgq : it << sh.lgR;
    eng::dispatch<C>(g, sh.fast(), [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      F<LGN> f{b, v1, sh.rm(), scale, out, vp, S, y0, sh.lgW, sh.W, ix0, ix1, iy0, iy1, vs_lgq};
      eng::run_fix<LGN, false, true>(g, b, tw, f);
    });
  }
  LoopTail tail;  // st != nullptr: Polak-Ribiere control in the last CTA (control.cuh)
  LS_D void finish(State& S, double* red) const {
    if (!vp) return;
    __syncthreads();
    block_sum<2>(S.acc, red);
    if (threadIdx.x == 0) {
      dots[2 * blockIdx.x] = S.acc[0];
      dots[2 * blockIdx.x + 1] = S.acc[1];
    }
    if (tail.st && last_block(&tail.st->ticket[1], red)) {
      after_grad_body(dots, gridDim.x, tail.restart_every, tail.st, red);
      release_ticket(&tail.st->ticket[1]);
    }
  }
};

// ===========================================================================
// TMA variants of the four kernel-looping passes.
//
// Measured on B200: the TMA engine's cost grows with the number of box rows,
// so a whole-tile column item (one contiguous 64 KB block) is fetched by one
// 1-D bulk copy rather than 2048 tensor-box rows of 32 B (F1 661 -> 581 us,
// A2 653 -> 566 us).  Row items keep natural [row][x] boxes: a row-group box
// (4 rows of a tile = 128 B per box row) needs a swizzled [tile][row] shared
// layout whose half-warp reads conflict 2-way, which measured slower.
//
// Same arithmetic as F1Op / F2Op / A1Op / A2Op; operands arrive by TMA
// (1-D bulk copies of contiguous rows / tiles, 4-D tensor copies for the
// column-tiled fields) into a 3-slot ring guarded by mbarriers, and the
// per-kernel output tile is written to shared memory by the last butterfly
// stage and streamed out by TMA stores.  Slot roles at step q: q%3 is being
// transformed, (q+1)%3 is being filled, (q+2)%3 == (q-1)%3 drains the
// previous step's stores.  No thread issues per-element global loads or
// stores of the streamed fields, so the LSU only serves the exchange.

// field layout seen by TMA: 8-byte words, dims {w*EW, W/w, H, NK}
struct TmaField {
  const void* base;
  int lgw;   // tile width (elements)
  int ew;    // 8-byte words per element (1: complex64, 2: complex128)
};

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// map over NK column-tiled fields of H x W elements; box in words/tiles/rows
inline CUtensorMap make_field_map(const TmaField& f, int H, int W, int NK, unsigned b0, unsigned b1, unsigned b2) {
  const uint64_t w = 1ull << f.lgw, es = 8ull * f.ew;
  cuuint64_t dim[4] = {w * f.ew, (uint64_t)W >> f.lgw, (uint64_t)H, (uint64_t)NK};
  cuuint64_t stride[3] = {(uint64_t)H * w * es, w * es, (uint64_t)H * W * es};
  cuuint32_t box[4] = {b0, b1, b2, 1};
  cuuint32_t est[4] = {1, 1, 1, 1};
  CUtensorMap m;
  CUresult r = tmap_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(f.base), dim, stride, box, est,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// TMA path usable for the row passes (F2, A1) / the column passes (F1, A2)
// of this geometry: compile-time FFT geometry along that axis, and for
// columns a slab of at least 16 B per tile row (a TMA box row).  The axes are
// independent: an 8192-point column slab is 8 B wide (one complex64 column)
// and stays on the cp.async path while the 8192-point rows stream by TMA.
inline bool tma_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("LSOPC_B200_NO_TMA");
    return e && e[0] == '1';
  }();
  return off;
}
template <typename R> bool tma_ok_rows(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  constexpr int LGE = eng::lg_full<C>();
  return !tma_disabled() && sh.fast() && sh.lgW >= eng::kFastMinLgn && sh.lgR == LGE - sh.lgW;
}
template <typename R> bool tma_ok_cols(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  constexpr int LGE = eng::lg_full<C>();
  if (tma_disabled() || !sh.fast() || sh.lgH < eng::kFastMinLgn || sh.lgS != LGE - sh.lgH) return false;
  const int ew = sizeof(C) / 8;
  const int S = 1 << sh.lgS, w = 1 << lg_tile<C>();
  return std::min(S, w) * ew * 8 >= 16 && S % std::min(S, w) == 0;
}

template <typename R, class Op>
__global__ void __launch_bounds__(eng::cta_threads<typename CT<R>::C>(), 1) k_pass_tma(const __grid_constant__ Op op,
                                                                                       StopFlag stop) {
  using C = typename CT<R>::C;
#if !defined(LSB_EXP_NOSTORE) && !defined(LSB_EXP_NOGATHER) && !defined(LSB_EXP_NOTMA)
  if (stop && *stop) return;
#endif
  extern __shared__ __align__(128) unsigned char smraw[];
  C* const base = reinterpret_cast<C*>(smraw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + 3 * (size_t)op.bufE * sizeof(C));  // 3 ring + 2 side
  typename Op::State S{};
  if ((int)blockIdx.x >= op.nitems) return;
  const bool leader = threadIdx.x == 0;
  if (leader) {
    for (int i = 0; i < 5; ++i) tma::mbar_init(&bar[i], 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  auto advance = [&](int& it, int& st) {
    if (++st == op.steps(it)) { st = 0; it += gridDim.x; }
  };
  int it = blockIdx.x, st = 0;
  int nit = it, nst = st;  // next step to load
  if (leader) {
#ifdef LSB_EXP_NOTMA  // experiment builds only: on-chip work without data movement
    tma::mbar_expect_tx(&bar[0], 0);
#else
    tma::mbar_expect_tx(&bar[0], op.load_bytes());
    op.load(nit, op.kbase(nit) + nst, base, &bar[0]);
#endif
  }
  advance(nit, nst);
  // side operand of step q (kSideLoad ops): in the idle slot (q+2)%3, own
  // mbarrier 3 + (q&1).  It is issued one step ahead, from inside step q-1
  // once that step's last butterfly stage has read its slot (q-1)%3 ==
  // (q+2)%3; only the first step of an item issues its own (the previous
  // step's slot is then still busy with the item's closing transform).
  bool side_pending = Op::kSideLoad;
  for (unsigned q = 0;; ++q) {
    const int slot = q % 3, nslot = (q + 1) % 3;
    C* const side = base + ((q + 2) % 3) * op.bufE;  // idle slot when the op stores nothing
    if (leader && nit < op.nitems) {
      if (Op::kStores) tma::bulk_wait_read<1>();  // slot nslot held the stores of step q-2
#ifdef LSB_EXP_NOTMA
      tma::mbar_expect_tx(&bar[nslot], 0);
#else
      tma::mbar_expect_tx(&bar[nslot], op.load_bytes());
      op.load(nit, op.kbase(nit) + nst, base + nslot * op.bufE, &bar[nslot]);
#endif
    }
    if constexpr (Op::kSideLoad) {
      if (leader && side_pending) {
#ifdef LSB_EXP_NOTMA
        tma::mbar_expect_tx(&bar[3 + (q & 1)], 0);
#else
        tma::mbar_expect_tx(&bar[3 + (q & 1)], op.load_bytes());
        op.side_load(it, op.kbase(it) + st, side, &bar[3 + (q & 1)]);
#endif
      }
    }
    tma::mbar_wait(&bar[slot], (q / 3) & 1);
    C* const cur = base + slot * op.bufE;
    if (st == 0) op.begin(S, it, cur);
    if constexpr (Op::kSideLoad) {
      const bool item_end = st == op.steps(it) - 1;
      op.step_side(S, it, op.kbase(it) + st, cur, side, q, bar, !item_end);
      side_pending = item_end;
    } else {
      op.step(S, it, op.kbase(it) + st, cur, side, q);
    }
    if (Op::kStores) {
      tma::fence_async_smem();
      __syncthreads();
      if (leader) {
#ifndef LSB_EXP_NOTMA
        op.store(it, op.kbase(it) + st, cur);
#endif
        tma::bulk_commit();
      }
    } else {
      __syncthreads();
    }
    if (st == op.steps(it) - 1) op.end(S, it, cur, cur);
    if (nit < op.nitems) advance(nit, nst);
    advance(it, st);
    if (it >= op.nitems) break;
  }
  if (leader && Op::kStores) tma::bulk_wait<0>();
  op.finish(S, reinterpret_cast<double*>(smraw));
}

// F1 on tall grids (k_pass_cluster): the transformed column stays in shared
// memory; the cluster gathers each CTA's row quarter of the 4 columns back
// through distributed shared memory and TMA stores it into the T_k tiles.
template <typename R> struct F1COp : F1Op<R> {
  using C = typename CT<R>::C;
  using State = typename F1Op<R>::State;
  static constexpr bool kGatherOut = true;
  alignas(64) CUtensorMap tmap_T;  // T fields, 4-column x 256-row boxes
  int koff[2];
  template <int LGN> struct FS {
    C* b;
    const State& S;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      return cmul(S.mh[slot], b[nat_col<LGN, ST, C>(seq, j, r, 0)]);
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { b[nat_col<LGN, ST, C>(seq, j, r, 0)] = v; }
  };
  LS_D void step_smem(State& S, C* b) const {
    const Geo g = this->sh.gcol();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        FS<LGN> f{b, S};
        eng::run_fix<LGN, true, true>(g, b, this->tw, f);
      }
    });
  }
  // rows [row0, row0 + rows) of the tile's 4 columns (natural [row][4]) -> T_k
  LS_D void store_quarter(int itl, int k, int x0, int row0, int rows, const C* src) const {
    const int set = itl >> this->lgnt;
    constexpr int w = 1 << kLgTileT;
    for (int b = 0; b * 256 < rows; ++b)
      tma::tensor_s2g(&tmap_T, x0 & (w - 1), x0 >> kLgTileT, row0 + b * 256, k + koff[set], src + (size_t)b * 256 * 4);
  }
};

// ---------------------------------------------------------------------------
// Column passes on tall grids wider than the split plan takes (8192-point
// columns with W > 2048 fp32, e.g. a whole 8192^2 tile as one grid; or with
// LSOPC_B200_NO_VSPLIT=1 -- split plans run 2048-point columns): a column
// item is one complex64 column, an 8-byte-wide slab of the 4-wide tiles, too
// narrow for TMA; per-element cp.async / stores make the pass LSU-bound.
// Here the four CTAs of a cluster take the four columns of one tile: each
// CTA fetches a 64 KB row quarter of the tile (all four columns) with one
// 1-D bulk copy, then the cluster scatters the quarters column-wise through
// distributed shared memory, so each CTA holds its whole column; the
// transform itself is the single-column op (F1Op / A2Op) unchanged.
// Shared memory: the op's exchange buffer (the column) and two quarter
// buffers, the next step's quarter streaming in while this step transforms.
constexpr int kClusterCols = 4;
template <class Op, class = void> struct has_gather_out : std::false_type {};
template <class Op> struct has_gather_out<Op, std::void_t<decltype(Op::kGatherOut)>> : std::true_type {};

template <typename R, class Op>
__global__ void __cluster_dims__(kClusterCols, 1, 1) __launch_bounds__(eng::cta_threads<typename CT<R>::C>(), 1)
k_pass_cluster(const __grid_constant__ Op op, StopFlag stop, int ntiles, int nsets) {
  using C = typename CT<R>::C;
  using Vec = typename std::conditional<sizeof(C) == 8, float2, double2>::type;
  if (stop && *stop) return;  // uniform across the cluster
  extern __shared__ __align__(128) unsigned char smraw[];
  C* const col = reinterpret_cast<C*>(smraw);
  const size_t colE = (size_t)op.bufE;                       // elements (rounded to 128 B)
  C* const quart = col + colE;                               // 2 x [H/4][4]
  const int qrows = op.sh.H / kClusterCols, qE = qrows * kClusterCols;
  uint64_t* bar = reinterpret_cast<uint64_t*>(quart + 2 * (size_t)qE);
  const unsigned rank = tma::cluster_rank();
  const int cid = blockIdx.x / kClusterCols, ncl = gridDim.x / kClusterCols;
  const int nit = ntiles * nsets;
  const bool leader = threadIdx.x == 0;
  if (leader) {
    tma::mbar_init(&bar[0], 1);
    tma::mbar_init(&bar[1], 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  // the single-column op's item for (tile item, rank): column 4 t + rank of the set
  auto legacy = [&](int it4) {
    const int set = it4 / ntiles, t = it4 - set * ntiles;
    return (set << op.lgnt) | (kClusterCols * t + (int)rank);
  };
  auto issue = [&](int it4, int k, int slot) {
    const int t = it4 % ntiles;
    const C* src = op.field(legacy(it4), k) + ((size_t)t * op.sh.H + (size_t)rank * qrows) * kClusterCols;
    tma::mbar_expect_tx(&bar[slot], (unsigned)(qE * sizeof(C)));
    tma::bulk_g2s(quart + (size_t)slot * qE, src, (unsigned)(qE * sizeof(C)), &bar[slot]);
  };
  if (cid >= nit) return;  // whole clusters idle together
  typename Op::State S{};
  int it4 = cid, st = 0;
  if (leader) issue(it4, 0, 0);
  for (unsigned q = 0;; ++q) {
    const int slot = q & 1;
    int nit4 = it4, nst = st + 1;  // next step
    if (nst == op.steps(legacy(it4))) {
      nst = 0;
      nit4 += ncl;
    }
    tma::mbar_wait(&bar[slot], (q >> 1) & 1);
    // every CTA's quarter has landed and every CTA is done with its column
    tma::cluster_sync();
    {
      const C* qb = quart + (size_t)slot * qE;
      unsigned dst[kClusterCols];
#pragma unroll
      for (int c = 0; c < kClusterCols; ++c) dst[c] = tma::cluster_map(col, c);
      for (int i = threadIdx.x; i < qrows; i += blockDim.x) {
        const Vec* row = reinterpret_cast<const Vec*>(qb + (size_t)i * kClusterCols);
        const unsigned off = (unsigned)(((size_t)rank * qrows + i) * sizeof(C));
#pragma unroll
        for (int c = 0; c < kClusterCols; ++c) tma::st_cluster(dst[c] + off, row[c]);
      }
    }
    tma::cluster_sync();  // columns complete; this step's quarters are free
    if (leader && nit4 < nit) {
      if constexpr (has_gather_out<Op>::value) tma::bulk_wait_read<0>();  // slot ^ 1 held step q-1's output
      issue(nit4, nst, slot ^ 1);
    }
    const int itl = legacy(it4);
    if (st == 0) op.begin(S, itl, col);
    if constexpr (has_gather_out<Op>::value) {
      op.step_smem(S, col);
      tma::cluster_sync();  // every column transformed
      // gather this CTA's row quarter of the 4 columns into the free quarter slot
      C* ob = quart + (size_t)slot * qE;
      unsigned srcs[kClusterCols];
#pragma unroll
      for (int c = 0; c < kClusterCols; ++c) srcs[c] = tma::cluster_map(col, c);
      for (int i = threadIdx.x; i < qrows; i += blockDim.x) {
        const unsigned off = (unsigned)(((size_t)rank * qrows + i) * sizeof(C));
        Vec v[kClusterCols];
#pragma unroll
        for (int c = 0; c < kClusterCols; ++c) tma::ld_cluster(srcs[c] + off, v[c]);
#pragma unroll
        for (int c = 0; c < kClusterCols; ++c) reinterpret_cast<Vec*>(ob + (size_t)i * kClusterCols)[c] = v[c];
      }
      tma::fence_async_smem();
      __syncthreads();
      if (leader) {
        const int t = it4 % ntiles;
        op.store_quarter(itl, st, kClusterCols * t, (int)rank * qrows, qrows, ob);
        tma::bulk_commit();
      }
    } else {
      op.step(S, itl, st, col, nullptr);
    }
    if (st == op.steps(itl) - 1) op.end(S, itl, col, col);
    it4 = nit4;
    st = nst;
    if (it4 >= nit) break;
  }
  if (leader && has_gather_out<Op>::value) tma::bulk_wait<0>();
  // no CTA may exit while a sibling could still write into its shared memory
  tma::cluster_sync();
}

// natural (dense) output position in a buffer; the TMA store box order
template <int LGN, int STRIDE, typename C, bool COLS> LS_D int nat_out(int seq, int j, int r) {
  if constexpr (COLS) return nat_col<LGN, STRIDE, C>(seq, j, r, 0);
  else return nat_row<LGN, STRIDE>(seq, j, r, 0);
}

// TMaskRows: M~ = FFT_x(mask) (K1 rows).  The item's mask rows (u8, or f64
// mask / phi) arrive by one 1-D bulk copy; the transform reads them from
// shared memory in the first stage; M~ rows leave by per-row tensor boxes
// into the column-tiled scratch (like TA1's U_k stores).
template <typename R, bool VS = false> struct TMaskRowsOp : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  static constexpr bool kStores = true;
  static constexpr bool kSideLoad = false;
  Shape<R> sh;
  const void* src;
  int kind;
  const C* tw;
  alignas(64) CUtensorMap tmap_out;  // M~ (one column-tiled field), row boxes
  int vs_lgq = -1;                   // split plan: log2 Q (rows per plane in an item)
  LS_D unsigned load_bytes() const { return (unsigned)((sh.W << sh.lgR) * (kind == SRC_U8 ? 1 : 8)); }
  LS_D void load(int it, int, C* dst, uint64_t* bar) const {
    const int es = kind == SRC_U8 ? 1 : 8;
    const unsigned char* s = static_cast<const unsigned char*>(src);
    if constexpr (VS) {  // natural rows n2_0 + q + 2048 m: four strips of Q rows
      const unsigned qb = (unsigned)(sh.W << vs_lgq) * es;
      for (int m = 0; m < 4; ++m)
        tma::bulk_g2s(reinterpret_cast<unsigned char*>(dst) + m * qb,
                      s + (size_t)vs_row(m << vs_lgq, vs_lgq, it << vs_lgq) * sh.W * es, qb, bar);
      return;
    }
    tma::bulk_g2s(dst, s + ((size_t)it << sh.lgR) * sh.W * es, load_bytes(), bar);
  }
  LS_D void store(int it, int, const C* src_s) const {
    constexpr int LGT = lg_tile<C>();
    const int y0 = it << sh.lgR, tiles = sh.W >> LGT, bt = tiles < 256 ? tiles : 256;
    for (int r = 0; r < (1 << sh.lgR); ++r) {
      const int y = VS ? vs_plane_row(r, vs_lgq, it << vs_lgq) : y0 + r;
      for (int b = 0; b * bt < tiles; ++b)
        tma::tensor_s2g(&tmap_out, 0, b * bt, y, 0, src_s + (r << sh.lgW) + ((b * bt) << LGT));
    }
  }
  template <int LGN> struct F {
    C* b;
    int kind;
    template <int ST> LS_D C load(int seq, int j, int r, int) const {
      const int p = nat_row<LGN, ST>(seq, j, r, 0);
      R m;
      if (kind == SRC_U8) {
        m = (R)reinterpret_cast<const unsigned char*>(b)[p];
      } else {
        const double v = reinterpret_cast<const double*>(b)[p];
        m = kind == SRC_PHI ? (R)(v <= 0.0) : (R)v;
      }
      return cmk(m, (R)0);
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { b[nat_out<LGN, ST, C, false>(seq, j, r)] = v; }
  };
  LS_D void step(State&, int it, int, C* b, C*, unsigned) const {
    const Geo g = sh.grow();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b, kind};
        eng::run_fix<LGN, false, false>(g, b, tw, f);
      }
    });
    if constexpr (VS) {
      __syncthreads();
      vs_fwd_combine(b, sh.lgW, vs_lgq, it << vs_lgq, tw, sh.twsH);
    }
  }
};

// TCols: out = FFT_y(in) of whole-tile column items (K1 columns): one 1-D bulk
// copy in, one out
template <typename R> struct TColsOp : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  static constexpr bool kStores = true;
  static constexpr bool kSideLoad = false;
  Shape<R> sh;
  const C* in;
  C* out;
  const C* tw;
  LS_D unsigned load_bytes() const { return (unsigned)((sh.H << sh.lgS) * sizeof(C)); }
  LS_D size_t tile_off(int it) const { return ((size_t)it << sh.lgS) * sh.H; }  // whole tiles: lgS == lgT
  LS_D void load(int it, int, C* dst, uint64_t* bar) const { tma::bulk_g2s(dst, in + tile_off(it), load_bytes(), bar); }
  LS_D void store(int it, int, const C* src_s) const { tma::bulk_s2g(out + tile_off(it), src_s, load_bytes()); }
  template <int LGN> struct F {
    C* b;
    template <int ST> LS_D C load(int seq, int j, int r, int) const { return b[nat_col<LGN, ST, C>(seq, j, r, 0)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { b[nat_out<LGN, ST, C, true>(seq, j, r)] = v; }
  };
  LS_D void step(State&, int, int, C* b, C*, unsigned) const {
    const Geo g = sh.gcol();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b};
        eng::run_fix<LGN, true, false>(g, b, tw, f);
      }
    });
  }
};

// TF1: T_k = IFFT_y(M^ . H_k)/(HW); H_k tile in by TMA, T_k slab out by TMA
template <typename R, bool VS = false> struct TF1Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  static constexpr bool kStores = true;
  static constexpr bool kSideLoad = false;
  using State = typename F1Op<R>::State;
  Shape<R> sh;
  SetArgs<R> a;
  const C* mhat;
  R scale;
  const C* tw;
  int lgnt;
  int spec_lgw;                    // tile width of the spectra layout
  alignas(64) CUtensorMap tmap_spec;   // spectra of set 0, column-item boxes
  alignas(64) CUtensorMap tmap_spec1;  // spectra of set 1
  alignas(64) CUtensorMap tmap_T;     // T fields, column-item boxes
  int koff[2];                      // first kernel index of each set in the stacked maps
  int vs_lgt = -1;                  // split plan: the item's virtual columns map to (column, plane) (tmap_T physical)
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnt)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnt) * kpg; }
  LS_D unsigned load_bytes() const { return (unsigned)((sh.H << sh.lgS) * sizeof(C)); }
  LS_D void load(int it, int k, C* dst, uint64_t* bar) const {
    const int set = set_of(it, lgnt), x0 = (it & ((1 << lgnt) - 1)) << sh.lgS;
    if (spec_lgw == sh.lgS) {  // the item is one whole tile: a contiguous block, one 1-D bulk copy
      tma::bulk_g2s(dst, a.spec[set] + (size_t)k * sh.H * sh.W + ((size_t)(x0 >> spec_lgw) * sh.H << spec_lgw),
                    load_bytes(), bar);
      return;
    }
    const CUtensorMap* m = set ? &tmap_spec1 : &tmap_spec;
    col_boxes(x0, k, spec_lgw, [&](int c0, int c1, int c2, int kk, int off) {
      tma::tensor_g2s(dst + off, m, c0, c1, c2, kk, bar);
    });
  }
  LS_D void store(int it, int k, const C* src) const {
    const int set = set_of(it, lgnt), xv = (it & ((1 << lgnt) - 1)) << sh.lgS;
    const int x0 = VS ? vs_col(xv, vs_lgt) : xv, y0 = VS ? vs_plane(xv, vs_lgt) << kLgVsM : 0;
    col_boxes(x0, k + koff[set], kLgTileT, [&](int c0, int c1, int c2, int kk, int off) {
      tma::tensor_s2g(&tmap_T, c0, c1, y0 + c2, kk, src + off);
    });
  }
  // boxes of a column item: {min(S,w) words-per-elem, S/w tiles, 256 rows}
  template <class Fn> LS_D void col_boxes(int x0, int kk, int lgw, Fn&& fn) const {
    const int ew = sizeof(C) / 8, w = 1 << lgw, S = 1 << sh.lgS;
    const int rows = sh.H < 256 ? sh.H : 256;
    for (int b = 0; b * rows < sh.H; ++b) fn((x0 & (w - 1)) * ew, x0 >> lgw, b * rows, kk, b * rows * S);
  }
  LS_D void begin(State& S, int it, C*) const {
    const int t = it & ((1 << lgnt) - 1);
    eng::dispatch<C>(sh.gcol(), true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0)
        eng::for_first_slots<LGN, true, C>(typename F1Op<R>::template LoadM<LGN>{S, mhat, sh.ct(), t << sh.lgS, scale});
    });
  }
  template <int LGN> struct F {
    C* b;
    const State& S;
    R scale;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      return cmul(S.mh[slot], b[nat_col<LGN, ST, C>(seq, j, r, 0)]);
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { b[nat_out<LGN, ST, C, true>(seq, j, r)] = v; }
  };
  LS_D void step(State& S, int, int, C* b, C*, unsigned) const {
    const Geo g = sh.gcol();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b, S, scale};
        eng::run_fix<LGN, true, true>(g, b, tw, f);
      }
    });
  }
};

// TF2: A_k = IFFT_x T_k (out by 1-D bulk), I_set = sum w |A_k|^2 (registers)
template <typename R, bool VS = false> struct TF2Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  static constexpr bool kStores = true;
  static constexpr bool kSideLoad = false;
  using State = typename F2Op<R>::State;
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  int split_lgq;                   // >= 0: T rows stored in split order (split_row)
  int vs_lgq = -1;                 // split plan (Grid::vsplit): log2 Q
  alignas(64) CUtensorMap tmap_T;  // T fields, row-item boxes
  int koff[2];
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnb)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnb) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D unsigned load_bytes() const { return (unsigned)((sh.W << sh.lgR) * sizeof(C)); }
  LS_D int n20(int it) const { return (it & ((1 << lgnb) - 1)) << vs_lgq; }
  LS_D void load(int it, int k, C* dst, uint64_t* bar) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    const int tiles = sh.W >> kLgTileT, bt = tiles < 256 ? tiles : 256;
    for (int r = 0; r < (1 << sh.lgR); ++r) {
      const int yr = VS ? vs_plane_row(r, vs_lgq, n20(it))
                                 : split_lgq >= 0 ? split_row(y0 + r, split_lgq) : y0 + r;
      for (int b = 0; b * bt < tiles; ++b)
        tma::tensor_g2s(dst + (r << sh.lgW) + ((b * bt) << kLgTileT), &tmap_T, 0, b * bt, yr, k + koff[set], bar);
    }
  }
  LS_D void store(int it, int k, const C* src) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    C* A = a.A[set] + (size_t)k * fsz();
    if constexpr (VS) {  // natural rows n2_0 + q + 2048 m: four strips of Q rows
      const unsigned qb = (unsigned)((sh.W << vs_lgq) * sizeof(C));
      for (int m = 0; m < 4; ++m)
        tma::bulk_s2g(A + ((size_t)vs_row(m << vs_lgq, vs_lgq, n20(it)) << sh.lgW), src + ((m << vs_lgq) << sh.lgW), qb);
      return;
    }
    tma::bulk_s2g(A + ((size_t)y0 << sh.lgW), src, load_bytes());
  }
  LS_D void begin(State& S, int, C*) const {
#pragma unroll
    for (int i = 0; i < P; ++i) S.acc[i] = (R)0;
  }
  template <int LGN> struct F {
    C* b;
    State& S;
    R w;
    template <int ST> LS_D C load(int seq, int j, int r, int) const { return b[nat_row<LGN, ST>(seq, j, r, 0)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int slot) {
      S.acc[slot] += w * (v.x * v.x + v.y * v.y);
      b[nat_out<LGN, ST, C, false>(seq, j, r)] = v;
    }
  };
  LS_D void step(State& S, int it, int k, C* b, C*, unsigned) const {
    const Geo g = sh.grow();
    if constexpr (VS) {
      vs_inv_combine(b, sh.lgW, vs_lgq, n20(it), tw, sh.twsH);
      __syncthreads();
    }
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b, S, a.w[set_of(it, lgnb)][k]};
        eng::run_fix<LGN, false, true>(g, b, tw, f);
      }
    });
  }
  template <int LGN> struct WriteIS {  // split plan: buffer row -> natural row
    R* I;
    const State& S;
    int lgq, n20, W;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      I[rm_row<LGN, ST>(W, vs_row(seq, lgq, n20), j, r)] = S.acc[slot];
    }
  };
  LS_D void end(State& S, int it, C*, C*) const {
    const int set = set_of(it, lgnb), blk = it & ((1 << lgnb) - 1), y0 = blk << sh.lgR;
    const Geo g = sh.grow();
    const size_t n = (size_t)sh.H * sh.W;
    R* dst = lgg ? a.Ipart + (size_t)((set << lgg) + grp_of(it, lgnb)) * n : a.I[set];
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (VS)
        eng::for_last_slots<LGN, false, C>(g, WriteIS<LGN>{dst, S, vs_lgq, n20(it), sh.W});
      else
        eng::for_last_slots<LGN, false, C>(g, typename F2Op<R>::template WriteI<LGN>{dst, S, y0, sh.W});
    });
    if (lgg)
      group_combine(a.Ipart + (size_t)(set << lgg) * n, n, a.I[set], (size_t)y0 * sh.W, 1 << sh.lgR, sh.W, sh.W,
                    1 << lgg, &a.tick[set * a.tick_stride + blk]);
  }
};

// TA1: U_k = FFT_x(gate . A_k): A_k rows in by 1-D bulk, U_k rows out by tensor map
template <typename R, bool VS = false> struct TA1Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  static constexpr bool kStores = true;
  static constexpr bool kSideLoad = false;
  using State = typename A1Op<R>::State;
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  alignas(64) CUtensorMap tmap_U;  // U fields (layout tile lg_tile<C>), row-item boxes
  int koff[2];
  int vs_lgq = -1;                 // split plan (Grid::vsplit): log2 Q
  LS_D int steps(int it) const { return lgg ? kpg : a.nk[set_of(it, lgnb)]; }
  LS_D int kbase(int it) const { return grp_of(it, lgnb) * kpg; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D unsigned load_bytes() const { return (unsigned)((sh.W << sh.lgR) * sizeof(C)); }
  LS_D int n20(int it) const { return (it & ((1 << lgnb) - 1)) << vs_lgq; }
  LS_D void load(int it, int k, C* dst, uint64_t* bar) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    const C* A = a.A[set] + (size_t)k * fsz();
    if constexpr (VS) {  // natural rows n2_0 + q + 2048 m: four strips of Q rows
      const unsigned qb = (unsigned)((sh.W << vs_lgq) * sizeof(C));
      for (int m = 0; m < 4; ++m)
        tma::bulk_g2s(dst + ((m << vs_lgq) << sh.lgW), A + ((size_t)vs_row(m << vs_lgq, vs_lgq, n20(it)) << sh.lgW),
                      qb, bar);
      return;
    }
    tma::bulk_g2s(dst, A + ((size_t)y0 << sh.lgW), load_bytes(), bar);
  }
  LS_D void store(int it, int k, const C* src) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    constexpr int LGT = lg_tile<C>();
    const int tiles = sh.W >> LGT, bt = tiles < 256 ? tiles : 256;
    for (int r = 0; r < (1 << sh.lgR); ++r) {
      const int y = VS ? vs_plane_row(r, vs_lgq, n20(it)) : y0 + r;
      for (int b = 0; b * bt < tiles; ++b)
        tma::tensor_s2g(&tmap_U, 0, b * bt, y, k + koff[set], src + (r << sh.lgW) + ((b * bt) << LGT));
    }
  }
  template <int LGN> struct LoadGS {  // split plan: buffer row -> natural row
    State& S;
    const R* gate;
    int lgq, n20, W;
    template <int ST> LS_D void operator()(int seq, int j, int r, int slot) const {
      S.g[slot] = __ldg(&gate[rm_row<LGN, ST>(W, vs_row(seq, lgq, n20), j, r)]);
    }
  };
  LS_D void begin(State& S, int it, C*) const {
    const int set = set_of(it, lgnb), y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    eng::dispatch<C>(sh.grow(), true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        if constexpr (VS)
          eng::for_first_slots<LGN, false, C>(LoadGS<LGN>{S, a.gate[set], vs_lgq, n20(it), sh.W});
        else
          eng::for_first_slots<LGN, false, C>(typename A1Op<R>::template LoadG<LGN>{S, a.gate[set], y0, sh.W});
      }
    });
  }
  template <int LGN> struct F {
    C* b;
    const State& S;
    template <int ST> LS_D C load(int seq, int j, int r, int slot) const {
      return b[nat_row<LGN, ST>(seq, j, r, 0)] * S.g[slot];
    }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int) { b[nat_out<LGN, ST, C, false>(seq, j, r)] = v; }
  };
  LS_D void step(State& S, int it, int, C* b, C*, unsigned) const {
    const Geo g = sh.grow();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b, S};
        eng::run_fix<LGN, false, false>(g, b, tw, f);
      }
    });
    if constexpr (VS) {
      __syncthreads();
      vs_fwd_combine(b, sh.lgW, vs_lgq, n20(it), tw, sh.twsH);
    }
  }
};

// TA2: V_set = IFFT_y(sum_k w_k conj(H_k) FFT_y U_k).  U_k tiles arrive in the
// ring; since the pass stores nothing per step, the ring's third slot is idle
// and holds H_k of the current step (TMA, own mbarrier), which the last
// butterfly stage reads from shared memory.  H_k of step q+1 is requested as
// soon as step q's last stage has read its operand slot, a full step ahead.
template <typename R, bool VS = false> struct TA2Op : A2Op<R, VS> {
  using C = typename CT<R>::C;
  using State = typename A2Op<R, VS>::State;
  static constexpr int P = eng::P_of<C>();
  static constexpr bool kStores = false;
  static constexpr bool kSideLoad = true;
  int u_lgw;
  alignas(64) CUtensorMap tmap_U;     // U fields, column-item boxes
  alignas(64) CUtensorMap tmap_spec;  // spectra of set 0, column-item boxes
  alignas(64) CUtensorMap tmap_spec1; // spectra of set 1
  int koff[2];
  LS_D unsigned load_bytes() const { return (unsigned)((this->sh.H << this->sh.lgS) * sizeof(C)); }
  template <class Fn> LS_D void col_boxes(int x0, Fn&& fn) const {
    const int ew = sizeof(C) / 8, w = 1 << u_lgw, S = 1 << this->sh.lgS;
    const int rows = this->sh.H < 256 ? this->sh.H : 256;
    for (int b = 0; b * rows < this->sh.H; ++b) fn((x0 & (w - 1)) * ew, x0 >> u_lgw, b * rows, b * rows * S);
  }
  // whole-tile items are contiguous blocks: one 1-D bulk copy each
  LS_D size_t tile_off(int x0) const { return (size_t)(x0 >> u_lgw) * this->sh.H << u_lgw; }
  LS_D void load(int it, int k, C* dst, uint64_t* bar) const {
    const int set = this->set_of(it, this->lgnt), x0 = (it & ((1 << this->lgnt) - 1)) << this->sh.lgS;
    if (u_lgw == this->sh.lgS) {
      tma::bulk_g2s(dst, this->a.T[0] + (size_t)(k + koff[set]) * this->sh.H * this->sh.W + tile_off(x0),
                    load_bytes(), bar);
      return;
    }
    col_boxes(x0, [&](int c0, int c1, int c2, int off) {
      tma::tensor_g2s(dst + off, &tmap_U, c0, c1, c2, k + koff[set], bar);
    });
  }
  LS_D void side_load(int it, int k, C* dst, uint64_t* bar) const {
    const int set = this->set_of(it, this->lgnt), x0 = (it & ((1 << this->lgnt) - 1)) << this->sh.lgS;
    if (u_lgw == this->sh.lgS) {
      tma::bulk_g2s(dst, this->a.spec[set] + (size_t)k * this->sh.H * this->sh.W + tile_off(x0), load_bytes(), bar);
      return;
    }
    const CUtensorMap* m = set ? &tmap_spec1 : &tmap_spec;
    col_boxes(x0, [&](int c0, int c1, int c2, int off) { tma::tensor_g2s(dst + off, m, c0, c1, c2, k, bar); });
  }
  LS_D void store(int, int, const C*) const {}
  template <int LGN> struct F {
    const C* b;
    const C* h;     // H_k tile (natural [y][S]) in the side slot
    uint64_t* bar;  // its mbarrier
    unsigned parity;
    State& S;
    R w;
    // next step's H_k, issued into this step's slot once every thread has
    // read it (the engine's barrier after the last stage's loads)
    const TA2Op* op;
    int it, knext;
    uint64_t* nbar;
    bool issue;
    LS_D void pre_store() const {
      if (issue && threadIdx.x == 0) {
#ifdef LSB_EXP_NOTMA
        tma::mbar_expect_tx(nbar, 0);
#else
        tma::mbar_expect_tx(nbar, op->load_bytes());
        op->side_load(it, knext, const_cast<C*>(b), nbar);
#endif
      }
      tma::mbar_wait(bar, parity);
    }
    template <int ST> LS_D C load(int seq, int j, int r, int) const { return b[nat_col<LGN, ST, C>(seq, j, r, 0)]; }
    template <int ST> LS_D void store(int seq, int j, int r, C v, int slot) {
      S.acc[slot] = S.acc[slot] + cmulc(v, h[nat_col<LGN, ST, C>(seq, j, r, 0)]) * w;
    }
  };
  LS_D void step_side(State& S, int it, int k, C* b, C* side, unsigned q, uint64_t* bars, bool issue_next) const {
    const Geo g = this->sh.gcol();
    eng::dispatch<C>(g, true, [&](auto fx) {
      constexpr int LGN = decltype(fx)::LGN;
      if constexpr (LGN > 0) {
        F<LGN> f{b, side, &bars[3 + (q & 1u)], (q >> 1) & 1u, S, this->a.w[this->set_of(it, this->lgnt)][k],
                 this, it, k + 1, &bars[3 + ((q + 1) & 1u)], issue_next};
        eng::run_fix<LGN, true, false>(g, b, this->tw, f);
      }
    });
  }
};

// ---------------------------------------------------------------------------
// launch plumbing

// the dynamic shared-memory allowance left beside a kernel's static shared
// memory (the kernel-group combine keeps a flag there), out of 227 KB
template <class K> int max_dyn_smem(K* kern) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kern);
  return 227 * 1024 - (int)fa.sharedSizeBytes;
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename R, class Op>
int launch_op(Op& op, int threads, int extra_bufs, StopFlag stop, cudaStream_t s, int max_grid = 0) {
  using C = typename CT<R>::C;
  const size_t smem =
      std::max((size_t)(Op::kStages + extra_bufs) * op.bufE * sizeof(C), (size_t)(64 * sizeof(double)));
  if (smem > 227 * 1024) throw std::runtime_error("spectral pass needs more than 227 KB of shared memory");
  auto kern = k_pass<R, Op>;
  static int per_sm = -1;
  static size_t per_sm_smem = 0;
  static int per_sm_threads = 0;
  if (per_sm < 0 || per_sm_smem != smem || per_sm_threads != threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem(kern));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem);
    per_sm = std::max(b, 1);
    per_sm_smem = smem;
    per_sm_threads = threads;
  }
  int grid = std::min(op.nitems, num_sms() * per_sm);
  if (max_grid > 0) grid = std::min(grid, max_grid);
  if (grid < 1) grid = 1;
  kern<<<grid, threads, smem, s>>>(op, stop);
  return grid;
}

template <typename R, class Op>
int launch_tma(Op& op, int threads, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const size_t smem = 3 * (size_t)op.bufE * sizeof(C) + 5 * sizeof(uint64_t);
  if (smem > 227 * 1024) throw std::runtime_error("TMA pass needs more than 227 KB of shared memory");
  auto kern = k_pass_tma<R, Op>;
  static int per_sm = -1;
  if (per_sm < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem(kern));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem);
    per_sm = std::max(b, 1);
  }
  const int grid = std::max(1, std::min(op.nitems, num_sms() * per_sm));
  kern<<<grid, threads, smem, s>>>(op, stop);
  return grid;
}

// ---------------------------------------------------------------------------
// Tall grids outside the split plan (see the column-pass note above), F1 as a
// four-step split across the cluster (H = 4M, M = 2048, complex64): the column
// transform of a 4-column tile is split across the 4-CTA cluster so every
// CTA runs the fast 4-column 2048-point engine.  With f = f2 + M c and
// n = 4 m + k1 (N = 4M):
//   inverse  x[4m + k1] = IFFT_M( y_k1 )[m],
//            y_k1[f2] = e^{+2 pi i f2 k1 / N} sum_c P[f2 + M c] i^{c k1}
// so F1 does the radix-4 step first: CTA r fetches the rows it combines
// (f2 in [M r / 4, M (r+1) / 4) at the four offsets M c: four 16 KB strips, one
// bulk copy each), forms y_k1 and pushes it to CTA k1 through distributed
// shared memory; then each CTA runs the local 4-column 2048-point inverse.
// CTA k1's output rows 4 m + k1 are stored as T_k rows k1 M + m (the row
// permutation `split_row`, undone by F2's per-row loads).  Measured (8192 x
// 2048 window): F1 8.3 -> 7.0 ms; the two cluster barriers per step
// (MEMBAR / ERRBAR / UCGABAR stalls in ncu) and the 64 KB of DSMEM stores per
// CTA per step are now the cost.  The adjoint column pass (A2) keeps the
// single-column cluster path.
constexpr int kSplitM = 2048;
LS_D float2 mul_ipow(float2 z, int e) {  // z * i^e
  switch (e & 3) {
    case 0: return z;
    case 1: return make_float2(-z.y, z.x);
    case 2: return make_float2(-z.x, -z.y);
    default: return make_float2(z.y, -z.x);
  }
}
LS_D void ld_row4(unsigned addr, float2 (&v)[4]) {
  const float4 a = tma::ld_cluster_f4(addr), b = tma::ld_cluster_f4(addr + 16);
  v[0] = make_float2(a.x, a.y);
  v[1] = make_float2(a.z, a.w);
  v[2] = make_float2(b.x, b.y);
  v[3] = make_float2(b.z, b.w);
}
LS_D void st_row4(unsigned addr, const float2 (&v)[4]) {
  tma::st_cluster_f4(addr, make_float4(v[0].x, v[0].y, v[1].x, v[1].y));
  tma::st_cluster_f4(addr + 16, make_float4(v[2].x, v[2].y, v[3].x, v[3].y));
}

struct F1SplitArgs {
  Shape<float> sh;
  SetArgs<float> a;
  const float2* mhat;
  float scale;
  const float2* tw;  // N entries, e^{-2 pi i j / N}
  int ntiles, nsets, bufE, lgnmax;
  alignas(64) CUtensorMap tmap_T;
  int koff[2];
};

// in-place natural [row][4] transform of the local quarter
template <int LGN> struct SplitF {
  float2* b;
  template <int ST> LS_D float2 load(int seq, int j, int r, int) const { return b[nat_col<LGN, ST, float2>(seq, j, r, 0)]; }
  template <int ST> LS_D void store(int seq, int j, int r, float2 v, int) { b[nat_col<LGN, ST, float2>(seq, j, r, 0)] = v; }
};

template <int V = 0>  // a template: the header is compiled in several translation units
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 1)
k_f1_split(const __grid_constant__ F1SplitArgs A, StopFlag stop) {
  using C = float2;
  constexpr int M = kSplitM, QE = M * 4, Q4 = M / 4;
  if (stop && *stop) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  C* const work = reinterpret_cast<C*>(smraw);
  C* const in = work + A.bufE;  // 2 x [M][4]
  uint64_t* bar = reinterpret_cast<uint64_t*>(in + 2 * QE);
  const unsigned rank = tma::cluster_rank();
  const int cid = blockIdx.x / 4, ncl = gridDim.x / 4, nit = A.ntiles * A.nsets;
  const bool leader = threadIdx.x == 0;
  const int H = A.sh.H, lgq = 11;  // storage quarter = 2^11 rows
  if (leader) {
    tma::mbar_init(&bar[0], 1);
    tma::mbar_init(&bar[1], 1);
    tma::fence_mbar_init();
  }
  __syncthreads();
  if (cid >= nit) return;
  // this CTA's rows of the radix-4 step: f2 in [Q4 r, Q4 (r+1)) at the four
  // offsets M c -- four contiguous 16 KB strips of the tile, one bulk copy each
  auto issue = [&](int it4, int k, int slot) {
    const int set = it4 / A.ntiles, t = it4 - set * A.ntiles;
    const C* tile = A.a.spec[set] + (size_t)k * H * A.sh.W + (size_t)t * H * 4;
    tma::mbar_expect_tx(&bar[slot], (unsigned)(QE * sizeof(C)));
    for (int c = 0; c < 4; ++c)
      tma::bulk_g2s(in + (size_t)slot * QE + (size_t)c * Q4 * 4, tile + ((size_t)M * c + (size_t)Q4 * rank) * 4,
                    (unsigned)(Q4 * 4 * sizeof(C)), &bar[slot]);
  };
  unsigned addr_work[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) addr_work[c] = tma::cluster_map(work, c);
  const int f2 = Q4 * (int)rank + (int)threadIdx.x;  // this thread's row of the radix-4 step
  C mh[4][4];                                        // M^ at rows f2 + M c, 4 columns
  int it4 = cid, st = 0;
  if (leader) issue(it4, 0, 0);
  for (unsigned q = 0;; ++q) {
    const int slot = q & 1, set = it4 / A.ntiles, t = it4 - set * A.ntiles, nk = A.a.nk[set];
    int nit4 = it4, nst = st + 1;
    if (nst == nk) {
      nst = 0;
      nit4 += ncl;
    }
    if (st == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4* row = reinterpret_cast<const float4*>(A.mhat + ((size_t)t * H + f2 + (size_t)M * c) * 4);
        const float4 u = __ldg(row), v = __ldg(row + 1);
        mh[c][0] = make_float2(u.x * A.scale, u.y * A.scale);
        mh[c][1] = make_float2(u.z * A.scale, u.w * A.scale);
        mh[c][2] = make_float2(v.x * A.scale, v.y * A.scale);
        mh[c][3] = make_float2(v.z * A.scale, v.w * A.scale);
      }
    }
    if (leader && nit4 < nit) issue(nit4, nst, slot ^ 1);  // the other strip buffer was consumed last step
    tma::mbar_wait(&bar[slot], (q >> 1) & 1);
    if (leader) tma::bulk_wait_read<0>();  // the previous step's T store has read `work`
    tma::cluster_sync();                     // every CTA's `work` is free
    {
      C p[4][4];
      const C* strips = in + (size_t)slot * QE;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4* row = reinterpret_cast<const float4*>(strips + ((size_t)c * Q4 + threadIdx.x) * 4);
        const float4 u = row[0], v = row[1];
        const C h[4] = {make_float2(u.x, u.y), make_float2(u.z, u.w), make_float2(v.x, v.y), make_float2(v.z, v.w)};
#pragma unroll
        for (int col = 0; col < 4; ++col) p[c][col] = cmul(mh[c][col], h[col]);
      }
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) {
        const C w = cconj(__ldg(&A.tw[f2 * k1]));
        C y[4];
#pragma unroll
        for (int col = 0; col < 4; ++col) {
          C acc = p[0][col];
#pragma unroll
          for (int c = 1; c < 4; ++c) acc = acc + mul_ipow(p[c][col], c * k1);
          y[col] = k1 ? cmul(acc, w) : acc;
        }
        st_row4(addr_work[k1] + (unsigned)(f2 * 4 * sizeof(C)), y);
      }
    }
    // (st.async with per-row mbarrier completion in place of this barrier measured slower)
    tma::cluster_sync();  // every CTA's y quarter complete
    {
      const Geo g{11, 2, A.lgnmax - 11};
      SplitF<11> f{work};
      eng::run_fix<11, true, true>(g, work, A.tw, f);
    }
    tma::fence_async_smem();
    __syncthreads();
    if (leader) {
      constexpr int w = 1 << kLgTileT;
      const int x0 = 4 * t;
      for (int b = 0; b * 256 < M; ++b)
        tma::tensor_s2g(&A.tmap_T, x0 & (w - 1), x0 >> kLgTileT, ((int)rank << lgq) + b * 256, st + A.koff[set],
                        work + (size_t)b * 256 * 4);
      tma::bulk_commit();
    }
    it4 = nit4;
    st = nst;
    if (it4 >= nit) break;
  }
  if (leader) tma::bulk_wait<0>();
  tma::cluster_sync();
}

// tall-grid column passes by 4-CTA clusters (k_pass_cluster): one complex64
// column per CTA of a 4-wide tile layout
template <typename R> bool cluster_ok(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  static const bool off = [] {
    const char* e = std::getenv("LSOPC_B200_NO_CLUSTER");
    return e && e[0] == '1';
  }();
  return !off && !tma_disabled() && sizeof(C) == 8 && sh.fast() && sh.lgS == 0 && sh.lgT == 2 &&
         sh.W % kClusterCols == 0 && sh.H % (kClusterCols * 16) == 0;
}
// four-step split path (k_f1_split / k_a2_split): H = 4 * 2048 complex64 rows
template <typename R> bool split_ok(const Shape<R>& sh) {
  static const bool off = [] {
    const char* e = std::getenv("LSOPC_B200_NO_SPLIT");
    return e && e[0] == '1';
  }();
  return !off && cluster_ok(sh) && sh.H == 4 * kSplitM && sh.W <= sh.H;
}
inline int max_clusters(const void* kern, int threads, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms() / 4 * 4);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 4;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = num_sms() / 4;
  }
  return n;
}
inline void launch_f1_split(F1SplitArgs& A, StopFlag stop, cudaStream_t s) {
  const size_t smem = (size_t)A.bufE * sizeof(float2) + 2 * (size_t)kSplitM * 4 * sizeof(float2) + 2 * sizeof(uint64_t);
  static int fit = 0;
  if (!fit) {
    cudaFuncSetAttribute(k_f1_split<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_f1_split<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    fit = max_clusters((const void*)k_f1_split<0>, 512, smem);
  }
  const int clusters = std::max(1, std::min(A.ntiles * A.nsets, fit));
  k_f1_split<0><<<clusters * 4, 512, smem, s>>>(A, stop);
}

template <typename R, class Op>
void launch_cluster(Op& op, int ntiles, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const size_t qE = (size_t)op.sh.H;  // a row quarter of a 4-wide tile: H/4 rows x 4
  const size_t smem = (size_t)op.bufE * sizeof(C) + 2 * qE * sizeof(C) + 2 * sizeof(uint64_t);
  if (smem > 227 * 1024) throw std::runtime_error("cluster column pass needs more than 227 KB of shared memory");
  auto kern = k_pass_cluster<R, Op>;
  // clusters live inside one GPC, so fewer than SMs / 4 may be co-resident:
  // launch exactly as many as fit (the kernel loops over the items)
  static int fit = 0;
  static size_t fit_smem = 0;
  if (!fit || fit_smem != smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem(kern));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(num_sms() / kClusterCols * kClusterCols);
    cfg.blockDim = dim3(eng::cta_threads<C>());
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = kClusterCols;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = num_sms() / kClusterCols;
    }
    fit = n;
    fit_smem = smem;
  }
  const int nit = ntiles * nsets;
  const int clusters = std::max(1, std::min(nit, fit));
  kern<<<clusters * kClusterCols, eng::cta_threads<C>(), smem, s>>>(op, stop, ntiles, nsets);
}

// slot size for the TMA ring: the padded exchange buffer, rounded to 128 B
template <typename R> int tma_bufE(int e) {
  using C = typename CT<R>::C;
  const int q = 128 / (int)sizeof(C);
  return (e + q - 1) / q * q;
}

template <typename R> int set_koff(const SetArgs<R>& a, int set, size_t n) {
  return (int)((a.T[set] - a.T[0]) / (std::ptrdiff_t)n);
}
template <typename R> int total_nk(const SetArgs<R>& a) { return a.nk[0] + (a.nsets > 1 ? a.nk[1] : 0); }

template <typename R> int col_threads(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return std::max(1, ((1 << sh.lgS) << sh.lgH) / eng::P_of<C>());
}
template <typename R> int row_threads(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return std::max(1, ((1 << sh.lgR) << sh.lgW) / eng::P_of<C>());
}
// stage-buffer sizes are rounded to 128 B so every ring slot stays aligned for
// 16 B cp.async and TMA destinations
template <typename R> int align_elems(int e) {
  using C = typename CT<R>::C;
  const int q = 128 / (int)sizeof(C);
  return (e + q - 1) / q * q;
}
template <typename R> int col_bufE(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return align_elems<R>(eng::buf_elems<C>(sh.H, 1 << sh.lgS));
}
template <typename R> int row_bufE(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  // the mask pass stages raw f64 input (8 B/elem) in a complex buffer
  return align_elems<R>(std::max(eng::buf_elems<C>(sh.W, 1 << sh.lgR), (int)(((1 << sh.lgR) << sh.lgW) * 8 / sizeof(C))));
}

template <typename R> SetArgs<R> set_args(const Grid& g, const SpecSet* sets, int nsets) {
  using C = typename CT<R>::C;
  SetArgs<R> a{};
  a.nsets = nsets;
  for (int i = 0; i < nsets; ++i) {
    if (sets[i].nk > kMaxK) throw std::runtime_error("at most 64 kernels per set are supported");
    a.nk[i] = sets[i].nk;
    a.spec[i] = static_cast<const C*>(sets[i].spec);
    a.T[i] = static_cast<C*>(sets[i].T);
    a.A[i] = static_cast<C*>(sets[i].A);
    a.I[i] = static_cast<R*>(sets[i].I);
    a.gate[i] = static_cast<const R*>(sets[i].gate);
    a.V[i] = static_cast<C*>(sets[i].V);
    for (int k = 0; k < sets[i].nk; ++k) a.w[i][k] = (R)sets[i].w[k];
  }
  a.Ipart = static_cast<R*>(sets[0].Ipart);
  a.Vpart = static_cast<C*>(sets[0].Vpart);
  a.tick = sets[0].tick;
  a.tick_stride = std::max(g.H, g.W);
  return a;
}

// Kernel groups for a pass with base_items (block x set) items: the largest
// power of two G <= 8 that keeps G * base_items within the SM count and
// divides every set's kernel count (sets of equal size), when the plan
// provides the partial buffers.  Returns log2 G.
template <typename R> int choose_lgg(int base_items, const SetArgs<R>& a) {
  if (!a.Ipart || !a.Vpart || !a.tick) return 0;
  if (a.nsets > 1 && a.nk[0] != a.nk[1]) return 0;
  int lgg = 0;
  while (lgg < 3) {
    const int G = 2 << lgg;
    if ((long)base_items * G > (long)num_sms() || a.nk[0] % G) break;
    ++lgg;
  }
  return lgg;
}

// split plans instantiate the ops with VS = true (compile-time: the unsplit
// passes keep their exact code)
template <class Fn> void with_vs(bool vs, Fn&& fn) {
  if (vs) fn(std::true_type{});
  else fn(std::false_type{});
}

// ---------------------------------------------------------------------------

template <typename R>
void mask_fft_impl(const Grid& g, const void* src, int kind, void* mhat, void* scratch, StopFlag stop,
                   cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  const size_t src_bytes = ((size_t)1 << sh.lgR) * g.W * (kind == SRC_U8 ? 1 : 8);
  const bool rows_tma = tma_ok_rows(sh) && src_bytes % 16 == 0 && src_bytes <= (size_t)row_bufE(sh) * sizeof(C) &&
                        reinterpret_cast<uintptr_t>(src) % 16 == 0;
  if (g.vsplit && !rows_tma) throw std::runtime_error("split plan: mask rows need the TMA path");
  if (rows_tma) {
    with_vs(g.vsplit, [&](auto vs) {
      TMaskRowsOp<R, decltype(vs)::value> mr;
      mr.sh = sh;
      mr.src = src;
      mr.kind = kind;
      mr.tw = static_cast<const C*>(g.tw);
      const int ew = sizeof(C) / 8, tiles = g.W >> sh.lgT;
      mr.tmap_out = make_field_map(TmaField{scratch, sh.lgT, ew}, g.H, g.W, 1, (unsigned)((1 << sh.lgT) * ew),
                                   (unsigned)std::min(tiles, 256), 1);
      mr.vs_lgq = g.vsplit ? sh.lgR - 2 : -1;
      mr.bufE = tma_bufE<R>(row_bufE(sh));
      mr.nitems = g.H >> sh.lgR;
      launch_tma<R>(mr, row_threads(sh), stop, s);
    });
  } else {
    MaskRowsOp<R> mr;
    mr.sh = sh;
    mr.src = src;
    mr.kind = kind;
    mr.out = static_cast<C*>(scratch);
    mr.tw = static_cast<const C*>(g.tw);
    mr.bufE = row_bufE(sh);
    mr.nitems = g.H >> sh.lgR;
    launch_op<R>(mr, row_threads(sh), 0, stop, s);
  }
  if (!mhat) return;  // the row pass only (M~ for the tensor-core F1)
  if (g.vsplit) {  // columns of the virtual 2048 x 4W grid
    const Grid gv = vs_grid(g);
    sh = shape_of<R>(gv);
    if (!(tma_ok_cols(sh) && sh.lgS == sh.lgT)) throw std::runtime_error("split plan: columns need the TMA path");
  }
  if (tma_ok_cols(sh) && sh.lgS == sh.lgT) {
    TColsOp<R> mc;
    mc.sh = sh;
    mc.in = static_cast<const C*>(scratch);
    mc.out = static_cast<C*>(mhat);
    mc.tw = static_cast<const C*>(g.tw);
    mc.bufE = tma_bufE<R>(col_bufE(sh));
    mc.nitems = sh.W >> sh.lgS;
    launch_tma<R>(mc, col_threads(sh), stop, s);
    return;
  }
  ColsOp<R, R, false> mc;
  mc.sh = sh;
  mc.in = static_cast<const C*>(scratch);
  mc.Lin = sh.ct();
  mc.Lout = sh.ct();
  mc.out = static_cast<C*>(mhat);
  mc.scale = (R)1;
  mc.tw = static_cast<const C*>(g.tw);
  mc.bufE = col_bufE(sh);
  mc.nitems = g.W >> sh.lgS;
  launch_op<R>(mc, col_threads(sh), 0, stop, s);
}

template <typename R>
void f1_impl(const Grid& gp, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const Grid g = gp.vsplit ? vs_grid(gp) : gp;  // split plans: the virtual 2048 x 4W grid
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  if (gp.vsplit && !tma_ok_cols(sh)) throw std::runtime_error("split plan: F1 needs the TMA path");
  if (tma_ok_cols(sh)) {
    with_vs(gp.vsplit, [&](auto vs) {
      TF1Op<R, decltype(vs)::value> f1;
      f1.sh = sh;
      f1.a = a;
      f1.mhat = static_cast<const C*>(mhat);
      f1.scale = (R)(1.0 / (double)g.n());
      f1.tw = static_cast<const C*>(g.tw);
      f1.lgnt = g.lgW - sh.lgS;
      f1.spec_lgw = sh.lgT;
      const int ew = sizeof(C) / 8, S = 1 << sh.lgS, rows = std::min(g.H, 256);
      auto colbox = [&](int lgw) { return std::make_pair((unsigned)(std::min(S, 1 << lgw) * ew),
                                                           (unsigned)std::max(1, S >> lgw)); };
      // spectra of each set: separate allocations -> separate maps (koff 0)
      for (int i = 0; i < nsets; ++i) {
        auto cb = colbox(sh.lgT);
        CUtensorMap m = make_field_map(TmaField{a.spec[i], sh.lgT, ew}, g.H, g.W, a.nk[i], cb.first, cb.second, rows);
        if (i == 0) f1.tmap_spec = m; else f1.tmap_spec1 = m;
      }
      auto cbT = colbox(kLgTileT);
      // T_k keeps the physical layout (the F2 row pass reads plane rows by coordinates)
      f1.tmap_T = make_field_map(TmaField{a.T[0], kLgTileT, ew}, gp.H, gp.W, total_nk(a), cbT.first, cbT.second, rows);
      f1.vs_lgt = gp.vsplit ? sh.lgT : -1;
      for (int i = 0; i < 2; ++i) f1.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
      f1.bufE = tma_bufE<R>(col_bufE(sh));
      f1.lgg = gp.vsplit ? 0 : choose_lgg<R>((1 << f1.lgnt) * nsets, a);
      f1.kpg = a.nk[0] >> f1.lgg;
      f1.nitems = ((1 << f1.lgnt) * nsets) << f1.lgg;
      launch_tma<R>(f1, col_threads(sh), stop, s);
    });
    return;
  }
  F1Op<R> f1;
  f1.sh = sh;
  f1.a = a;
  f1.mhat = static_cast<const C*>(mhat);
  f1.scale = (R)(1.0 / (double)g.n());
  f1.tw = static_cast<const C*>(g.tw);
  f1.lgnt = g.lgW - sh.lgS;
  f1.bufE = col_bufE(sh);
  f1.nitems = (1 << f1.lgnt) * nsets;
  if constexpr (sizeof(C) == 8) {
    if (split_ok(sh)) {
      F1SplitArgs A;
      A.sh = sh;
      A.a = a;
      A.mhat = static_cast<const float2*>(mhat);
      A.scale = (float)(1.0 / (double)g.n());
      A.tw = static_cast<const float2*>(g.tw);
      A.ntiles = g.W / 4;
      A.nsets = nsets;
      A.lgnmax = g.lgnmax;
      // the local buffer holds 4 columns x 2048 rows with the exchange padding
      A.bufE = tma_bufE<R>(align_elems<R>(eng::buf_elems<C>(kSplitM, 4)));
      A.tmap_T = make_field_map(TmaField{a.T[0], kLgTileT, 1}, g.H, g.W, total_nk(a), 4u, 1, 256);
      for (int i = 0; i < 2; ++i) A.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
      launch_f1_split(A, stop, s);
      return;
    }
  }
  if (cluster_ok(sh)) {
    F1COp<R> fc;
    static_cast<F1Op<R>&>(fc) = f1;
    fc.bufE = tma_bufE<R>(col_bufE(sh));
    const int ew = sizeof(C) / 8;
    fc.tmap_T = make_field_map(TmaField{a.T[0], kLgTileT, ew}, g.H, g.W, total_nk(a), (unsigned)(kClusterCols * ew),
                               1, 256);
    for (int i = 0; i < 2; ++i) fc.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
    launch_cluster<R>(fc, g.W / kClusterCols, nsets, stop, s);
    return;
  }
  launch_op<R>(f1, col_threads(sh), 0, stop, s);
}

template <typename R>
void f2_impl(const Grid& g, const SpecSet* sets, int nsets, double2* a0_out, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  if (g.vsplit && !tma_ok_rows(sh)) throw std::runtime_error("split plan: F2 needs the TMA path");
  if (tma_ok_rows(sh)) {
    with_vs(g.vsplit, [&](auto vs) {
      TF2Op<R, decltype(vs)::value> f2;
      f2.sh = sh;
      f2.a = a;
      f2.tw = static_cast<const C*>(g.tw);
      f2.lgnb = g.lgH - sh.lgR;
      f2.split_lgq = !g.vsplit && split_ok(sh) ? 11 : -1;
      f2.vs_lgq = g.vsplit ? sh.lgR - 2 : -1;
      const int ew = sizeof(C) / 8, tiles = g.W >> kLgTileT;
      f2.tmap_T = make_field_map(TmaField{a.T[0], kLgTileT, ew}, g.H, g.W, total_nk(a), (unsigned)((1 << kLgTileT) * ew),
                                 (unsigned)std::min(tiles, 256), 1);
      for (int i = 0; i < 2; ++i) f2.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
      f2.bufE = tma_bufE<R>(row_bufE(sh));
      f2.lgg = g.vsplit ? 0 : choose_lgg<R>((1 << f2.lgnb) * nsets, a);
      f2.kpg = a.nk[0] >> f2.lgg;
      f2.nitems = ((1 << f2.lgnb) * nsets) << f2.lgg;
      launch_tma<R>(f2, row_threads(sh), stop, s);
    });
  } else {
    F2Op<R> f2;
    f2.sh = sh;
    f2.a = a;
    f2.tw = static_cast<const C*>(g.tw);
    f2.lgnb = g.lgH - sh.lgR;
    f2.bufE = row_bufE(sh);
    f2.nitems = (1 << f2.lgnb) * nsets;
    launch_op<R>(f2, row_threads(sh), 0, stop, s);
  }
  if (a0_out)  // convolve(): the first set's first field A_0
    k_ct_to_c128<R><<<148 * 4, 256, 0, s>>>(g.n(), sh.rm(), g.W, a.A[0], a0_out);
}

template <typename R>
void a1_impl(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  if (g.vsplit && !tma_ok_rows(sh)) throw std::runtime_error("split plan: A1 needs the TMA path");
  if (tma_ok_rows(sh)) {
    with_vs(g.vsplit, [&](auto vs) {
      TA1Op<R, decltype(vs)::value> a1;
      a1.vs_lgq = g.vsplit ? sh.lgR - 2 : -1;
      a1.sh = sh;
      a1.a = a;
      a1.tw = static_cast<const C*>(g.tw);
      a1.lgnb = g.lgH - sh.lgR;
      const int ew = sizeof(C) / 8, tiles = g.W >> sh.lgT;
      a1.tmap_U = make_field_map(TmaField{a.T[0], sh.lgT, ew}, g.H, g.W, total_nk(a), (unsigned)((1 << sh.lgT) * ew),
                                 (unsigned)std::min(tiles, 256), 1);
      for (int i = 0; i < 2; ++i) a1.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
      a1.bufE = tma_bufE<R>(row_bufE(sh));
      a1.lgg = g.vsplit ? 0 : choose_lgg<R>((1 << a1.lgnb) * nsets, a);
      a1.kpg = a.nk[0] >> a1.lgg;
      a1.nitems = ((1 << a1.lgnb) * nsets) << a1.lgg;
      launch_tma<R>(a1, row_threads(sh), stop, s);
    });
    return;
  }
  A1Op<R> a1;
  a1.sh = sh;
  a1.a = a;
  a1.tw = static_cast<const C*>(g.tw);
  a1.lgnb = g.lgH - sh.lgR;
  a1.bufE = row_bufE(sh);
  a1.nitems = (1 << a1.lgnb) * nsets;
  launch_op<R>(a1, row_threads(sh), 0, stop, s);
}

template <typename R>
void a2_impl(const Grid& gp, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  const Grid g = gp.vsplit ? vs_grid(gp) : gp;  // split plans: the virtual 2048 x 4W grid
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  if (gp.vsplit && !tma_ok_cols(sh)) throw std::runtime_error("split plan: A2 needs the TMA path");
  if (tma_ok_cols(sh)) {
    with_vs(gp.vsplit, [&](auto vs) {
      TA2Op<R, decltype(vs)::value> a2;
      a2.sh = sh;
      a2.vs_lgt = gp.vsplit ? sh.lgT : -1;
      a2.vs_W = gp.W;
      a2.a = a;
      a2.tw = static_cast<const C*>(g.tw);
      a2.lgnt = g.lgW - sh.lgS;
      a2.u_lgw = sh.lgT;
      const int ew = sizeof(C) / 8, S = 1 << sh.lgS, w = 1 << sh.lgT;
      a2.tmap_U = make_field_map(TmaField{a.T[0], sh.lgT, ew}, g.H, g.W, total_nk(a), (unsigned)(std::min(S, w) * ew),
                                 (unsigned)std::max(1, S / w), (unsigned)std::min(g.H, 256));
      for (int i = 0; i < nsets; ++i) {
        CUtensorMap m = make_field_map(TmaField{a.spec[i], sh.lgT, ew}, g.H, g.W, a.nk[i],
                                       (unsigned)(std::min(S, w) * ew), (unsigned)std::max(1, S / w),
                                       (unsigned)std::min(g.H, 256));
        if (i == 0) a2.tmap_spec = m; else a2.tmap_spec1 = m;
      }
      for (int i = 0; i < 2; ++i) a2.koff[i] = i < nsets ? set_koff(a, i, g.n()) : 0;
      a2.bufE = tma_bufE<R>(col_bufE(sh));
      a2.lgg = gp.vsplit ? 0 : choose_lgg<R>((1 << a2.lgnt) * nsets, a);
      a2.kpg = a.nk[0] >> a2.lgg;
      a2.nitems = ((1 << a2.lgnt) * nsets) << a2.lgg;
      launch_tma<R>(a2, col_threads(sh), stop, s);
    });
    return;
  }
  A2Op<R> a2;
  a2.sh = sh;
  a2.a = a;
  a2.tw = static_cast<const C*>(g.tw);
  a2.lgnt = g.lgW - sh.lgS;
  a2.bufE = col_bufE(sh);
  a2.nitems = (1 << a2.lgnt) * nsets;
  if (cluster_ok(sh)) {
    a2.bufE = tma_bufE<R>(col_bufE(sh));
    launch_cluster<R>(a2, g.W / kClusterCols, nsets, stop, s);
    return;
  }
  launch_op<R>(a2, col_threads(sh), 0, stop, s);
}

template <typename R>
int finish_impl(const Grid& g, const void* V0, const void* V1, double scale, double* out, const double* vp,
                double* dots, StopFlag stop, cudaStream_t s, int ix0, int ix1, const LoopTail* tail, int iy0,
                int iy1) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  int grid = 0;
  with_vs(g.vsplit, [&](auto vs) {
    A3Op<R, decltype(vs)::value> a3;
    a3.sh = sh;
    a3.V0 = static_cast<const C*>(V0);
    a3.V1 = static_cast<const C*>(V1);
    a3.tw = static_cast<const C*>(g.tw);
    a3.scale = scale;
    a3.out = out;
    a3.vp = vp;
    a3.dots = dots;
    a3.ix0 = ix0;
    a3.ix1 = ix1 > 0 ? ix1 : g.W;
    a3.iy0 = iy0;
    a3.iy1 = iy1 < g.H ? iy1 : g.H;
    a3.tail = tail && vp ? *tail : LoopTail{};
    a3.vs_lgq = g.vsplit ? sh.lgR - 2 : -1;
    a3.bufE = row_bufE(sh);
    a3.nitems = g.H >> sh.lgR;
    grid = launch_op<R>(a3, row_threads(sh), 0, stop, s, finish_max_blocks());
  });
  return vp ? grid : 0;
}


}  // namespace spec
}  // namespace lsb
