// SOCS forward model and adjoint as persistent, pipelined spectral passes.
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
//        I_set = sum_k w_k |IFFT_x T_k|^2          accumulated in registers
//   A1  (rows, item = row block x set, loop over kernels):
//        U_k = FFT_x(gate_set . IFFT_x T_k)        A_k recomputed, U_k overwrites T_k
//   A2  (cols, item = column tile x set, loop over kernels):
//        V_set = IFFT_y( sum_k w_k conj(H_k) . FFT_y U_k )   accumulated in registers
//   A3  (rows): g = scale . Re IFFT_x(V_f + V_d)  (+ CG dot partials)
//
// The adjoint uses conj(t) = IFFT2(FFT2(gate A) conj(H)) (equal real part to
// the reference's IFFT2(FFT2(gate conj A) H(-f))), so forward and adjoint read
// the same spectrum at the same frequency.  T_k lives in HBM between F1 and
// F2/A1 (it is the 2-D transform's transpose point); every other intermediate
// stays on chip.
#include "common.cuh"
#include "engine.cuh"
#include "internal.h"

#include <algorithm>
#include <stdexcept>

namespace lsb {

namespace {

using eng::Geo;
using eng::Lay;

constexpr int kMaxK = 64;  // kernels per set carried in a launch

template <typename R> struct Shape {
  int H, W, lgH, lgW;
  int lgS, lgR;     // log2 columns per column item / rows per row item
  int twsH, twsW;   // twiddle-table shifts for the two axes
  LS_HD Geo gcol() const { return Geo{lgH, lgS, twsH}; }
  LS_HD Geo grow() const { return Geo{lgW, lgR, twsW}; }
  LS_HD Lay ct() const { return Lay{H, lgS}; }   // column-tiled layout of spectral fields
  LS_HD Lay rm() const { return Lay{H, lgW}; }   // row-major
};

template <typename R> Shape<R> shape_of(const Grid& g) {
  using C = typename CT<R>::C;
  const int E = 512 * eng::P_of<C>();
  Shape<R> s;
  s.H = g.H; s.W = g.W; s.lgH = g.lgH; s.lgW = g.lgW;
  s.lgS = std::max(0, std::min(g.lgW, ilog2i(E) - g.lgH));
  s.lgR = std::max(0, std::min(g.lgH, ilog2i(E) - g.lgW));
  s.twsH = g.lgnmax - g.lgH;
  s.twsW = g.lgnmax - g.lgW;
  return s;
}

template <typename R>
__global__ void k_ct_to_c128(size_t n, Lay L, int W, const typename CT<R>::C* __restrict__ a, double2* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i % W);
    const auto v = a[L.at(y, x)];
    out[i] = make_double2((double)v.x, (double)v.y);
  }
}

// ---------------------------------------------------------------------------
// persistent skeleton: flattened (item, step) sequence per CTA, operands of
// step q+1 stream in (cp.async) while step q is transformed.

template <typename R, class Op>
__global__ void __launch_bounds__(512, 1) k_pass(Op op, StopFlag stop) {
  using C = typename CT<R>::C;
  if (stop && *stop) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  C* const b0 = reinterpret_cast<C*>(smraw);
  C* const b1 = b0 + op.bufE;
  C* extra = reinterpret_cast<C*>(smraw) + 2 * op.bufE;
  typename Op::State S{};
  int it = blockIdx.x;
  if (it >= op.nitems) return;
  int st = 0, par = 0;
  op.prefetch(it, 0, b0, extra);
  eng::cp_commit();
  while (true) {
    int nit = it, nst = st + 1;
    if (nst == op.steps(it)) { nst = 0; nit = it + gridDim.x; }
    const bool more = nit < op.nitems;
    if (more) op.prefetch(nit, nst, par ? b0 : b1, extra);
    eng::cp_commit();
    eng::cp_wait<1>();
    __syncthreads();
    C* const cur = par ? b1 : b0;
    if (st == 0) op.begin(S, it, extra);
    op.step(S, it, st, cur, extra);
    __syncthreads();
    if (st == op.steps(it) - 1) op.end(S, it, cur, extra);
    if (!more) break;
    it = nit;
    st = nst;
    par ^= 1;
  }
  op.finish(S, reinterpret_cast<double*>(smraw));
}

struct NoState {};
struct OpBase {
  int bufE = 0, nitems = 0;
  LS_D int steps(int) const { return 1; }
  template <class S, class C> LS_D void begin(S&, int, C*) const {}
  template <class S, class C> LS_D void end(S&, int, C*, C*) const {}
  template <class S> LS_D void finish(S&, double*) const {}
};

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
  struct F {
    const unsigned char* raw;
    int kind, y0, lgn;
    C* out;
    Lay L;
    LS_D C load(int seq, int idx) const {
      const int p = (seq << lgn) + idx;
      R m;
      if (kind == SRC_U8) m = (R)raw[p];
      else {
        const double v = reinterpret_cast<const double*>(raw)[p];
        m = kind == SRC_PHI ? (R)(v <= 0.0) : (R)v;
      }
      return cmk(m, (R)0);
    }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(y0 + seq, idx)] = v; }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    F f{reinterpret_cast<const unsigned char*>(b), kind, it << sh.lgR, sh.lgW, out, sh.ct()};
    eng::run_any<false, false>(sh.grow(), b, tw, f);
  }
};

// ---------------------------------------------------------------------------
// generic column transform: out = scale * FFT_y(in) (or IFFT_y), column-tiled in/out

template <typename R, typename RO, bool INV> struct ColsOp : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  using CO = typename CT<RO>::C;
  Shape<R> sh;
  const C* in;
  Lay Lin, Lout;
  CO* out;
  R scale;
  const C* tw;
  LS_D void prefetch(int it, int, C* b, C*) const {
    eng::gather_rect<sizeof(C)>(b, in, Lin, 0, sh.lgH, it << sh.lgS, sh.lgS);
  }
  struct F {
    const C* b;
    CO* out;
    Lay L;
    int x0, lgS;
    R scale;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<true>(seq, idx, lgS, 0)] * scale; }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(idx, x0 + seq)] = cmk((RO)v.x, (RO)v.y); }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    F f{b, out, Lout, it << sh.lgS, sh.lgS, scale};
    eng::run_any<true, INV>(sh.gcol(), b, tw, f);
  }
};

// generic row transform of a complex column-tiled field: out = FFT_x(in) (or IFFT_x)
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
  struct F {
    const C* b;
    C* out;
    Lay L;
    int y0, lgn;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<false>(seq, idx, 0, lgn)]; }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(y0 + seq, idx)] = v; }
  };
  template <class St> LS_D void step(St&, int it, int, C* b, C*) const {
    F f{b, out, Lout, it << sh.lgR, sh.lgW};
    eng::run_any<false, INV>(sh.grow(), b, tw, f);
  }
};

// ---------------------------------------------------------------------------
// per-set parameters of the kernel-looping passes

template <typename R> struct SetArgs {
  using C = typename CT<R>::C;
  int nsets;
  int nk[2];
  const C* spec[2];      // nk x field, column-tiled
  C* T[2];               // nk x field, column-tiled (T_k, then U_k in place)
  R* I[2];               // row-major intensity per set
  const R* gate[2];      // row-major gate per set
  C* V[2];               // column-tiled adjoint accumulator per set
  R w[2][kMaxK];         // kernel weights (sigma_k)
};

// F1: T_k = IFFT_y(M^ . H_k) / (HW)
template <typename R> struct F1Op : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  Shape<R> sh;
  SetArgs<R> a;
  const C* mhat;
  R scale;
  const C* tw;
  int lgnt;
  LS_D int steps(int it) const { return a.nk[it >> lgnt]; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = it >> lgnt, t = it & ((1 << lgnt) - 1);
    eng::gather_rect<sizeof(C)>(b, a.spec[set] + (size_t)k * fsz(), sh.ct(), 0, sh.lgH, t << sh.lgS, sh.lgS);
  }
  LS_D void begin(State&, int it, C* mh) const {
    const int t = it & ((1 << lgnt) - 1);
    eng::gather_rect<sizeof(C)>(mh, mhat, sh.ct(), 0, sh.lgH, t << sh.lgS, sh.lgS);
    eng::cp_commit();
    eng::cp_wait<0>();
    __syncthreads();
  }
  struct F {
    const C* b;
    const C* mh;
    C* out;
    Lay L;
    int x0, lgS;
    R scale;
    LS_D C load(int seq, int idx) const {
      const int p = eng::naddr<true>(seq, idx, lgS, 0);
      return cmul(mh[p], b[p]) * scale;
    }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(idx, x0 + seq)] = v; }
  };
  LS_D void step(State&, int it, int k, C* b, C* mh) const {
    const int set = it >> lgnt, t = it & ((1 << lgnt) - 1);
    F f{b, mh, a.T[set] + (size_t)k * fsz(), sh.ct(), t << sh.lgS, sh.lgS, scale};
    eng::run_any<true, true>(sh.gcol(), b, tw, f);
  }
};

// F2: I_set = sum_k w_k |IFFT_x T_k|^2, accumulated in registers, written once
template <typename R> struct F2Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { R acc[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  LS_D int steps(int it) const { return a.nk[it >> lgnb]; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = it >> lgnb, yb = it & ((1 << lgnb) - 1);
    eng::gather_rect<sizeof(C)>(b, a.T[set] + (size_t)k * fsz(), sh.ct(), yb << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  LS_D void begin(State& S, int, C*) const {
#pragma unroll
    for (int i = 0; i < P; ++i) S.acc[i] = (R)0;
  }
  struct F {
    const C* b;
    State& S;
    R w;
    int lgn;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<false>(seq, idx, 0, lgn)]; }
    LS_D void store(int, int, C v, int slot) { S.acc[slot] += w * (v.x * v.x + v.y * v.y); }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    F f{b, S, a.w[it >> lgnb][k], sh.lgW};
    eng::run_any<false, true>(sh.grow(), b, tw, f);
  }
  LS_D void end(State& S, int it, C*, C*) const {
    const int set = it >> lgnb, y0 = (it & ((1 << lgnb) - 1)) << sh.lgR;
    const Geo g = sh.grow();
    R* I = a.I[set];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      int seq, idx;
      eng::last_pos_any<false, C>(g, s, seq, idx);
      I[(size_t)(y0 + seq) * sh.W + idx] = S.acc[s];
    }
  }
};

// A1: U_k = FFT_x(gate . IFFT_x T_k), in place over T_k
template <typename R> struct A1Op : OpBase {
  using C = typename CT<R>::C;
  using State = NoState;
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnb;
  LS_D int steps(int it) const { return a.nk[it >> lgnb]; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = it >> lgnb, yb = it & ((1 << lgnb) - 1);
    eng::gather_rect<sizeof(C)>(b, a.T[set] + (size_t)k * fsz(), sh.ct(), yb << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  struct FInv {
    C* b;
    const R* gate;
    int y0, lgn, W;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<false>(seq, idx, 0, lgn)]; }
    LS_D void store(int seq, int idx, C v, int) {
      b[eng::naddr<false>(seq, idx, 0, lgn)] = v * __ldg(&gate[(size_t)(y0 + seq) * W + idx]);
    }
  };
  struct FFwd {
    const C* b;
    C* out;
    Lay L;
    int y0, lgn;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<false>(seq, idx, 0, lgn)]; }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(y0 + seq, idx)] = v; }
  };
  LS_D void step(State&, int it, int k, C* b, C*) const {
    const int set = it >> lgnb, yb = it & ((1 << lgnb) - 1);
    const int y0 = yb << sh.lgR;
    FInv fi{b, a.gate[set], y0, sh.lgW, sh.W};
    eng::run_any<false, true>(sh.grow(), b, tw, fi);
    __syncthreads();
    FFwd ff{b, a.T[set] + (size_t)k * fsz(), sh.ct(), y0, sh.lgW};
    eng::run_any<false, false>(sh.grow(), b, tw, ff);
  }
};

// A2: V_set = IFFT_y( sum_k w_k conj(H_k) . FFT_y U_k )
template <typename R> struct A2Op : OpBase {
  using C = typename CT<R>::C;
  static constexpr int P = eng::P_of<C>();
  struct State { C acc[P]; };
  Shape<R> sh;
  SetArgs<R> a;
  const C* tw;
  int lgnt;
  LS_D int steps(int it) const { return a.nk[it >> lgnt]; }
  LS_D size_t fsz() const { return (size_t)sh.H * sh.W; }
  LS_D void prefetch(int it, int k, C* b, C*) const {
    const int set = it >> lgnt, t = it & ((1 << lgnt) - 1);
    eng::gather_rect<sizeof(C)>(b, a.T[set] + (size_t)k * fsz(), sh.ct(), 0, sh.lgH, t << sh.lgS, sh.lgS);
  }
  LS_D void begin(State& S, int, C*) const {
#pragma unroll
    for (int i = 0; i < P; ++i) S.acc[i] = cmk((R)0, (R)0);
  }
  struct F {
    const C* b;
    State& S;
    const C (&h)[P];
    R w;
    int lgS;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<true>(seq, idx, lgS, 0)]; }
    LS_D void store(int, int, C v, int slot) { S.acc[slot] = S.acc[slot] + cmulc(v, h[slot]) * w; }
  };
  LS_D void step(State& S, int it, int k, C* b, C*) const {
    const int set = it >> lgnt, t = it & ((1 << lgnt) - 1);
    const int x0 = t << sh.lgS;
    const Geo g = sh.gcol();
    const C* spec = a.spec[set] + (size_t)k * fsz();
    const Lay L = sh.ct();
    C h[P];
#pragma unroll
    for (int s = 0; s < P; ++s) {
      int seq, idx;
      eng::last_pos_any<true, C>(g, s, seq, idx);
      h[s] = __ldg(&spec[L.at(idx, x0 + seq)]);
    }
    F f{b, S, h, a.w[set][k], sh.lgS};
    eng::run_any<true, false>(g, b, tw, f);
  }
  struct FOut {
    const C* b;
    C* out;
    Lay L;
    int x0, lgS;
    LS_D C load(int seq, int idx) const { return b[eng::naddr<true>(seq, idx, lgS, 0)]; }
    LS_D void store(int seq, int idx, C v, int) { out[L.at(idx, x0 + seq)] = v; }
  };
  LS_D void end(State& S, int it, C* b, C*) const {
    const int set = it >> lgnt, t = it & ((1 << lgnt) - 1);
    const Geo g = sh.gcol();
#pragma unroll
    for (int s = 0; s < P; ++s) {
      int seq, idx;
      eng::last_pos_any<true, C>(g, s, seq, idx);
      b[eng::naddr<true>(seq, idx, sh.lgS, 0)] = S.acc[s];
    }
    __syncthreads();
    FOut f{b, a.V[set], sh.ct(), t << sh.lgS, sh.lgS};
    eng::run_any<true, true>(sh.gcol(), b, tw, f);
    __syncthreads();
  }
};

// A3: out = scale * Re IFFT_x(V_0 [+ V_1]) (f64 row-major) + CG dot partials per CTA
template <typename R> struct A3Op : OpBase {
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
  LS_D void prefetch(int it, int, C* b, C*) const {
    eng::gather_rect<sizeof(C)>(b, V0, sh.ct(), it << sh.lgR, sh.lgR, 0, sh.lgW);
  }
  struct F {
    const C* b;
    const C* v1;  // second accumulator, read directly (column-tiled)
    Lay L;
    double scale;
    double* out;
    const double* vp;
    State& S;
    int y0, lgn, W;
    LS_D C load(int seq, int idx) const {
      const C x = b[eng::naddr<false>(seq, idx, 0, lgn)];
      return v1 ? x + __ldg(&v1[L.at(y0 + seq, idx)]) : x;
    }
    LS_D void store(int seq, int idx, C v, int) {
      const size_t p = (size_t)(y0 + seq) * W + idx;
      const double val = scale * (double)v.x;
      out[p] = val;
      if (vp) {
        const double q = vp[p];
        S.acc[0] += val * (val - q);
        S.acc[1] += q * q;
      }
    }
  };
  LS_D void step(State& S, int it, int, C* b, C*) const {
    F f{b, V1, sh.ct(), scale, out, vp, S, it << sh.lgR, sh.lgW, sh.W};
    eng::run_any<false, true>(sh.grow(), b, tw, f);
  }
  LS_D void finish(State& S, double* red) const {
    if (!vp) return;
    __syncthreads();
    block_sum<2>(S.acc, red);
    if (threadIdx.x == 0) {
      dots[2 * blockIdx.x] = S.acc[0];
      dots[2 * blockIdx.x + 1] = S.acc[1];
    }
  }
};

// ---------------------------------------------------------------------------
// launch plumbing

int num_sms() {
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
  const size_t smem = std::max((size_t)(2 + extra_bufs) * op.bufE * sizeof(C), (size_t)(64 * sizeof(double)));
  if (smem > 227 * 1024) throw std::runtime_error("spectral pass needs more than 227 KB of shared memory");
  auto kern = k_pass<R, Op>;
  static int per_sm = -1;
  static size_t per_sm_smem = 0;
  static int per_sm_threads = 0;
  if (per_sm < 0 || per_sm_smem != smem || per_sm_threads != threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
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

template <typename R> int col_threads(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return std::max(1, ((1 << sh.lgS) << sh.lgH) / eng::P_of<C>());
}
template <typename R> int row_threads(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return std::max(1, ((1 << sh.lgR) << sh.lgW) / eng::P_of<C>());
}
template <typename R> int col_bufE(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  return eng::buf_elems<C>(sh.H, 1 << sh.lgS);
}
template <typename R> int row_bufE(const Shape<R>& sh) {
  using C = typename CT<R>::C;
  // the mask pass stages raw f64 input (8 B/elem) in a complex buffer
  return std::max(eng::buf_elems<C>(sh.W, 1 << sh.lgR), (int)(((1 << sh.lgR) << sh.lgW) * 8 / sizeof(C)));
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
    a.I[i] = static_cast<R*>(sets[i].I);
    a.gate[i] = static_cast<const R*>(sets[i].gate);
    a.V[i] = static_cast<C*>(sets[i].V);
    for (int k = 0; k < sets[i].nk; ++k) a.w[i][k] = (R)sets[i].w[k];
  }
  return a;
}

// ---------------------------------------------------------------------------

template <typename R>
void mask_fft_impl(const Grid& g, const void* src, int kind, void* mhat, void* scratch, StopFlag stop,
                   cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  MaskRowsOp<R> mr;
  mr.sh = sh;
  mr.src = src;
  mr.kind = kind;
  mr.out = static_cast<C*>(scratch);
  mr.tw = static_cast<const C*>(g.tw);
  mr.bufE = row_bufE(sh);
  mr.nitems = g.H >> sh.lgR;
  launch_op<R>(mr, row_threads(sh), 0, stop, s);
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
void f1_impl(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  F1Op<R> f1;
  f1.sh = sh;
  f1.a = a;
  f1.mhat = static_cast<const C*>(mhat);
  f1.scale = (R)(1.0 / (double)g.n());
  f1.tw = static_cast<const C*>(g.tw);
  f1.lgnt = g.lgW - sh.lgS;
  f1.bufE = col_bufE(sh);
  f1.nitems = (1 << f1.lgnt) * nsets;
  launch_op<R>(f1, col_threads(sh), 1, stop, s);
}

template <typename R>
void f2_impl(const Grid& g, const SpecSet* sets, int nsets, double2* a0_out, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  F2Op<R> f2;
  f2.sh = sh;
  f2.a = a;
  f2.tw = static_cast<const C*>(g.tw);
  f2.lgnb = g.lgH - sh.lgR;
  f2.bufE = row_bufE(sh);
  f2.nitems = (1 << f2.lgnb) * nsets;
  launch_op<R>(f2, row_threads(sh), 0, stop, s);
  if (a0_out) {  // convolve(): A_0 = IFFT_x T_0 of the first set, to complex128 row-major
    RowsOp<R, true> ro;
    ro.sh = sh;
    ro.in = a.T[0];
    ro.Lin = sh.ct();
    ro.Lout = sh.rm();
    ro.out = static_cast<C*>(sets[0].V);
    ro.tw = static_cast<const C*>(g.tw);
    ro.bufE = row_bufE(sh);
    ro.nitems = g.H >> sh.lgR;
    launch_op<R>(ro, row_threads(sh), 0, stop, s);
    k_ct_to_c128<R><<<148 * 4, 256, 0, s>>>(g.n(), sh.rm(), g.W, static_cast<const C*>(sets[0].V), a0_out);
  }
}

template <typename R>
void a1_impl(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
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
void a2_impl(const Grid& g, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  SetArgs<R> a = set_args<R>(g, sets, nsets);
  A2Op<R> a2;
  a2.sh = sh;
  a2.a = a;
  a2.tw = static_cast<const C*>(g.tw);
  a2.lgnt = g.lgW - sh.lgS;
  a2.bufE = col_bufE(sh);
  a2.nitems = (1 << a2.lgnt) * nsets;
  launch_op<R>(a2, col_threads(sh), 0, stop, s);
}

template <typename R>
int finish_impl(const Grid& g, const void* V0, const void* V1, double scale, double* out, const double* vp,
                double* dots, StopFlag stop, cudaStream_t s) {
  using C = typename CT<R>::C;
  Shape<R> sh = shape_of<R>(g);
  A3Op<R> a3;
  a3.sh = sh;
  a3.V0 = static_cast<const C*>(V0);
  a3.V1 = static_cast<const C*>(V1);
  a3.tw = static_cast<const C*>(g.tw);
  a3.scale = scale;
  a3.out = out;
  a3.vp = vp;
  a3.dots = dots;
  a3.bufE = row_bufE(sh);
  a3.nitems = g.H >> sh.lgR;
  int grid = launch_op<R>(a3, row_threads(sh), 0, stop, s, finish_max_blocks());
  return vp ? grid : 0;
}

__global__ void k_embed(int K, int H, int W, const double2* __restrict__ coeffs, double2* out) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * K) return;
  int i = t / K, j = t % K;
  int y = ((i - K / 2) % H + H) % H;
  int x = ((j - K / 2) % W + W) % W;
  out[(size_t)y * W + x] = coeffs[t];
}

}  // namespace

// ============================================================================

int finish_max_blocks() { return 148 * 2; }

void launch_mask_fft(const Grid& g, const uint8_t* mu8, const double* mf, const double* phi, void* mhat,
                     void* scratch, StopFlag stop, cudaStream_t s) {
  const void* src = mu8 ? (const void*)mu8 : mf ? (const void*)mf : (const void*)phi;
  const int kind = mu8 ? SRC_U8 : mf ? SRC_F64 : SRC_PHI;
  if (g.prec == F64) mask_fft_impl<double>(g, src, kind, mhat, scratch, stop, s);
  else mask_fft_impl<float>(g, src, kind, mhat, scratch, stop, s);
}

void launch_f1(const Grid& g, const void* mhat, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
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
                          const double* vp, double* dots, StopFlag stop, cudaStream_t s) {
  if (g.prec == F64) return finish_impl<double>(g, V0, V1, scale, out, vp, dots, stop, s);
  return finish_impl<float>(g, V0, V1, scale, out, vp, dots, stop, s);
}

// K0: spectra in float64 (row pass then column pass), stored column-tiled in
// the plan's precision.  scratch, scratch2: >= H*W*16 bytes each.
void launch_kernel_spectra(const Grid& g, int nk, int K, const double* coeffs_dev, void* spec, void* scratch,
                           void* scratch2, cudaStream_t s) {
  Grid g64 = g;
  g64.prec = F64;
  g64.tw = g.tw64;
  Shape<double> sh = shape_of<double>(g64);
  const size_t n = g.n();
  const int lgS_out = g.prec == F64 ? sh.lgS : shape_of<float>(g).lgS;
  for (int k = 0; k < nk; ++k) {
    cudaMemsetAsync(scratch, 0, n * sizeof(double2), s);
    const int nt = K * K;
    k_embed<<<(nt + 255) / 256, 256, 0, s>>>(K, g.H, g.W, reinterpret_cast<const double2*>(coeffs_dev) + (size_t)k * nt,
                                            static_cast<double2*>(scratch));
    RowsOp<double, false> rr;
    rr.sh = sh;
    rr.in = static_cast<const double2*>(scratch);
    rr.Lin = sh.rm();
    rr.Lout = sh.ct();
    rr.out = static_cast<double2*>(scratch2);
    rr.tw = static_cast<const double2*>(g.tw64);
    rr.bufE = row_bufE(sh);
    rr.nitems = g.H >> sh.lgR;
    launch_op<double>(rr, row_threads(sh), 0, nullptr, s);
    if (g.prec == F64) {
      ColsOp<double, double, false> cc;
      cc.sh = sh;
      cc.in = static_cast<const double2*>(scratch2);
      cc.Lin = sh.ct();
      cc.Lout = Lay{g.H, lgS_out};
      cc.out = static_cast<double2*>(spec) + (size_t)k * n;
      cc.scale = 1.0;
      cc.tw = static_cast<const double2*>(g.tw64);
      cc.bufE = col_bufE(sh);
      cc.nitems = g.W >> sh.lgS;
      launch_op<double>(cc, col_threads(sh), 0, nullptr, s);
    } else {
      ColsOp<double, float, false> cc;
      cc.sh = sh;
      cc.in = static_cast<const double2*>(scratch2);
      cc.Lin = sh.ct();
      cc.Lout = Lay{g.H, lgS_out};
      cc.out = static_cast<float2*>(spec) + (size_t)k * n;
      cc.scale = 1.0;
      cc.tw = static_cast<const double2*>(g.tw64);
      cc.bufE = col_bufE(sh);
      cc.nitems = g.W >> sh.lgS;
      launch_op<double>(cc, col_threads(sh), 0, nullptr, s);
    }
  }
}

// spectrum field (plan precision, column-tiled) -> complex128 row-major
void launch_spec_to_c128(const Grid& g, const void* field, double* out, cudaStream_t s) {
  if (g.prec == F64) {
    Lay L{g.H, shape_of<double>(g).lgS};
    k_ct_to_c128<double><<<148 * 4, 256, 0, s>>>(g.n(), L, g.W, static_cast<const double2*>(field),
                                                   reinterpret_cast<double2*>(out));
  } else {
    Lay L{g.H, shape_of<float>(g).lgS};
    k_ct_to_c128<float><<<148 * 4, 256, 0, s>>>(g.n(), L, g.W, static_cast<const float2*>(field),
                                                  reinterpret_cast<double2*>(out));
  }
}

}  // namespace lsb
