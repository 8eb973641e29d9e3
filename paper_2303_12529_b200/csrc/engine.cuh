// Pipelined shared-memory FFT engine for the DSO spectral passes.
//
// A pass is a persistent kernel: each CTA walks a static list of work items
// (a block of columns or rows of one field, times the kernels of one SOCS
// set) and, for every (item, step), transforms S sequences of length
// n = 2^lgn that sit in a shared-memory stage buffer.  While step q is being
// transformed, the operands of step q+1 are already streaming into the other
// stage buffer with cp.async (Ampere+ LDGSTS, 16 B per op), so HBM traffic of
// the next step overlaps the butterflies of this one.  Pointwise work before
// and after each 1-D transform (spectral products, |A|^2 accumulation,
// resist gates, conj(H) accumulation) lives in the load / store functors of
// the first and last butterfly stage and never costs an extra pass over HBM.
//
// Layouts.  Every field is stored "column-tiled": element (y, x) of an H x W
// field with tile width w lives at ((x / w) * H + y) * w + x % w.  w = W is
// plain row-major; w = S (the column-pass width) makes one column item a
// single contiguous block and one row item a set of R*w-element contiguous
// chunks (128 B for the FP32 tier at 2048^2).
//
// Thread -> data maps inside a buffer (natural, unpadded, as loaded):
//   COLS: buffer is [n][S] (sequence = column, fast index = column)
//   ROWS: buffer is [S][n] (sequence = row)
// Intermediate butterfly stages exchange through the same buffer with a
// padded address map (one pad slot every 16 / 8 elements) to avoid bank
// conflicts.  Radix-16 stages for complex64 (16 values per thread), radix-8
// for complex128 (8 values per thread).
#pragma once
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace eng {

// 16 complex values per thread in both precisions (radix-16 stages); a CTA
// is 512 threads for complex64 (<= 128 registers) and 256 threads for
// complex128 (<= 255 registers), i.e. 64 KB of operands per stage buffer.
#ifndef LSB_C128_LGP  // experiment builds may give complex128 8 values per thread (-DLSB_C128_LGP=3: 512 threads)
#define LSB_C128_LGP 4
#endif
template <typename C> constexpr int LGP_of() { return sizeof(C) == 8 ? 4 : LSB_C128_LGP; }
template <typename C> constexpr int P_of() { return 1 << LGP_of<C>(); }
#ifndef LSB_C64_THREADS  // experiment builds may shrink the complex64 CTA (LSB_DEFINES=-DLSB_C64_THREADS=256)
#define LSB_C64_THREADS 512
#endif
template <typename C> constexpr int cta_threads() { return sizeof(C) == 8 ? LSB_C64_THREADS : 4096 / P_of<C>(); }

// ---- radix-R DFTs in registers, forward sign (exp(-2 pi i rk/R)), natural order out

template <typename C> LS_D void dft2(C& a, C& b) {
  C t = a - b;
  a = a + b;
  b = t;
}

template <typename C> LS_D void dft4(C& x0, C& x1, C& x2, C& x3) {
  C s02 = x0 + x2, d02 = x0 - x2, s13 = x1 + x3, d13 = mul_mi(x1 - x3);
  x0 = s02 + s13;
  x2 = s02 - s13;
  x1 = d02 + d13;
  x3 = d02 - d13;
}

template <typename C, typename R> LS_D C rot(C a, R c, R s) {  // a * (c + i s)
  return cmk(a.x * c - a.y * s, a.x * s + a.y * c);
}

template <typename C> LS_D void dft8(C* v) {
  using R = decltype(v[0].x);
  const R h = (R)0.70710678118654752440084436210484903928;
  dft4(v[0], v[2], v[4], v[6]);
  dft4(v[1], v[3], v[5], v[7]);
  C y1 = rot(v[3], h, -h);
  C y2 = mul_mi(v[5]);
  C y3 = rot(v[7], -h, -h);
  C y0 = v[1];
  C x0 = v[0], x1 = v[2], x2 = v[4], x3 = v[6];
  v[0] = x0 + y0; v[4] = x0 - y0;
  v[1] = x1 + y1; v[5] = x1 - y1;
  v[2] = x2 + y2; v[6] = x2 - y2;
  v[3] = x3 + y3; v[7] = x3 - y3;
}

template <typename C> LS_D void dft16(C* v) {
  using R = decltype(v[0].x);
  const R c1 = (R)0.92387953251128675612818318939678828682;  // cos(pi/8)
  const R s1 = (R)0.38268343236508977172845998403039886676;  // sin(pi/8)
  const R h = (R)0.70710678118654752440084436210484903928;
  dft4(v[0], v[4], v[8], v[12]);
  dft4(v[1], v[5], v[9], v[13]);
  dft4(v[2], v[6], v[10], v[14]);
  dft4(v[3], v[7], v[11], v[15]);
  v[5] = rot(v[5], c1, -s1);
  v[9] = rot(v[9], h, -h);
  v[13] = rot(v[13], s1, -c1);
  v[6] = rot(v[6], h, -h);
  v[10] = mul_mi(v[10]);
  v[14] = rot(v[14], -h, -h);
  v[7] = rot(v[7], s1, -c1);
  v[11] = rot(v[11], -h, -h);
  v[15] = rot(v[15], -c1, s1);
  C t[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i] = v[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    C a0 = t[4 * k1 + 0], a1 = t[4 * k1 + 1], a2 = t[4 * k1 + 2], a3 = t[4 * k1 + 3];
    dft4(a0, a1, a2, a3);
    v[k1] = a0;
    v[k1 + 4] = a1;
    v[k1 + 8] = a2;
    v[k1 + 12] = a3;
  }
}

template <int RAD, typename C> LS_D void dft(C* v) {
  if constexpr (RAD == 2) dft2(v[0], v[1]);
  else if constexpr (RAD == 4) dft4(v[0], v[1], v[2], v[3]);
  else if constexpr (RAD == 8) dft8(v);
  else dft16(v);
}

// ---- buffer geometry ---------------------------------------------------------

template <typename C> constexpr int pad_shift() { return 4; }  // 1 pad element per 16: 16j+r -> 17j+r, conflict-free first-stage writes for 8- and 16-byte elements
template <typename C> LS_HD int padded(int i) { return i + (i >> pad_shift<C>()); }
template <typename C> LS_HD int padded_len(int n) { return n + (n >> pad_shift<C>()) + 1; }
// elements of one stage buffer holding S sequences of length n (natural or padded)
template <typename C> LS_HD int buf_elems(int n, int S) { return padded_len<C>(n) * S; }

struct Geo {
  int lgn;  // log2 sequence length
  int lgS;  // log2 sequences per buffer
  int tws;  // log2(twiddle table length / n)
};

template <typename C, bool COLS> LS_D int xaddr(int seq, int idx, int lgS, int ld) {
  if constexpr (COLS) return (padded<C>(idx) << lgS) + seq;
  else return seq * ld + padded<C>(idx);
}
// natural (as-loaded) position of (seq, idx) in a buffer
template <bool COLS> LS_D int naddr(int seq, int idx, int lgS, int lgn) {
  if constexpr (COLS) return (idx << lgS) + seq;
  else return (seq << lgn) + idx;
}

LS_HD int num_stages(int lgn, int lgp) { return (lgn + lgp - 1) / lgp; }
LS_HD int stage_bits(int lgn, int lgp, int s) {
  int nst = num_stages(lgn, lgp);
  int base = lgn / nst, extra = lgn - base * nst;
  return base + (s < extra ? 1 : 0);
}

// One radix-RAD Stockham stage over the buffer's S sequences.  FIRST reads
// through f.load<STRIDE>(seq, j, r) and LAST writes through
// f.store<STRIDE>(seq, j, r, value, slot), both for index idx = j + r*STRIDE
// (STRIDE is a compile-time constant on the fast path, 0 = "j is the index"
// on the generic path), so functors can fold addresses to base + r*const.
// slot = i*RAD + r is stable per thread across calls of the same geometry
// (accumulators can live in registers).  Inverse transforms use
// conj(FFT(conj x)), unnormalised.  The read and write phases of every stage
// are separated by a barrier, so load/store functors may use the buffer
// itself (in-place).
template <int RAD, bool FIRST, bool LAST, bool COLS, bool INV, typename C, class F>
LS_D void stage(C (&v)[P_of<C>()], const Geo& g, int lgNs, C* sm, const C* __restrict__ tw, F& f) {
  constexpr int LGR = RAD == 2 ? 1 : RAD == 4 ? 2 : RAD == 8 ? 3 : 4;
  constexpr int P = P_of<C>();
  const int n = 1 << g.lgn;
  const int nr = n >> LGR;
  const int nt = blockDim.x;
  const int ld = padded_len<C>(n);
  const int Ns = 1 << lgNs;
  const int S = 1 << g.lgS;
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * nt;
    int seq, j;
    if constexpr (COLS) { seq = b & (S - 1); j = b >> g.lgS; }
    else { j = b & (nr - 1); seq = b >> (g.lgn - LGR); }
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      const int idx = j + r * nr;
      C x;
      if constexpr (FIRST) {
        x = f.template load<0>(seq, idx, 0, i * RAD + r);
        if constexpr (INV) x = cconj(x);
      } else {
        x = sm[xaddr<C, COLS>(seq, idx, g.lgS, ld)];
      }
      v[i * RAD + r] = x;
    }
    if constexpr (!FIRST) {
      const int k = j & (Ns - 1);
      const int sh = g.lgn - lgNs - LGR + g.tws;
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[i * RAD + r] = cmul(v[i * RAD + r], __ldg(&tw[(r * k) << sh]));
    }
    dft<RAD>(&v[i * RAD]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * nt;
    int seq, j;
    if constexpr (COLS) { seq = b & (S - 1); j = b >> g.lgS; }
    else { j = b & (nr - 1); seq = b >> (g.lgn - LGR); }
    const int base = ((j >> lgNs) << (lgNs + LGR)) + (j & (Ns - 1));
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      const int idx = base + r * Ns;
      C x = v[i * RAD + r];
      if constexpr (LAST) {
        if constexpr (INV) x = cconj(x);
        f.template store<0>(seq, idx, 0, x, i * RAD + r);
      } else {
        sm[xaddr<C, COLS>(seq, idx, g.lgS, ld)] = x;
      }
    }
  }
  if constexpr (!LAST) __syncthreads();
}

template <bool FIRST, bool LAST, bool COLS, bool INV, typename C, class F>
LS_D void stage_rt(int bits, C (&v)[P_of<C>()], const Geo& g, int lgNs, C* sm, const C* tw, F& f) {
  switch (bits) {
    case 1: stage<2, FIRST, LAST, COLS, INV>(v, g, lgNs, sm, tw, f); break;
    case 2: stage<4, FIRST, LAST, COLS, INV>(v, g, lgNs, sm, tw, f); break;
    case 3: stage<8, FIRST, LAST, COLS, INV>(v, g, lgNs, sm, tw, f); break;
    default:
      if constexpr (P_of<C>() >= 16) stage<16, FIRST, LAST, COLS, INV>(v, g, lgNs, sm, tw, f);
      break;
  }
}

// Full 1-D transform of the buffer's S sequences (blockDim.x == S*n/P).
// On return every thread has passed the final store; callers that reuse the
// buffer must __syncthreads() first.
template <bool COLS, bool INV, typename C, class F>
LS_D void run(const Geo& g, C* sm, const C* __restrict__ tw, F& f) {
  constexpr int LGP = LGP_of<C>();
  C v[P_of<C>()];
  const int nst = num_stages(g.lgn, LGP);
  if (nst == 1) {
    stage_rt<true, true, COLS, INV>(stage_bits(g.lgn, LGP, 0), v, g, 0, sm, tw, f);
    return;
  }
  int lgNs = 0;
  int b0 = stage_bits(g.lgn, LGP, 0);
  stage_rt<true, false, COLS, INV>(b0, v, g, 0, sm, tw, f);
  lgNs += b0;
  for (int s = 1; s < nst - 1; ++s) {
    int bs = stage_bits(g.lgn, LGP, s);
    stage_rt<false, false, COLS, INV>(bs, v, g, lgNs, sm, tw, f);
    lgNs += bs;
  }
  stage_rt<false, true, COLS, INV>(stage_bits(g.lgn, LGP, nst - 1), v, g, lgNs, sm, tw, f);
}

// (seq, idx) written by slot `slot` of this thread in the LAST stage of run()
template <bool COLS, typename C>
LS_D void last_pos(const Geo& g, int slot, int& seq, int& idx) {
  constexpr int LGP = LGP_of<C>();
  const int nst = num_stages(g.lgn, LGP);
  const int lgr = stage_bits(g.lgn, LGP, nst - 1);
  const int rad = 1 << lgr;
  const int i = slot >> lgr, r = slot & (rad - 1);
  const int b = threadIdx.x + i * blockDim.x;
  const int nr = (1 << g.lgn) >> lgr;
  int j;
  if constexpr (COLS) { seq = b & ((1 << g.lgS) - 1); j = b >> g.lgS; }
  else { j = b & (nr - 1); seq = b >> (g.lgn - lgr); }
  idx = j + r * nr;  // last stage: Ns == nr, base == j
}
// number of slots a thread owns in the last stage (= P, or fewer when the
// last stage radix does not divide P evenly -- never: P/RAD*RAD == P)
template <typename C> constexpr int nslots() { return P_of<C>(); }

// ---- compile-time geometry fast path ------------------------------------------
// Used when the buffer is full (S * n == 512 * P, blockDim.x == 512): every
// index expression folds to shifts and immediate offsets, and each non-first
// stage loads ONE twiddle per butterfly from the table and derives the other
// RAD-2 powers by binary splitting (depth <= 4 multiplications), keeping the
// shared-memory / L1 pipe free for the data exchange.

template <int LGN, int LGP> struct StagePlan {
  static constexpr int nst = (LGN + LGP - 1) / LGP;
  static constexpr int bits(int s) { return LGN / nst + (s < LGN - (LGN / nst) * nst ? 1 : 0); }
  static constexpr int before(int s) { return s == 0 ? 0 : before(s - 1) + bits(s - 1); }
};

template <int RAD, typename C> LS_D void apply_twiddles(C* v, C w1) {
  if constexpr (RAD >= 2) v[1] = cmul(v[1], w1);
  if constexpr (RAD >= 4) {
    const C w2 = cmul(w1, w1), w3 = cmul(w2, w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    if constexpr (RAD >= 8) {
      const C w4 = cmul(w2, w2), w5 = cmul(w4, w1), w6 = cmul(w4, w2), w7 = cmul(w4, w3);
      v[4] = cmul(v[4], w4);
      v[5] = cmul(v[5], w5);
      v[6] = cmul(v[6], w6);
      v[7] = cmul(v[7], w7);
      if constexpr (RAD >= 16) {
        const C w8 = cmul(w4, w4);
        v[8] = cmul(v[8], w8);
        v[9] = cmul(v[9], cmul(w8, w1));
        v[10] = cmul(v[10], cmul(w8, w2));
        v[11] = cmul(v[11], cmul(w8, w3));
        v[12] = cmul(v[12], cmul(w8, w4));
        v[13] = cmul(v[13], cmul(w8, w5));
        v[14] = cmul(v[14], cmul(w8, w6));
        v[15] = cmul(v[15], cmul(w8, w7));
      }
    }
  }
}

template <typename C> constexpr int padg() { return 1 << pad_shift<C>(); }
template <typename C> constexpr int cpadded(int i) { return i + (i >> pad_shift<C>()); }

// exchange address of (seq, idx) with idx = base + r * stride, split so that
// the r-dependent part is an immediate when `stride` is a multiple of the pad group
template <typename C, bool COLS, int LGS, int LD, int STRIDE>
LS_D int xaddr_t(int seq, int base, int r) {
  int pidx;
  if constexpr (STRIDE % padg<C>() == 0) pidx = padded<C>(base) + r * cpadded<C>(STRIDE);
  else pidx = padded<C>(base + r * STRIDE);
  if constexpr (COLS) return (pidx << LGS) + seq;
  else return seq * LD + pidx;
}

// optional functor hook run by every thread just before the last stage's
// stores (e.g. waiting for an operand the stores consume)
template <class F, class = void> struct has_pre_store : std::false_type {};
template <class F> struct has_pre_store<F, std::void_t<decltype(std::declval<F&>().pre_store())>> : std::true_type {};

template <int LGN, int LGS, int LGR, int LGNS, bool FIRST, bool LAST, bool COLS, bool INV, typename C, class F>
LS_D void stage_t(C (&v)[P_of<C>()], C* sm, const C* __restrict__ tw, int tws, F& f) {
  constexpr int RAD = 1 << LGR, P = P_of<C>();
  constexpr int n = 1 << LGN, nr = n >> LGR, S = 1 << LGS, Ns = 1 << LGNS;
  constexpr int NT = (n << LGS) / P;
  constexpr int LD = n + (n >> pad_shift<C>()) + 1;
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * NT;
    int seq, j;
    if constexpr (COLS) { seq = b & (S - 1); j = b >> LGS; }
    else { j = b & (nr - 1); seq = b >> (LGN - LGR); }
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      C x;
      if constexpr (FIRST) {
        x = f.template load<nr>(seq, j, r, i * RAD + r);
        if constexpr (INV) x = cconj(x);
      } else {
        x = sm[xaddr_t<C, COLS, LGS, LD, nr>(seq, j, r)];
      }
      v[i * RAD + r] = x;
    }
    if constexpr (!FIRST) {
      const int k = j & (Ns - 1);
      apply_twiddles<RAD>(&v[i * RAD], __ldg(&tw[k << (LGN - LGNS - LGR + tws)]));
    }
    dft<RAD>(&v[i * RAD]);
  }
  __syncthreads();
  if constexpr (LAST && has_pre_store<F>::value) f.pre_store();
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * NT;
    int seq, j;
    if constexpr (COLS) { seq = b & (S - 1); j = b >> LGS; }
    else { j = b & (nr - 1); seq = b >> (LGN - LGR); }
    const int base = ((j >> LGNS) << (LGNS + LGR)) + (j & (Ns - 1));
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      C x = v[i * RAD + r];
      if constexpr (LAST) {
        if constexpr (INV) x = cconj(x);
        f.template store<Ns>(seq, base, r, x, i * RAD + r);
      } else {
        sm[xaddr_t<C, COLS, LGS, LD, Ns>(seq, base, r)] = x;
      }
    }
  }
  if constexpr (!LAST) __syncthreads();
}

template <int LGN, int LGS, int SI, bool COLS, bool INV, typename C, class F>
LS_D void run_stages(C (&v)[P_of<C>()], C* sm, const C* tw, int tws, F& f) {
  using PL = StagePlan<LGN, LGP_of<C>()>;
  constexpr int LGR = PL::bits(SI), LGNS = PL::before(SI);
  stage_t<LGN, LGS, LGR, LGNS, SI == 0, SI == PL::nst - 1, COLS, INV>(v, sm, tw, tws, f);
  if constexpr (SI + 1 < PL::nst) run_stages<LGN, LGS, SI + 1, COLS, INV>(v, sm, tw, tws, f);
}

template <typename C> constexpr int lg_full() { return sizeof(C) == 8 && LSB_C64_THREADS == 512 ? 13 : 12; }  // log2(cta_threads * P)
constexpr int kFastMinLgn = 8;

// (seq, idx) of slot `slot` in the last stage (fast path)
template <int LGN, int LGS, bool COLS, typename C>
LS_D void last_pos_t(int slot, int& seq, int& idx) {
  using PL = StagePlan<LGN, LGP_of<C>()>;
  constexpr int LGR = PL::bits(PL::nst - 1), RAD = 1 << LGR, nr = (1 << LGN) >> LGR;
  constexpr int NT = ((1 << LGN) << LGS) / P_of<C>();
  const int i = slot >> LGR, r = slot & (RAD - 1);
  const int b = threadIdx.x + i * NT;
  int j;
  if constexpr (COLS) { seq = b & ((1 << LGS) - 1); j = b >> LGS; }
  else { j = b & (nr - 1); seq = b >> (LGN - LGR); }
  idx = j + r * nr;
}

// Compile-time geometry handle passed to op bodies: LGN > 0 on the fast path
// (LGS = log2(512 P) - LGN), LGN == 0 on the runtime-geometry path.
template <int LGN_> struct Fix { static constexpr int LGN = LGN_; };

// Calls body(Fix<LGN>{}) once with the geometry folded to constants when the
// buffer is full and n >= 256 (every production size), else body(Fix<0>{}).
#define ENG_FAST_CASES(X) X(8) X(9) X(10) X(11) X(12) X(13)
template <typename C, class Body>
LS_D void dispatch(const Geo& g, bool allow, Body&& body) {
  constexpr int LGE = lg_full<C>();
  if (allow && g.lgS == LGE - g.lgn && g.lgn >= kFastMinLgn) {
    switch (g.lgn) {
#define ENG_CASE(L) \
  case L: if constexpr (L <= LGE) { body(Fix<L>{}); return; } break;
      ENG_FAST_CASES(ENG_CASE)
#undef ENG_CASE
      default: break;
    }
  }
  body(Fix<0>{});
}

// Run the transform with the geometry chosen by dispatch().
template <int LGN, bool COLS, bool INV, typename C, class F>
LS_D void run_fix(const Geo& g, C* sm, const C* __restrict__ tw, F& f) {
  if constexpr (LGN > 0) {
    C v[P_of<C>()];
    run_stages<LGN, lg_full<C>() - LGN, 0, COLS, INV>(v, sm, tw, g.tws, f);
  } else {
    run<COLS, INV>(g, sm, tw, f);
  }
}

// Calls fn(seq, j, r, slot) for every slot this thread reads in the FIRST
// stage (the load functor's arguments), fast path only.
template <int LGN, bool COLS, typename C, class Fn>
LS_D void for_first_slots(Fn&& fn) {
  constexpr int P = P_of<C>();
  using PL = StagePlan<LGN, LGP_of<C>()>;
  constexpr int LGR = PL::bits(0), RAD = 1 << LGR, nr = (1 << LGN) >> LGR;
  constexpr int LGS = lg_full<C>() - LGN;
  constexpr int NT = ((1 << LGN) << LGS) / P;
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * NT;
    int seq, j;
    if constexpr (COLS) { seq = b & ((1 << LGS) - 1); j = b >> LGS; }
    else { j = b & (nr - 1); seq = b >> (LGN - LGR); }
#pragma unroll
    for (int r = 0; r < RAD; ++r) fn.template operator()<nr>(seq, j, r, i * RAD + r);
  }
}

// Calls fn(seq, j, r, slot) for every slot this thread owns in the LAST
// stage (idx = j + r*STRIDE with STRIDE passed as a template argument of fn's
// call operator via Fix-like constant).  Mirrors stage_t / stage exactly.
template <int LGN, bool COLS, typename C, class Fn>
LS_D void for_last_slots(const Geo& g, Fn&& fn) {
  constexpr int P = P_of<C>();
  if constexpr (LGN > 0) {
    using PL = StagePlan<LGN, LGP_of<C>()>;
    constexpr int LGR = PL::bits(PL::nst - 1), RAD = 1 << LGR, nr = (1 << LGN) >> LGR;
    constexpr int LGS = lg_full<C>() - LGN;
    constexpr int NT = ((1 << LGN) << LGS) / P;
#pragma unroll
    for (int i = 0; i < P / RAD; ++i) {
      const int b = threadIdx.x + i * NT;
      int seq, j;
      if constexpr (COLS) { seq = b & ((1 << LGS) - 1); j = b >> LGS; }
      else { j = b & (nr - 1); seq = b >> (LGN - LGR); }
#pragma unroll
      for (int r = 0; r < RAD; ++r) fn.template operator()<nr>(seq, j, r, i * RAD + r);
    }
  } else {
#pragma unroll
    for (int s = 0; s < P; ++s) {
      int seq, idx;
      last_pos<COLS, C>(g, s, seq, idx);
      fn.template operator()<0>(seq, idx, 0, s);
    }
  }
}

// ---- layouts -----------------------------------------------------------------

// column-tiled layout: (y, x) -> ((x >> lgw) * H + y) << lgw | (x & (w-1))
struct Lay {
  int H, lgw;
  LS_HD size_t at(int y, int x) const {
    return ((((size_t)(x >> lgw) * H + y)) << lgw) | (size_t)(x & ((1 << lgw) - 1));
  }
};

// ---- cp.async ------------------------------------------------------------------

LS_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
LS_D void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
LS_D void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
LS_D void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
LS_D void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> LS_D void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Copy the rectangle [y0, y0+ny) x [x0, x0+nx) of a column-tiled field
// (element size ES bytes) into shared memory as a row-major [ny][nx] array.
// All threads of the CTA participate; pieces are enumerated in source-address
// order (tile, row, chunk) so a warp reads contiguous memory.
template <int ES> constexpr int lg_es() { return ES == 1 ? 0 : ES == 2 ? 1 : ES == 4 ? 2 : ES == 8 ? 3 : 4; }

// all extents are powers of two (log2 arguments)
template <int ES>
LS_D void gather_rect(void* dst, const void* src, Lay L, int y0, int lgny, int x0, int lgnx) {
  constexpr int LGES = lg_es<ES>();
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const int nt = blockDim.x;
  // (a) the rectangle is whole tiles of full tile width (column items, or a
  //     row-major source): each tile chunk of ny*w elements is contiguous.
  if (lgnx >= L.lgw && L.lgw + LGES >= 4) {
    const int lgw = L.lgw;
    const int lgppt = lgny + lgw + LGES - 4;          // 16 B pieces per tile chunk
    const int total = 1 << (lgnx - lgw + lgppt);
    if (lgnx == lgw) {                                // single tile: plain copy
      const char* s0 = s + ((L.at(y0, x0)) << LGES);
      for (int p = threadIdx.x; p < total; p += nt) cp16(d + ((size_t)p << 4), s0 + ((size_t)p << 4));
      return;
    }
    if (nt >= (1 << lgppt)) {                         // each thread keeps its offset inside a chunk
      const int rem = threadIdx.x & ((1 << lgppt) - 1);
      const int e = rem << (4 - LGES);                // element offset inside the chunk
      const int r = e >> lgw, c = e & ((1 << lgw) - 1);
      int t = threadIdx.x >> lgppt;
      const int tstep = nt >> lgppt;
      const char* sp = s + ((L.at(y0 + r, x0 + (t << lgw) + c)) << LGES);
      char* dp = d + ((((size_t)r << lgnx) + (t << lgw) + c) << LGES);
      const size_t sstride = ((size_t)tstep * L.H) << (lgw + LGES);
      const size_t dstride = (size_t)tstep << (lgw + LGES);
      for (int p = threadIdx.x; p < total; p += nt) {
        cp16(dp, sp);
        sp += sstride;
        dp += dstride;
      }
      return;
    }
  }
  // (b) a slab narrower than one tile (column items of a wider tiling): one
  //     contiguous row segment of nx elements per row, 16 B pieces
  if (lgnx < L.lgw && lgnx + LGES >= 4) {
    const int lgprs = lgnx + LGES - 4;                // pieces per row segment
    const int total = 1 << (lgny + lgprs);
    const char* s0 = s + ((L.at(y0, x0)) << LGES);
    const int lgrow = L.lgw + LGES;                   // bytes per tile row
    for (int p = threadIdx.x; p < total; p += nt) {
      const int r = p >> lgprs, cc = p & ((1 << lgprs) - 1);
      cp16(d + ((size_t)p << 4), s0 + ((size_t)r << lgrow) + (cc << 4));
    }
    return;
  }
  // (c) general: pieces in source-address order (tile, row, chunk)
  const int lgwc = lgnx < L.lgw ? lgnx : L.lgw;      // columns per tile chunk
  int lgpb = lgwc + LGES;                            // bytes per contiguous row segment
  lgpb = lgpb > 4 ? 4 : lgpb;
  const int lgepp = lgpb - LGES > 0 ? lgpb - LGES : 0;  // elements per piece
  const int lgprs = lgwc - lgepp;                    // pieces per row segment
  const int lgppt = lgny + lgprs;                    // pieces per tile chunk
  const int total = 1 << (lgnx - lgwc + lgppt);
  for (int p = threadIdx.x; p < total; p += nt) {
    const int t = p >> lgppt, rem = p & ((1 << lgppt) - 1);
    const int r = rem >> lgprs, c = ((rem & ((1 << lgprs) - 1)) << lgepp) + (t << lgwc);
    const size_t so = L.at(y0 + r, x0 + c) << LGES;
    const size_t dof = (((size_t)r << lgnx) + c) << LGES;
    if (lgpb == 4) cp16(d + dof, s + so);
    else if (lgpb == 3) cp8(d + dof, s + so);
    else cp4(d + dof, s + so);
  }
}

}  // namespace eng
