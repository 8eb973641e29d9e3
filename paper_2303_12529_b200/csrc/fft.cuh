// Shared-memory Stockham FFT engine for power-of-two lengths (2 .. 8192).
//
// One CTA transforms `nb` independent sequences of length n = 2^lgn with
// every thread holding P = 16 complex values in registers.  A transform is
// ceil(lgn/4) radix-2^b stages (b <= 4); stage 0 gathers straight from the
// caller's load functor (global memory, coalesced), the last stage scatters
// straight to the caller's store functor (natural order, coalesced), and the
// stages in between exchange through padded shared memory.  Pointwise work
// on either side of a transform (mask threshold, spectral products, |A|^2
// accumulation, gates, accumulation of the adjoint spectrum) lives in the
// functors, so it never costs an extra pass over HBM.
//
// Two thread->data maps:
//   ROWS (SEQ_FAST=false): sequences are rows of a row-major [H][W] grid;
//     consecutive threads walk along a row.
//   COLS (SEQ_FAST=true):  sequences are columns; consecutive threads walk
//     across the nb adjacent columns first, so each warp reads nb*sizeof(C)
//     contiguous bytes per row (>= one 32 B sector for nb*sizeof(C) >= 32).
//
// Inverse transforms use conj(FFT(conj(x))) (unnormalised); the caller folds
// the 1/(HW) factor of numpy.fft.ifft2 into its epilogue.
#pragma once
#include "common.cuh"

namespace fft {

// complex values held per thread: 16 for complex64 (radix <= 16), 8 for
// complex128 (radix <= 8), keeping the register file at <= 64 regs/thread so
// two 512-thread CTAs fit per SM.
template <typename C> constexpr int P_of() { return sizeof(C) == 8 ? 16 : 8; }
template <typename C> constexpr int LGP_of() { return sizeof(C) == 8 ? 4 : 3; }

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
  // Y1[k1] *= W8^k1 ; Y0 lives in v[0],v[2],v[4],v[6] as k1 = 0..3
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
  // stage 1: for b = 0..3, DFT4 over a of x[4a + b] -> Y_b[k1] stored in v[4a+b] slot k1=a
  dft4(v[0], v[4], v[8], v[12]);
  dft4(v[1], v[5], v[9], v[13]);
  dft4(v[2], v[6], v[10], v[14]);
  dft4(v[3], v[7], v[11], v[15]);
  // twiddles W16^{b k1}: element Y_b[k1] sits at v[4*k1 + b]
  v[5] = rot(v[5], c1, -s1);    // b=1,k1=1: W^1
  v[9] = rot(v[9], h, -h);      // b=1,k1=2: W^2
  v[13] = rot(v[13], s1, -c1);  // b=1,k1=3: W^3
  v[6] = rot(v[6], h, -h);      // b=2,k1=1: W^2
  v[10] = mul_mi(v[10]);        // b=2,k1=2: W^4
  v[14] = rot(v[14], -h, -h);   // b=2,k1=3: W^6
  v[7] = rot(v[7], s1, -c1);    // b=3,k1=1: W^3
  v[11] = rot(v[11], -h, -h);   // b=3,k1=2: W^6
  v[15] = rot(v[15], -c1, s1);  // b=3,k1=3: W^9 = (cos(9pi/8), -sin(9pi/8))
  // stage 2: for each k1, DFT4 over b -> X[k1 + 4 k2]
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

// padded shared-memory addressing
template <typename C> constexpr int pad_shift() { return sizeof(C) == 8 ? 4 : 3; }
template <typename C> LS_HD int padded(int i) { return i + (i >> pad_shift<C>()); }
template <typename C> LS_HD size_t smem_bytes(int n, int nb) {
  return (size_t)(n + (n >> pad_shift<C>()) + 1) * nb * sizeof(C);
}

template <typename C, bool SEQ_FAST>
LS_D int sm_addr(int seq, int idx, int nb, int ld) {
  if constexpr (SEQ_FAST) return padded<C>(idx) * nb + seq;
  else return seq * ld + padded<C>(idx);
}

struct Geo {
  int lgn;    // log2 length
  int nb;     // sequences per CTA
  int lgnb;   // log2 nb
  int tws;    // log2(table length / n)
};

// Stage radices: ceil(lgn/lgp) stages, bits spread as evenly as possible.
LS_HD int num_stages(int lgn, int lgp) { return (lgn + lgp - 1) / lgp; }
LS_D int stage_bits(int lgn, int lgp, int s) {
  int nst = num_stages(lgn, lgp);
  int base = lgn / nst, extra = lgn - base * nst;
  return base + (s < extra ? 1 : 0);
}

template <int RAD, bool FIRST, bool LAST, bool SEQ_FAST, bool INV, typename C, class F>
LS_D void stage(C (&v)[P_of<C>()], const Geo& g, int lgNs, C* sm, const C* __restrict__ tw, F& f) {
  constexpr int LGR = RAD == 2 ? 1 : RAD == 4 ? 2 : RAD == 8 ? 3 : 4;
  constexpr int P = P_of<C>();
  const int n = 1 << g.lgn;
  const int nr = n >> LGR;  // butterflies per sequence
  const int nt = blockDim.x;
  const int ld = n + (n >> pad_shift<C>()) + 1;
  const int Ns = 1 << lgNs;
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * nt;
    int seq, j;
    if constexpr (SEQ_FAST) { seq = b & (g.nb - 1); j = b >> g.lgnb; }
    else { j = b & (nr - 1); seq = b >> (g.lgn - LGR); }
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      const int idx = j + r * nr;
      C x;
      if constexpr (FIRST) {
        x = f.load(seq, idx);
        if constexpr (INV) x = cconj(x);
      } else {
        x = sm[sm_addr<C, SEQ_FAST>(seq, idx, g.nb, ld)];
      }
      v[i * RAD + r] = x;
    }
    if (!FIRST) {
      const int k = j & (Ns - 1);
      const int sh = g.lgn - lgNs - LGR + g.tws;
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[i * RAD + r] = cmul(v[i * RAD + r], __ldg(&tw[(r * k) << sh]));
    }
    dft<RAD>(&v[i * RAD]);
  }
  if (!FIRST) __syncthreads();  // all smem reads of this stage done
#pragma unroll
  for (int i = 0; i < P / RAD; ++i) {
    const int b = threadIdx.x + i * nt;
    int seq, j;
    if constexpr (SEQ_FAST) { seq = b & (g.nb - 1); j = b >> g.lgnb; }
    else { j = b & (nr - 1); seq = b >> (g.lgn - LGR); }
    const int base = ((j >> lgNs) << (lgNs + LGR)) + (j & (Ns - 1));
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      const int idx = base + r * Ns;
      C x = v[i * RAD + r];
      if constexpr (LAST) {
        if constexpr (INV) x = cconj(x);
        f.store(seq, idx, x);
      } else {
        sm[sm_addr<C, SEQ_FAST>(seq, idx, g.nb, ld)] = x;
      }
    }
  }
  if (!LAST) __syncthreads();
}

template <bool FIRST, bool LAST, bool SEQ_FAST, bool INV, typename C, class F>
LS_D void stage_rt(int bits, C (&v)[P_of<C>()], const Geo& g, int lgNs, C* sm, const C* tw, F& f) {
  switch (bits) {
    case 1: stage<2, FIRST, LAST, SEQ_FAST, INV>(v, g, lgNs, sm, tw, f); break;
    case 2: stage<4, FIRST, LAST, SEQ_FAST, INV>(v, g, lgNs, sm, tw, f); break;
    case 3: stage<8, FIRST, LAST, SEQ_FAST, INV>(v, g, lgNs, sm, tw, f); break;
    default:
      if constexpr (P_of<C>() >= 16) stage<16, FIRST, LAST, SEQ_FAST, INV>(v, g, lgNs, sm, tw, f);
      break;
  }
}

// Full transform of the CTA's nb sequences.  blockDim.x must equal nb*n/P
// (the launcher guarantees it).  The first stage peels the twiddle (Ns=1).
template <bool SEQ_FAST, bool INV, typename C, class F>
LS_D void run(const Geo& g, C* sm, const C* __restrict__ tw, F& f) {
  constexpr int LGP = LGP_of<C>();
  C v[P_of<C>()];
  const int nst = num_stages(g.lgn, LGP);
  if (nst == 1) {
    stage_rt<true, true, SEQ_FAST, INV>(stage_bits(g.lgn, LGP, 0), v, g, 0, sm, tw, f);
    return;
  }
  int lgNs = 0;
  int b0 = stage_bits(g.lgn, LGP, 0);
  stage_rt<true, false, SEQ_FAST, INV>(b0, v, g, 0, sm, tw, f);
  lgNs += b0;
  for (int s = 1; s < nst - 1; ++s) {
    int bs = stage_bits(g.lgn, LGP, s);
    stage_rt<false, false, SEQ_FAST, INV>(bs, v, g, lgNs, sm, tw, f);
    lgNs += bs;
  }
  stage_rt<false, true, SEQ_FAST, INV>(stage_bits(g.lgn, LGP, nst - 1), v, g, lgNs, sm, tw, f);
}

}  // namespace fft
