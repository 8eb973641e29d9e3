// F1 on the tensor cores (fp32 tier): the column half of the forward model
// as a dense complex contraction over the kernel taps.
//
// Replaces (reference, /root/reference/pkg/src/lsopc): the y-direction half of
//   IFFT2(FFT2(mask) . FFT2(embed(h_k)))         litho.py:114-126, fields.py:61-74
//
// A K x K kernel's spectrum is a K-term sum along y,
//   H_k(u, v) = sum_i e^(-2 pi i u tr_i / H) G_k(i, v),
//   G_k(i, v) = sum_j h_k(i, j) e^(-2 pi i v tc_j / W)      (the taps' row DFT)
// with tr_i = (i - K/2) mod H, tc_j = (j - K/2) mod W, so the column pass
// T_k = IFFT_y(M^ . H_k) / (HW) is a K-tap column convolution of the mask's
// row transform M~ = FFT_x(mask):
//   T_k(y, v) = sum_i G_k(i, v) / W . M~(y - tr_i, v)
// For one column v and a 128-row tile that is a [128 x K] (Toeplitz in M~)
// by [K x N_k] complex GEMM -- tcgen05.mma kind::tf32 with error-compensated
// split-TF32 operands (x = hi + lo; hi.hi + hi.lo + lo.hi, ~1e-6 relative),
// complex products as real GEMMs with the negation in the instruction
// descriptor, accumulators in TMEM.  It reads G (K x N_k per column, 27 MB
// for 48 kernels at 2048^2) instead of the 2-D spectra (1.5 GB), and M~
// instead of M^ (the mask's column FFT is skipped).
//
// Item = (4 columns, one kernel set, 128 rows); per column B = G (hi / lo,
// re / im stacks) and A = the Toeplitz tile (re, im) built from a 168-row
// slab of M~, first its hi then its lo half; see k_f1_tc for the pipeline.
//
// MEASURED, NOT ADOPTED (opt-in with LSOPC_B200_TCF1=1): correct (2048^2,
// 24 + 24 kernels: intensity 2.6e-6 of max against the float64 tier, the
// FFT F1 2.0e-6; ILT gradient 1.4e-5 vs 6.6e-6), but 1.60-2.21 ms per
// launch across four variants against 0.58 ms for the FFT F1.  ncu: tensor
// pipe 10-13% active, the rest is CUDA-core work building the Toeplitz
// operands (35x expansion of M~ into shared memory, split into hi / lo) and
// the tensor core re-reading A from shared memory for every B part (about
// 1 MB of shared-memory traffic per item: ~0.47 ms at 128 B / clock even if
// perfectly overlapped).  The O(log N) column FFT does less work per output.
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "internal.h"
#include "tcgen05.cuh"

namespace lsb {
namespace {

constexpr int kThreads = 256;
constexpr int kM = 128;                // rows per item (MMA M)
constexpr int kKp = 40;                // taps padded to the MMA K step (8)
constexpr int kN = 32;                 // kernels per set, padded
constexpr int kND = 2 * kN;            // accumulator columns per item column: [re | im] (MMA N = 64)
constexpr int kCols = 4;               // columns per item
constexpr int kTaps = 35;              // G rows cached per column (the kernel side, <= kTaps)
constexpr int kSlab = kM + kKp;        // M~ rows an item reads (>= kM + K - 1)
constexpr int kTmemCols = 512;         // 2 buffers x kCols x kND
constexpr int kLgTileT = 3;            // T_k layout tile width (spectral.cuh)
constexpr uint32_t kAPart = kM * kKp * 4;     // one of re / im of one split half
constexpr uint32_t kBStack = kND * kKp * 4;   // one B stack (64 rows)
constexpr size_t kSmA = 2ull * 2 * kAPart;    // 2 buffers x (re, im)
constexpr size_t kSmB = 2ull * 4 * kBStack;   // 2 buffers x (S1 hi, S1 lo, S2 hi, S2 lo)
constexpr size_t kSmSlab = (size_t)kSlab * kCols * 8;
constexpr size_t kSmG = (size_t)kCols * kTaps * kN * 8;  // the column group's G_k(i, v), [c][i][k]
constexpr size_t kSmem = kSmA + kSmB + kSmSlab + kSmG + 64;

struct Args {
  const float2* mt;      // M~ = FFT_x(mask), column-tiled, tile width 4
  int H, W;
  const float2* G[2];    // per set: [W][K][nk] complex64, G_k(i, v) / W
  float2* T[2];          // per set: T_k fields, column-tiled with tile width 8
  int nk[2], nsets, K;
  int mtiles, items;
  const int* stop;
};

__device__ __forceinline__ void st_f4(unsigned char* base, uint32_t off, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(base + off) = make_float4(a, b, c, d);
}

// Software pipeline over "halves" (one split half of one column's A operand)
// with two A buffers, two B buffers (one column's stacks each) and two TMEM
// accumulator buffers (one item, 4 columns x [re | im] x 32 kernels): every
// buffer's reuse waits on the mbarrier its last MMAs committed to, and an
// item's epilogue runs after the next item's MMAs are queued, so the tensor
// core works while the CTA stores.  B stacks: S1 = [B re; B im], S2 =
// [-B im; B re] (64 rows, hi and lo parts separately), so A_re x S1 + A_im x
// S2 accumulates (re, im) of A . B in one 64-column block.  Each CTA takes a
// contiguous range of items, M-tiles fastest, so the column group's G stays
// in shared memory across its 16 M-tiles.
__global__ void __launch_bounds__(kThreads, 1) k_f1_tc(const __grid_constant__ Args a) {
  if (a.stop && *a.stop) return;
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* A = sm;                                   // [buf][re | im] K-major [kM][kKp]
  unsigned char* B = sm + kSmA;                            // [buf][S1h | S1l | S2h | S2l] K-major [kND][kKp]
  float2* slab = reinterpret_cast<float2*>(sm + kSmA + kSmB);          // [c][s]
  float2* gs = reinterpret_cast<float2*>(sm + kSmA + kSmB + kSmSlab);  // [c][i][k]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kSmA + kSmB + kSmSlab + kSmG);  // A[2], B[2], D[2]
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 6);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (warp == 0) tc::tmem_alloc<kTmemCols>(tbase);
  if (t == 0)
    for (int i = 0; i < 6; ++i) tc::mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc::tc_before();
  __syncthreads();
  tc::tc_after();
  const uint32_t tm = *tbase;
  const uint32_t aA = tc::smem_u32(A), aB = tc::smem_u32(B);
  constexpr uint32_t kSBO = (kKp / 4) * 128;  // 8-row group stride of the K-major layout
  const size_t n = (size_t)a.H * a.W;
  const int K = a.K, c0 = K / 2;
  int nA = 0, nC = 0, nI = 0;                 // halves, columns, items issued so far
  int pset = 0, py0 = 0, pv0 = 0;             // the item awaiting its epilogue
  int gkey = -1;                              // (set, group) whose G is in gs

  auto wait_use = [&](int b, int uses) {     // the (uses-1)-th completion of barrier b
    if (uses >= 1) tc::mbar_wait(&bar[b], (uint32_t)((uses - 1) & 1));
  };
  auto epilogue = [&](int idx, int set, int y0, int v0) {
    const int tb = idx & 1;
    wait_use(4 + tb, (idx >> 1) + 1);
    tc::tc_after();
    const int q = warp & 3, h = warp >> 2, nk = a.nk[set];
    const int y = y0 + 32 * q + lane;
    const uint32_t d0 = tm + ((uint32_t)(32 * q) << 16) + (uint32_t)(tb * kCols * kND);
    const size_t rowoff = (((size_t)(v0 >> kLgTileT) * a.H + y) << kLgTileT) + (v0 & ((1 << kLgTileT) - 1));
    for (int kg = 0; kg < 2; ++kg) {
      const int kb = 16 * h + 8 * kg;
      if (kb >= nk) break;  // warp-uniform
      float re[kCols][8], im[kCols][8];
#pragma unroll
      for (int c = 0; c < kCols; ++c) {
        tc::tmem_ld8(d0 + (uint32_t)(c * kND + kb), re[c]);
        tc::tmem_ld8(d0 + (uint32_t)(c * kND + kN + kb), im[c]);
      }
      tc::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (kb + j >= nk) break;
        float4* dst = reinterpret_cast<float4*>(a.T[set] + (size_t)(kb + j) * n + rowoff);
        dst[0] = make_float4(re[0][j], im[0][j], re[1][j], im[1][j]);
        dst[1] = make_float4(re[2][j], im[2][j], re[3][j], im[3][j]);
      }
    }
    tc::tc_before();
  };

  const int per = (a.items + gridDim.x - 1) / gridDim.x;
  const int it0 = blockIdx.x * per, it1 = min(a.items, it0 + per);
  for (int it = it0; it < it1; ++it) {
    const int m = it % a.mtiles, rest = it / a.mtiles, set = rest % a.nsets, grp = rest / a.nsets;
    const int y0 = m * kM, v0 = grp * kCols, nk = a.nk[set];
    __syncthreads();  // every thread is done reading the previous item's slab / G
    {
      // M~ slab: rows y0 + c0 - (K - 1) + s of the item's 4 columns (one M~ tile), per column
      const float2* mt = a.mt + (size_t)(v0 >> 2) * a.H * 4;
      const int ybase = y0 + c0 - (K - 1);
      for (int e = t; e < (kM + K - 1) * kCols; e += kThreads) {
        const int s = e >> 2, c = e & 3;
        slab[c * kSlab + s] = mt[(size_t)((ybase + s) & (a.H - 1)) * 4 + c];
      }
      if (rest != gkey) {  // a new column group: its G (one contiguous block)
        gkey = rest;
        const float2* G = a.G[set] + (size_t)v0 * K * nk;
        for (int e = t; e < kCols * K * nk; e += kThreads) {
          const int c = e / (K * nk), rem = e - c * K * nk, i = rem / nk, k = rem - i * nk;
          gs[(c * kTaps + i) * kN + k] = __ldg(&G[e]);
        }
      }
    }
    __syncthreads();
    const int tb = nI & 1;
    const uint32_t dbase = tm + (uint32_t)(tb * kCols * kND);
    for (int c = 0; c < kCols; ++c) {
      const int bb = nC & 1;
      wait_use(2 + bb, nC >> 1);  // the column two back (same B buffer) is done
      unsigned char* Bb = B + bb * 4 * kBStack;
      for (int e = t; e < kN * (kKp / 4); e += kThreads) {
        const int k = e % kN, i4 = e / kN;
        float rh[4], rl[4], ih[4], il[4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int i = i4 * 4 + qq;
          const float2 g = (k < nk && i < K) ? gs[(c * kTaps + i) * kN + k] : make_float2(0.f, 0.f);
          tc::split_tf32(g.x, rh[qq], rl[qq]);
          tc::split_tf32(g.y, ih[qq], il[qq]);
        }
        const uint32_t o0 = tc::kmaj_off(k, i4 * 4, kKp), o1 = tc::kmaj_off(kN + k, i4 * 4, kKp);
        st_f4(Bb, o0, rh[0], rh[1], rh[2], rh[3]);                          // S1 hi: [re; im]
        st_f4(Bb, o1, ih[0], ih[1], ih[2], ih[3]);
        st_f4(Bb, kBStack + o0, rl[0], rl[1], rl[2], rl[3]);                // S1 lo
        st_f4(Bb, kBStack + o1, il[0], il[1], il[2], il[3]);
        st_f4(Bb, 2 * kBStack + o0, -ih[0], -ih[1], -ih[2], -ih[3]);        // S2 hi: [-im; re]
        st_f4(Bb, 2 * kBStack + o1, rh[0], rh[1], rh[2], rh[3]);
        st_f4(Bb, 3 * kBStack + o0, -il[0], -il[1], -il[2], -il[3]);        // S2 lo
        st_f4(Bb, 3 * kBStack + o1, rl[0], rl[1], rl[2], rl[3]);
      }
      for (int half = 0; half < 2; ++half) {  // 0: A_hi, 1: A_lo
        const int ab = nA & 1;
        wait_use(ab, nA >> 1);  // the half two back (same A buffer) is done
        unsigned char* Ab = A + ab * 2 * kAPart;
        for (int e = t; e < kM * (kKp / 4); e += kThreads) {
          const int r = e % kM, i4 = e / kM;
          float re[4], im[4];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const int i = i4 * 4 + qq;
            float2 x = make_float2(0.f, 0.f);
            if (i < K) x = slab[c * kSlab + r + K - 1 - i];
            float hh, ll;
            tc::split_tf32(x.x, hh, ll);
            re[qq] = half ? ll : hh;
            tc::split_tf32(x.y, hh, ll);
            im[qq] = half ? ll : hh;
          }
          const uint32_t o = tc::kmaj_off(r, i4 * 4, kKp);
          st_f4(Ab, o, re[0], re[1], re[2], re[3]);
          st_f4(Ab, kAPart + o, im[0], im[1], im[2], im[3]);
        }
        tc::fence_async_smem();
        tc::tc_before();
        __syncthreads();
        tc::tc_after();
        if (t == 0) {
          const uint32_t are = aA + ab * 2 * kAPart, aim = are + kAPart;
          const uint32_t s1h = aB + bb * 4 * kBStack, s1l = s1h + kBStack, s2h = s1h + 2 * kBStack,
                         s2l = s1h + 3 * kBStack;
          const uint32_t d = dbase + (uint32_t)(c * kND);
          const uint32_t idesc = tc::idesc_tf32(kM, kND);
          auto mma = [&](uint32_t x, uint32_t y, int kk, uint32_t acc) {
            tc::mma_tf32(d, tc::smem_desc(x + kk * 256, 128, kSBO), tc::smem_desc(y + kk * 256, 128, kSBO), idesc,
                         acc);
          };
#pragma unroll
          for (int kk = 0; kk < kKp / 8; ++kk) {
            if (half == 0) {  // A_hi x (B_hi + B_lo)
              mma(are, s1h, kk, kk > 0);
              mma(are, s1l, kk, 1u);
              mma(aim, s2h, kk, 1u);
              mma(aim, s2l, kk, 1u);
            } else {          // A_lo x B_hi
              mma(are, s1h, kk, 1u);
              mma(aim, s2h, kk, 1u);
            }
          }
          tc::mma_commit(&bar[ab]);
          if (half) tc::mma_commit(&bar[2 + bb]);
        }
        ++nA;
      }
      ++nC;
    }
    if (t == 0) tc::mma_commit(&bar[4 + tb]);
    // the previous item's epilogue, while this one's MMAs run
    if (nI >= 1) epilogue(nI - 1, pset, py0, pv0);
    pset = set;
    py0 = y0;
    pv0 = v0;
    ++nI;
  }
  if (nI >= 1) epilogue(nI - 1, pset, py0, pv0);
  tc::tc_before();
  __syncthreads();
  tc::tc_after();
  if (warp == 0) tc::tmem_free<kTmemCols>(tm);
}

// G_k(i, v) / W for one kernel set, float64 sums of the taps, stored complex64
__global__ void k_tap_rows(int K, int W, int nk, int lgnmax, const double2* __restrict__ h,
                           const double2* __restrict__ tw, float2* G) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y, k = blockIdx.z;
  if (v >= W) return;
  const int step = (1 << lgnmax) / W;
  double2 acc = make_double2(0.0, 0.0);
  for (int j = 0; j < K; ++j) {
    const int tcj = ((j - K / 2) % W + W) % W;
    const double2 w = tw[(int)(((long long)v * tcj) % W) * step];
    acc = acc + cmul(h[((size_t)k * K + i) * K + j], w);
  }
  G[((size_t)v * K + i) * nk + k] = make_float2((float)(acc.x / W), (float)(acc.y / W));
}

// Opt-in (LSOPC_B200_TCF1=1): correct, but slower than the FFT F1 (see the
// header note and DESIGN.md §8)
bool tcf1_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LSOPC_B200_TCF1");
    return e && e[0] == '1';
  }();
  return on;
}

}  // namespace

bool tcf1_plan_ok(int H, int W, int prec, int vsplit) {
  return tcf1_enabled() && prec == F32 && !vsplit && H >= 256 && H % kM == 0 && W >= 8 && W % 8 == 0;
}
bool tcf1_kset_ok(int nk, int K) { return nk <= kN && K <= kTaps && K <= kSlab - kM + 1; }

bool use_tc_f1(const Grid& g, const SpecSet* sets, int nsets) {
  if (!g.tcf1) return false;
  for (int i = 0; i < nsets; ++i)
    if (!sets[i].G) return false;
  return true;
}

void launch_tap_rows(const Grid& g, int nk, int K, const double* coeffs_dev, void* G, cudaStream_t s) {
  k_tap_rows<<<dim3((g.W + 127) / 128, K, nk), 128, 0, s>>>(K, g.W, nk, g.lgnmax,
                                                           reinterpret_cast<const double2*>(coeffs_dev),
                                                           static_cast<const double2*>(g.tw64), static_cast<float2*>(G));
}

void launch_f1_tc(const Grid& g, const void* mtilde, const SpecSet* sets, int nsets, StopFlag stop, cudaStream_t s) {
  Args a{};
  a.mt = static_cast<const float2*>(mtilde);
  a.H = g.H;
  a.W = g.W;
  a.nsets = nsets;
  a.K = sets[0].K;
  for (int i = 0; i < nsets; ++i) {
    if (sets[i].K != a.K) throw std::runtime_error("tensor-core F1: kernel sets of different sides");
    a.G[i] = static_cast<const float2*>(sets[i].G);
    a.T[i] = static_cast<float2*>(sets[i].T);
    a.nk[i] = sets[i].nk;
  }
  a.mtiles = g.H / kM;
  a.items = (g.W / kCols) * nsets * a.mtiles;
  a.stop = stop;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_f1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(a.items, sms));
  k_f1_tc<<<grid, kThreads, kSmem, s>>>(a);
}

}  // namespace lsb
