// Exact truncated signed distance field (K8), replacing tsdf_from_mask
// (levelset.py:86-101), whose reference arithmetic is
// scipy.ndimage.distance_transform_edt: the Euclidean distance from each
// pixel to the nearest opposite-phase pixel centre, sqrt of an integer.
//
// Separable exact EDT.  Column pass: vertical distance g to the nearest
// feature pixel in the same column, computed by (column, row-segment) threads;
// the nearest feature rows of the other segments are folded in as the row
// pass loads g (k_edt_cols_near).  Row pass: per pixel, the minimum of
// (x - q)^2 + g(q)^2 by an outward scan bounded by the best value so far and
// by the truncation, skipping 8- and 64-column chunks whose minimum g cannot win
// (k_edt_rows_scan).  Squared distances are exact
// integers, so phi = -/+ (sqrt(d2) - 0.5) is bit-identical to the reference.
#include <algorithm>
#include <climits>
#include <cmath>

#include "common.cuh"
#include "internal_ls.h"

namespace lsb {

namespace {

constexpr int kInf = 1 << 29;
constexpr int kSegs = 64;  // row segments per column in the column pass
// row pass pruning geometry and block size (measured at 2048^2: 8/4/64 with
// 512 threads beat 256 threads and chunk/near/super 32/32/-, 16/16/-, 16/4/64,
// 8/8/-, 8/8/64, 8/8/128, 8/4/128, 16/4/128, 16/8/256, 32/4/256, 4/4/64)
#ifndef LSB_TSDF_CHUNK
#define LSB_TSDF_CHUNK 8  // columns per chunk minimum (divides 32)
#endif
#ifndef LSB_TSDF_NEAR
#define LSB_TSDF_NEAR 4  // offsets scanned column by column before chunk pruning
#endif
#ifndef LSB_TSDF_SUPER
#define LSB_TSDF_SUPER 64  // columns per super-chunk minimum (multiple of the chunk)
#endif
#ifndef LSB_TSDF_THREADS
#define LSB_TSDF_THREADS 512  // row-pass block size
#endif
static_assert(32 % LSB_TSDF_CHUNK == 0 && LSB_TSDF_SUPER % LSB_TSDF_CHUNK == 0, "TSDF chunk geometry");

// phi of a pixel from its exact squared distance (levelset.py:86-101): lit
// pixels -(d - 0.5), dark pixels d - 0.5, clipped to [d_lower, d_upper]
template <typename D>
__device__ __forceinline__ double tsdf_value(D best, D clip, bool lit, double d_upper, double d_lower) {
  if (best >= clip) return lit ? d_lower : d_upper;  // truncated whatever the exact distance
  const double d = sqrt((double)best);
  const double val = lit ? -(d - 0.5) : d - 0.5;
  return fmin(fmax(val, d_lower), d_upper);
}

// g layout: g[f][y][x], f = 0: distance to the nearest lit pixel (mask != 0),
// f = 1: distance to the nearest dark pixel.  seg[f][s][x] = {first, last}
// feature row inside segment s (or -1).
__global__ void k_edt_cols_local(int H, int W, const uint8_t* __restrict__ mask, int* g, int2* seg, const int* skip) {
  if (skip && *skip) return;  // reinitialisation gate (lsopc loop)
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (x >= W) return;
  const int len = (H + kSegs - 1) / kSegs, y0 = s * len, y1 = min(H, y0 + len);
  int* g1 = g;                  // f = 0: nearest lit
  int* g0 = g + (size_t)H * W;  // f = 1: nearest dark
  int r1 = kInf, r0 = kInf, f1 = -1, l1 = -1, f0 = -1, l0 = -1;
  for (int y = y0; y < y1; ++y) {
    const bool lit = mask[(size_t)y * W + x] != 0;
    if (lit) { r1 = 0; l1 = y; if (f1 < 0) f1 = y; r0 = r0 >= kInf ? kInf : r0 + 1; }
    else { r0 = 0; l0 = y; if (f0 < 0) f0 = y; r1 = r1 >= kInf ? kInf : r1 + 1; }
    g1[(size_t)y * W + x] = r1;
    g0[(size_t)y * W + x] = r0;
  }
  r1 = kInf;
  r0 = kInf;
  for (int y = y1 - 1; y >= y0; --y) {
    const size_t p = (size_t)y * W + x;
    const bool lit = mask[p] != 0;
    r1 = lit ? 0 : (r1 >= kInf ? kInf : r1 + 1);
    r0 = lit ? (r0 >= kInf ? kInf : r0 + 1) : 0;
    if (r1 < g1[p]) g1[p] = r1;
    if (r0 < g0[p]) g0[p] = r0;
  }
  seg[((size_t)0 * kSegs + s) * W + x] = make_int2(f1, l1);
  seg[((size_t)1 * kSegs + s) * W + x] = make_int2(f0, l0);
}

// fold in the nearest feature rows of the other segments of the column
__global__ void k_edt_cols_fix(int H, int W, const int2* __restrict__ seg, int* g, const int* skip) {
  if (skip && *skip) return;  // reinitialisation gate (lsopc loop)
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (x >= W) return;
  const int len = (H + kSegs - 1) / kSegs, y0 = s * len, y1 = min(H, y0 + len);
  for (int f = 0; f < 2; ++f) {
    int above = -1, below = -1;  // last feature row above y0, first below y1
    for (int t = s - 1; t >= 0 && above < 0; --t) above = seg[((size_t)f * kSegs + t) * W + x].y;
    for (int t = s + 1; t < kSegs && below < 0; ++t) below = seg[((size_t)f * kSegs + t) * W + x].x;
    if (above < 0 && below < 0) continue;
    int* gf = g + (size_t)f * H * W;
    for (int y = y0; y < y1; ++y) {
      const size_t p = (size_t)y * W + x;
      int d = gf[p];
      if (above >= 0) d = min(d, y - above);
      if (below >= 0) d = min(d, below - y);
      gf[p] = d;
    }
  }
}

// nearest feature rows outside each segment, nb[f][s][x] = {last feature row
// above the segment, first below it} (-1: none); the staged row pass folds
// them into g as it loads a row, in place of k_edt_cols_fix
__global__ void k_edt_cols_near(int W, const int2* __restrict__ seg, int2* nb, const int* skip) {
  if (skip && *skip) return;  // reinitialisation gate (lsopc loop)
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.y, f = blockIdx.z;
  if (x >= W) return;
  int above = -1, below = -1;
  for (int t = s - 1; t >= 0 && above < 0; --t) above = seg[((size_t)f * kSegs + t) * W + x].y;
  for (int t = s + 1; t < kSegs && below < 0; ++t) below = seg[((size_t)f * kSegs + t) * W + x].x;
  nb[((size_t)f * kSegs + s) * W + x] = make_int2(above, below);
}

// Row pass.  d2(x) = min over q of (x - q)^2 + g(q)^2.  Each pixel scans
// outward from q = x: a candidate at offset t costs at least t^2, so the scan
// stops as soon as t^2 reaches the best d2 found so far (then d2 is exact), or
// reaches `clip`, a squared distance beyond which the truncated value is the
// clip bound whatever the exact distance is.  One block per row keeps all SMs
// busy (the Felzenszwalb-Huttenlocher envelope is sequential along the row).
// All comparisons are on exact integers.
//
// k_edt_rows_scan: rows too wide to stage in shared memory; reads the fixed-up
// g (k_edt_cols_fix) from global memory, column by column.
template <typename D>  // D: unsigned when every squared distance fits (sides <= 32768), else long long
__global__ void __launch_bounds__(256) k_edt_rows_scan(int H, int W, const uint8_t* __restrict__ mask,
                                                      const int* __restrict__ g, D clip_dark, D clip_lit,
                                                      double d_upper, double d_lower, double* phi, const int* skip) {
  if (skip && *skip) return;  // reinitialisation gate (lsopc loop)
  const int y = blockIdx.x;
  const int* g1 = g + (size_t)y * W;                   // f = 0: distance to the nearest lit pixel
  const int* g0 = g + (size_t)H * W + (size_t)y * W;   // f = 1: distance to the nearest dark pixel
  constexpr D kBig = sizeof(D) == 4 ? (D)UINT_MAX : (D)LLONG_MAX;
  auto sq = [](int v) -> D { return v < kInf ? (D)v * (D)v : kBig; };  // columns without a feature: none
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const size_t p = (size_t)y * W + x;
    const bool lit = mask[p] != 0;
    // lit pixels take the distance to the nearest dark pixel, dark pixels to the nearest lit one
    const int* G = lit ? g0 : g1;
    const D clip = lit ? clip_lit : clip_dark;
    D best = sq(G[x]);
    D lim = best < clip ? best : clip;
    const int reach = max(x, W - 1 - x);
    D t2 = 1;
    for (int t = 1; t <= reach && t2 < lim; ++t, t2 += 2 * t - 1) {
      const int l = G[max(x - t, 0)], r = G[min(x + t, W - 1)];  // clamped reads, masked below
      const D cl = x - t >= 0 ? sq(l) : kBig, cr = x + t < W ? sq(r) : kBig;
      const D c = cl < cr ? cl : cr;
      if (c < kBig && t2 + c < best) best = t2 + c;
      lim = best < clip ? best : clip;
    }
    phi[p] = tsdf_value(best, clip, lit, d_upper, d_lower);
  }
}

// k_edt_rows_pruned: the row staged in shared memory, g squared on load (with
// the nearest feature rows of the other column segments folded in, in place of
// k_edt_cols_fix), plus the minimum of every 8-column chunk and 64-column
// super-chunk.  After the first few offsets each side is scanned chunk by
// chunk: a (super-)chunk whose bound t0^2 + min(g^2) cannot beat the current
// limit is skipped whole, any other chunk is evaluated as one unrolled block.
// Far pixels (the dark background, up to the 900-pixel truncation) then read a
// few minima instead of every column (2048^2 clip: 1.60 -> 0.40 ms per TSDF).
// Skipped candidates cannot lower d2 below the limit, and a whole-chunk block
// only adds candidates that cannot change the output (cost >= best, or >= clip
// where the value is truncated anyway), so the result is the same integer.
template <typename D>
__global__ void __launch_bounds__(LSB_TSDF_THREADS) k_edt_rows_pruned(int H, int W, const uint8_t* __restrict__ mask,
                                                                      const int* __restrict__ g,
                                                                      const int2* __restrict__ nb, D clip_dark,
                                                                      D clip_lit, double d_upper, double d_lower,
                                                                      double* phi, const int* skip) {
  if (skip && *skip) return;  // reinitialisation gate (lsopc loop)
  constexpr int kChunk = LSB_TSDF_CHUNK, kNear = LSB_TSDF_NEAR;  // kChunk divides 32
  constexpr int kSuper = LSB_TSDF_SUPER, kPer = kSuper / kChunk;  // super-chunk = kPer chunks
  // no feature in the column; sums with any offset^2 stay below overflow
  constexpr D kNone = sizeof(D) == 4 ? (D)0x80000000u : (D)(1LL << 62);
  extern __shared__ __align__(16) unsigned char tsdf_sm[];
  const int y = blockIdx.x;
  const int nch = (W + kChunk - 1) / kChunk, nsup = (W + kSuper - 1) / kSuper;
  D* s2 = reinterpret_cast<D*>(tsdf_sm);  // [2][W] squared g: f = 0 nearest lit, f = 1 nearest dark
  D* cm = s2 + 2 * W;                     // [2][nch] chunk minima
  D* cs = cm + 2 * nch;                   // [2][nsup] super-chunk minima
  {
    const int* g1 = g + (size_t)y * W;
    const int* g0 = g + (size_t)H * W + (size_t)y * W;
    const int sgi = y / ((H + kSegs - 1) / kSegs);  // this row's column segment
    const int2* n1 = nb + (size_t)sgi * W;
    const int2* n0 = nb + ((size_t)kSegs + sgi) * W;
    auto fold = [y](int d, int2 n) -> D {
      if (n.x >= 0) d = min(d, y - n.x);
      if (n.y >= 0) d = min(d, n.y - y);
      return d < kInf ? (D)d * (D)d : kNone;
    };
    for (int i = threadIdx.x; i < W; i += blockDim.x) {
      s2[i] = fold(g1[i], n1[i]);
      s2[W + i] = fold(g0[i], n0[i]);
    }
  }
  __syncthreads();
  constexpr int cpw = 32 / kChunk;  // chunks per warp step
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int it = threadIdx.x >> 5; it * cpw < 2 * nch; it += nw) {
    const int c = it * cpw + lane / kChunk, f = c >= nch, i = (c - f * nch) * kChunk + lane % kChunk;
    D v = c < 2 * nch && i < W ? s2[f * W + i] : kNone;
#pragma unroll
    for (int o = kChunk / 2; o > 0; o >>= 1) {
      const D u = __shfl_xor_sync(0xffffffffu, v, o);
      v = u < v ? u : v;
    }
    if (lane % kChunk == 0 && c < 2 * nch) cm[c] = v;
  }
  __syncthreads();
  for (int c2 = threadIdx.x; c2 < 2 * nsup; c2 += blockDim.x) {
    const int f = c2 >= nsup, j = (c2 - f * nsup) * kPer;
    D v = kNone;
    for (int k = 0; k < kPer && j + k < nch; ++k) v = min(v, cm[f * nch + j + k]);
    cs[c2] = v;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const size_t p = (size_t)y * W + x;
    const bool lit = mask[p] != 0;
    // lit pixels take the distance to the nearest dark pixel, dark pixels to the nearest lit one
    const D* G = lit ? s2 + W : s2;
    const D* M = lit ? cm + nch : cm;
    const D* MS = lit ? cs + nsup : cs;
    const D clip = lit ? clip_lit : clip_dark;
    D best = G[x];
    D lim = min(best, clip);
    D t2 = 1;
    int t = 1;
    for (; t <= kNear && t2 < lim; ++t, t2 += 2 * t - 1) {
      if (x - t >= 0) best = min(best, t2 + G[x - t]);
      if (x + t < W) best = min(best, t2 + G[x + t]);
      lim = min(best, clip);
    }
    if (t2 < lim) {
      // right side from offset t; chunks start at q % kChunk == 0
      for (int q = x + t; q < W;) {
        const D o = (D)(q - x), dd = o * o;
        if (dd >= lim) break;
        if ((q & (kSuper - 1)) == 0 && MS[q / kSuper] >= lim - dd) { q += kSuper; continue; }
        if ((q & (kChunk - 1)) == 0) {
          if (M[q / kChunk] >= lim - dd) { q += kChunk; continue; }
          if (q + kChunk <= W) {
            D b = best, oo = dd, step = 2 * o + 1;
#pragma unroll
            for (int k = 0; k < kChunk; ++k) { b = min(b, oo + G[q + k]); oo += step; step += 2; }
            best = b;
            lim = min(best, clip);
            q += kChunk;
            continue;
          }
        }
        best = min(best, dd + G[q]);
        lim = min(best, clip);
        ++q;
      }
      // left side; chunks end at q % kChunk == kChunk - 1 (always whole)
      for (int q = x - t; q >= 0;) {
        const D o = (D)(x - q), dd = o * o;
        if (dd >= lim) break;
        if ((q & (kSuper - 1)) == kSuper - 1 && MS[q / kSuper] >= lim - dd) { q -= kSuper; continue; }
        if ((q & (kChunk - 1)) == kChunk - 1) {
          if (M[q / kChunk] >= lim - dd) { q -= kChunk; continue; }
          D b = best, oo = dd, step = 2 * o + 1;
#pragma unroll
          for (int k = 0; k < kChunk; ++k) { b = min(b, oo + G[q - k]); oo += step; step += 2; }
          best = b;
          lim = min(best, clip);
          q -= kChunk;
          continue;
        }
        best = min(best, dd + G[q]);
        lim = min(best, clip);
        --q;
      }
    }
    phi[p] = tsdf_value(best >= kNone ? clip : best, clip, lit, d_upper, d_lower);
  }
}

// shared bytes of the staged row pass: squared g rows, chunk and super-chunk minima
size_t tsdf_row_smem(int W, size_t elem) {
  const size_t nch = (W + LSB_TSDF_CHUNK - 1) / LSB_TSDF_CHUNK, nsup = (W + LSB_TSDF_SUPER - 1) / LSB_TSDF_SUPER;
  return (2 * (size_t)W + 2 * nch + 2 * nsup) * elem;
}

// smallest squared integer distance from which the truncated value is the
// clip bound with margin: d >= bound + 1 (the value is d - 0.5 past the bound
// by at least 0.5, so rounding of sqrt cannot matter)
long long clip_d2(double bound) {
  const double d = std::fabs(bound) + 1.0;
  const double d2 = std::ceil(d * d);
  return d2 >= 4.0e18 ? (long long)4.0e18 : (long long)d2;
}

}  // namespace

size_t tsdf_scratch_i32(int H, int W) {
  return (size_t)2 * H * W + (size_t)2 * kSegs * W * 2 * 2;  // g, segments, nearest rows outside them
}
size_t tsdf_scratch_f64(int H, int W) { return 1; }

void launch_tsdf(int H, int W, const uint8_t* mask, double d_upper, double d_lower, double* phi,
                 int* si, double* sf, cudaStream_t s, const int* skip) {
  (void)sf;
  int* g = si;
  int2* seg = reinterpret_cast<int2*>(si + (size_t)2 * H * W);
  int2* nb = seg + (size_t)2 * kSegs * W;
  const dim3 cg((W + 127) / 128, kSegs);
  k_edt_cols_local<<<cg, 128, 0, s>>>(H, W, mask, g, seg, skip);
  // dark pixels: value d - 0.5 reaches D_u; lit pixels: -(d - 0.5) reaches D_l
  const long long clip_dark = clip_d2(d_upper + 0.5), clip_lit = clip_d2(0.5 - d_lower);
  const bool narrow = H <= 32768 && W <= 32768;  // t^2 + g^2 < 2^31
  auto run = [&](auto zero) {
    using D = decltype(zero);
    const long long big = sizeof(D) == 4 ? (long long)UINT_MAX : LLONG_MAX;
    const D cd = (D)std::min<long long>(clip_dark, big), cl = (D)std::min<long long>(clip_lit, big);
    const size_t sm = tsdf_row_smem(W, sizeof(D));
    if (sm <= 200 * 1024) {
      k_edt_cols_near<<<dim3((W + 127) / 128, kSegs, 2), 128, 0, s>>>(W, seg, nb, skip);
      auto k = k_edt_rows_pruned<D>;
      if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k<<<H, LSB_TSDF_THREADS, sm, s>>>(H, W, mask, g, nb, cd, cl, d_upper, d_lower, phi, skip);
    } else {  // rows too wide to stage: fix g in place, scan it in global memory
      k_edt_cols_fix<<<cg, 128, 0, s>>>(H, W, seg, g, skip);
      k_edt_rows_scan<D><<<H, 256, 0, s>>>(H, W, mask, g, cd, cl, d_upper, d_lower, phi, skip);
    }
  };
  if (narrow) run(0u);
  else run(0LL);
}

}  // namespace lsb
