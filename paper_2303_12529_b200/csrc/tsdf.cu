// Exact truncated signed distance field (K8), replacing tsdf_from_mask
// (levelset.py:86-101), whose reference arithmetic is
// scipy.ndimage.distance_transform_edt: the Euclidean distance from each
// pixel to the nearest opposite-phase pixel centre, sqrt of an integer.
//
// Separable exact EDT.  Column pass: vertical distance g to the nearest
// feature pixel in the same column, computed by (column, row-segment) threads
// and a fix-up across segments.  Row pass: per pixel, the minimum of
// (x - q)^2 + g(q)^2 by an outward scan bounded by the best value so far and
// by the truncation (k_edt_rows_scan).  Squared distances are exact
// integers, so phi = -/+ (sqrt(d2) - 0.5) is bit-identical to the reference.
#include <algorithm>
#include <climits>
#include <cmath>

#include "common.cuh"
#include "internal_ls.h"

namespace lsb {

namespace {

constexpr int kInf = 1 << 29;
constexpr int kSegs = 16;  // row segments per column in the column pass

// g layout: g[f][y][x], f = 0: distance to the nearest lit pixel (mask != 0),
// f = 1: distance to the nearest dark pixel.  seg[f][s][x] = {first, last}
// feature row inside segment s (or -1).
__global__ void k_edt_cols_local(int H, int W, const uint8_t* __restrict__ mask, int* g, int2* seg) {
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
__global__ void k_edt_cols_fix(int H, int W, const int2* __restrict__ seg, int* g) {
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

// Row pass.  d2(x) = min over q of (x - q)^2 + g(q)^2.  Each pixel scans
// outward from q = x: a candidate at offset t costs at least t^2, so the scan
// stops as soon as t^2 reaches the best d2 found so far (then d2 is exact), or
// reaches `clip`, a squared distance beyond which the truncated value is the
// clip bound whatever the exact distance is.  Work per pixel is therefore
// min(distance, clip distance); with the TSDF's truncation (D_u = 900,
// D_l = -100) every pixel of a 2048^2 clip finishes in a few hundred steps,
// and one block per row keeps all SMs busy (the Felzenszwalb-Huttenlocher
// envelope it replaces is sequential along the row: one thread per row).
// The row's g values (both features) are staged in shared memory; all
// comparisons are on exact integers.
template <typename D>  // D: unsigned when every squared distance fits (sides <= 32768), else long long
__global__ void __launch_bounds__(256) k_edt_rows_scan(int H, int W, const uint8_t* __restrict__ mask,
                                                      const int* __restrict__ g, D clip_dark, D clip_lit,
                                                      double d_upper, double d_lower, double* phi, int staged) {
  extern __shared__ int sg[];  // [2][W] when staged
  const int y = blockIdx.x;
  const int* g1 = g + (size_t)y * W;                   // f = 0: distance to the nearest lit pixel
  const int* g0 = g + (size_t)H * W + (size_t)y * W;   // f = 1: distance to the nearest dark pixel
  if (staged) {
    for (int i = threadIdx.x; i < W; i += blockDim.x) {
      sg[i] = g1[i];
      sg[W + i] = g0[i];
    }
    __syncthreads();
    g1 = sg;
    g0 = sg + W;
  }
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
    double val;
    if (best >= clip) {
      val = lit ? d_lower : d_upper;  // truncated whatever the exact distance
    } else {
      const double d = sqrt((double)best);
      val = lit ? -(d - 0.5) : d - 0.5;
      val = fmin(fmax(val, d_lower), d_upper);
    }
    phi[p] = val;
  }
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
  return (size_t)2 * H * W + (size_t)2 * kSegs * W * 2;  // g, segments
}
size_t tsdf_scratch_f64(int H, int W) { return 1; }

void launch_tsdf(int H, int W, const uint8_t* mask, double d_upper, double d_lower, double* phi,
                 int* si, double* sf, cudaStream_t s) {
  (void)sf;
  int* g = si;
  int2* seg = reinterpret_cast<int2*>(si + (size_t)2 * H * W);
  const dim3 cg((W + 127) / 128, kSegs);
  k_edt_cols_local<<<cg, 128, 0, s>>>(H, W, mask, g, seg);
  k_edt_cols_fix<<<cg, 128, 0, s>>>(H, W, seg, g);
  // dark pixels: value d - 0.5 reaches D_u; lit pixels: -(d - 0.5) reaches D_l
  const long long clip_dark = clip_d2(d_upper + 0.5), clip_lit = clip_d2(0.5 - d_lower);
  const size_t sm = (size_t)2 * W * sizeof(int);
  const int staged = sm <= 200 * 1024;
  const bool narrow = H <= 32768 && W <= 32768;  // t^2 + g^2 < 2^31
  auto run = [&](auto zero) {
    using D = decltype(zero);
    auto k = k_edt_rows_scan<D>;
    if (staged && sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const long long big = sizeof(D) == 4 ? (long long)UINT_MAX : LLONG_MAX;
    k<<<H, 256, staged ? sm : 0, s>>>(H, W, mask, g, (D)std::min<long long>(clip_dark, big),
                                     (D)std::min<long long>(clip_lit, big), d_upper, d_lower, phi, staged);
  };
  if (narrow) run(0u);
  else run(0LL);
}

}  // namespace lsb
