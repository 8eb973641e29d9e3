// Exact truncated signed distance field (K8), replacing tsdf_from_mask
// (levelset.py:86-101), whose reference arithmetic is
// scipy.ndimage.distance_transform_edt: the Euclidean distance from each
// pixel to the nearest opposite-phase pixel centre, sqrt of an integer.
//
// Separable exact EDT.  Column pass: vertical distance g to the nearest
// feature pixel in the same column, computed by (column, row-segment) threads
// and a fix-up across segments.  Row pass: Felzenszwalb & Huttenlocher lower
// envelope of the parabolas (x - q)^2 + g(q)^2, one thread per (row,
// feature), with parabola intersections compared as exact integer fractions.  Squared distances are
// exact integers, so phi = -/+ (sqrt(d2) - 0.5) is bit-identical to the
// reference.
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

// Row pass.  One thread per (row, feature) pair; the envelope stack lives in
// global scratch laid out [k][thread] (coalesced across the warp, L1/L2
// resident).  Parabola p_q(x) = (x - q)^2 + g(q)^2; the intersection of p_a
// and p_b (a < b) is at x = num / den with num = key(b) - key(a),
// key(q) = q^2 + g(q)^2, den = 2 (b - a) > 0; intersections are compared as
// exact 64-bit integer fractions (no floating-point division).
__global__ void __launch_bounds__(128) k_edt_rows(int H, int W, const uint8_t* __restrict__ mask,
                                                 const int* __restrict__ g, int* stack, double d_upper,
                                                 double d_lower, double* phi) {
  const int nt = 2 * H;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int f = t / H, y = t % H;
  int* V = stack;                   // column q
  int* G = stack + (size_t)W * nt;  // g(q)
#define SV(i) V[(size_t)(i) * nt + t]
#define SG(i) G[(size_t)(i) * nt + t]
  const int* gr = g + (size_t)f * H * W + (size_t)y * W;
  auto key = [](long long q, long long gq) { return gq * gq + q * q; };
  int k = -1;
  long long kt = 0, kp = 0;  // keys of the stack top and of the entry below it
  long long vt = 0, vp = 0;
  for (int q = 0; q < W; ++q) {
    const int gq = gr[q];
    if (gq >= kInf) continue;
    const long long kq = key(q, gq);
    // pop while s(top, q) <= z(top): (kq - kt)(vt - vp) <= (kt - kp)(q - vt)
    while (k >= 1 && (kq - kt) * (vt - vp) <= (kt - kp) * (q - vt)) {
      --k;
      vt = vp;
      kt = kp;
      if (k >= 1) {
        vp = SV(k - 1);
        kp = key(vp, SG(k - 1));
      }
    }
    ++k;
    SV(k) = q;
    SG(k) = gq;
    vp = vt;
    kp = kt;
    vt = q;
    kt = kq;
  }
  // k >= 0: the feature set is non-empty (uniform masks are rejected upstream)
  int j = 0;
  long long vj = SV(0), kj = key(vj, SG(0));
  long long vn = k >= 1 ? SV(1) : 0, kn = k >= 1 ? key(vn, SG(1)) : 0;
  for (int x = 0; x < W; ++x) {
    // advance while the next parabola's start z(j+1) = (kn - kj) / (2 (vn - vj)) < x
    while (j < k && kn - kj < (long long)x * 2 * (vn - vj)) {
      ++j;
      vj = vn;
      kj = kn;
      if (j < k) {
        vn = SV(j + 1);
        kn = key(vn, SG(j + 1));
      }
    }
    const long long d2 = (x - vj) * (x - vj) + (kj - vj * vj);
    const size_t p = (size_t)y * W + x;
    const bool lit = mask[p] != 0;
    // feature 0 = lit pixels -> distances for dark pixels; feature 1 -> lit pixels
    if ((f == 0) != lit) {
      const double d = sqrt((double)d2);
      const double val = lit ? -(d - 0.5) : d - 0.5;
      phi[p] = fmin(fmax(val, d_lower), d_upper);
    }
  }
#undef SV
#undef SG
}

}  // namespace

size_t tsdf_scratch_i32(int H, int W) {
  return (size_t)2 * H * W + (size_t)2 * kSegs * W * 2 + (size_t)2 * W * 2 * H;  // g, segments, stacks
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
  int* stack = si + (size_t)2 * H * W + (size_t)2 * kSegs * W * 2;
  k_edt_rows<<<(2 * H + 127) / 128, 128, 0, s>>>(H, W, mask, g, stack, d_upper, d_lower, phi);
}

}  // namespace lsb
