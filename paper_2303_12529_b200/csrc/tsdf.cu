// Exact truncated signed distance field (K8), replacing tsdf_from_mask
// (levelset.py:86-101), whose reference arithmetic is
// scipy.ndimage.distance_transform_edt: the Euclidean distance from each
// pixel to the nearest opposite-phase pixel centre, sqrt of an integer.
//
// Separable exact EDT (Felzenszwalb & Huttenlocher lower envelope of
// parabolas): a column pass computes the vertical distance to the nearest
// feature in each column, a row pass takes the lower envelope of
// (x - q)^2 + g(q)^2 over q.  Squared distances are exact integers, so
// phi = -/+ (sqrt(d2) - 0.5) is bit-identical to the reference.
#include "common.cuh"
#include "internal_ls.h"

namespace lsb {

namespace {

constexpr int kInf = 1 << 29;

// one thread per column; g[f][y][x] for f = 0 (nearest lit pixel), 1 (nearest dark pixel)
__global__ void k_edt_cols(int H, int W, const uint8_t* __restrict__ mask, int* g) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  int* g1 = g;                       // distance to nearest mask != 0
  int* g0 = g + (size_t)H * W;       // distance to nearest mask == 0
  int r1 = kInf, r0 = kInf;
  for (int y = 0; y < H; ++y) {
    bool lit = mask[(size_t)y * W + x] != 0;
    r1 = lit ? 0 : (r1 >= kInf ? kInf : r1 + 1);
    r0 = lit ? (r0 >= kInf ? kInf : r0 + 1) : 0;
    g1[(size_t)y * W + x] = r1;
    g0[(size_t)y * W + x] = r0;
  }
  r1 = kInf;
  r0 = kInf;
  for (int y = H - 1; y >= 0; --y) {
    size_t p = (size_t)y * W + x;
    bool lit = mask[p] != 0;
    r1 = lit ? 0 : (r1 >= kInf ? kInf : r1 + 1);
    r0 = lit ? (r0 >= kInf ? kInf : r0 + 1) : 0;
    if (r1 < g1[p]) g1[p] = r1;
    if (r0 < g0[p]) g0[p] = r0;
  }
}

// one thread per (row, feature).  Feature 0 (lit) serves dark pixels,
// feature 1 (dark) serves lit pixels.  v/z are per-thread envelope arrays laid
// out [q][thread] for coalescing.
__global__ void k_edt_rows(int H, int W, const uint8_t* __restrict__ mask, const int* __restrict__ g,
                           int* vbuf, double* zbuf, double d_upper, double d_lower, double* phi) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = 2 * H;
  if (t >= nt) return;
  const int f = t / H, y = t % H;
  const int* gr = g + (size_t)f * H * W + (size_t)y * W;
  auto F = [&](int q) -> long long {
    int d = gr[q];
    return d >= kInf ? -1 : (long long)d * d;
  };
  int* v = vbuf;
  double* z = zbuf;
#define V(i) v[(size_t)(i) * nt + t]
#define Z(i) z[(size_t)(i) * nt + t]
  int k = -1;
  for (int q = 0; q < W; ++q) {
    long long fq = F(q);
    if (fq < 0) continue;
    if (k < 0) {
      k = 0;
      V(0) = q;
      Z(0) = -CUDART_INF;
      Z(1) = CUDART_INF;
      continue;
    }
    double s;
    while (true) {  // Z(0) = -inf stops the walk at k = 0
      int vk = V(k);
      long long fv = F(vk);
      s = (double)((fq + (long long)q * q) - (fv + (long long)vk * vk)) / (double)(2 * q - 2 * vk);
      if (s <= Z(k)) { --k; continue; }
      break;
    }
    ++k;
    V(k) = q;
    Z(k) = s;
    Z(k + 1) = CUDART_INF;
  }
  // k >= 0 because the feature set is non-empty (uniform masks are rejected)
  int j = 0;
  for (int x = 0; x < W; ++x) {
    while (Z(j + 1) < (double)x) ++j;
    int vj = V(j);
    long long d2 = (long long)(x - vj) * (x - vj) + F(vj);
    size_t p = (size_t)y * W + x;
    bool lit = mask[p] != 0;
    // feature 0 = lit pixels -> distances for dark pixels; feature 1 -> lit pixels
    if ((f == 0) != lit) {
      double d = sqrt((double)d2);
      double val = lit ? -(d - 0.5) : d - 0.5;
      phi[p] = fmin(fmax(val, d_lower), d_upper);
    }
  }
#undef V
#undef Z
}

}  // namespace

size_t tsdf_scratch_i32(int H, int W) { return (size_t)2 * H * W + (size_t)2 * H * W; }
size_t tsdf_scratch_f64(int H, int W) { return (size_t)2 * H * (W + 1); }

void launch_tsdf(int H, int W, const uint8_t* mask, double d_upper, double d_lower, double* phi,
                 int* si, double* sf, cudaStream_t s) {
  int* g = si;
  int* v = si + (size_t)2 * H * W;
  k_edt_cols<<<(W + 127) / 128, 128, 0, s>>>(H, W, mask, g);
  k_edt_rows<<<(2 * H + 127) / 128, 128, 0, s>>>(H, W, mask, g, v, sf, d_upper, d_lower, phi);
}

}  // namespace lsb
