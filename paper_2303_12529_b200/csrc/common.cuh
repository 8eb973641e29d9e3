// Shared device helpers: complex arithmetic on float2/double2, precision
// traits, deterministic block reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math_constants.h>

#define LS_HD __host__ __device__ __forceinline__
#define LS_D __device__ __forceinline__

template <typename R> struct CT;
template <> struct CT<float> { using C = float2; };
template <> struct CT<double> { using C = double2; };

LS_HD float2 cmk(float a, float b) { return make_float2(a, b); }
LS_HD double2 cmk(double a, double b) { return make_double2(a, b); }
LS_HD float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
LS_HD double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
LS_HD float2 operator-(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
LS_HD double2 operator-(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
LS_HD float2 operator*(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
LS_HD double2 operator*(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

template <typename C> LS_HD C cmul(C a, C b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename C> LS_HD C cmulc(C a, C b) {
  return cmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename C> LS_HD C cconj(C a) { return cmk(a.x, -a.y); }
// multiply by -i (forward-sign quarter turn)
template <typename C> LS_HD C mul_mi(C a) { return cmk(a.y, -a.x); }

// ---------------------------------------------------------------------------
// flat pixel index -> (row, column) without a 64-bit divide: a shift and mask
// for power-of-two widths (every plan grid), a 32-bit divide otherwise.
struct RowSplit {
  uint32_t w, mask;
  int sh;  // log2(w), or -1 when w is not a power of two
};
LS_HD RowSplit row_split(int W) {
  RowSplit r{(uint32_t)W, (uint32_t)W - 1u, -1};
  if (W > 0 && (W & (W - 1)) == 0) {
    int s = 0;
    while ((1 << s) < W) ++s;
    r.sh = s;
  }
  return r;
}
LS_D uint32_t col_of(const RowSplit& r, size_t i) {
  return r.sh >= 0 ? (uint32_t)i & r.mask : (uint32_t)(i % r.w);
}
LS_D uint32_t row_of(const RowSplit& r, size_t i) {
  return r.sh >= 0 ? (uint32_t)(i >> r.sh) : (uint32_t)(i / r.w);
}

// ---------------------------------------------------------------------------
// deterministic reductions: warp shuffle -> smem -> one value per block; the
// per-block partials are combined later by a single block in fixed order.

// NaN-propagating max / clamp: numpy's np.max, np.maximum and np.clip return
// NaN when an operand is NaN, where fmax / fmin drop it (litho.py:126,
// optimizer.py:148,262-268 on non-finite fields).
LS_HD double nmax(double a, double b) { return (a > b || a != a) ? a : b; }
LS_HD double nclip(double x, double lo, double hi) { return x != x ? x : fmin(fmax(x, lo), hi); }

template <typename T> LS_D T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T> LS_D T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block sum of NV values per thread; result valid in thread 0.  `red` must
// hold NV * 32 entries.  Fixed combination order -> bit-reproducible.
template <int NV> LS_D void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i * 32 + warp] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < nw ? red[i * 32 + lane] : 0.0;
      v[i] = warp_sum(t);
    }
  }
}
template <int NV> LS_D void block_max(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_max(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i * 32 + warp] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < nw ? red[i * 32 + lane] : 0.0;
      v[i] = warp_max(t);
    }
  }
}
