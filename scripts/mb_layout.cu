// Microbenchmark: memory efficiency of the spectral passes' access patterns
// without the FFT.  48 fields of 2048^2 complex64 in the column-tiled layout
// (tile width 4).  Each variant streams every field once (read + write).
//   cols      : column items, contiguous 64 KB tile gather, contiguous store
//   rows_stg  : row items (4 rows), cp.async gather of 512 x 128 B chunks,
//               STG.64 stores in the CT layout (the F2/A1 pattern)
//   rows_v16  : same gather, stores staged through smem, 16 B vector stores
//   rows_rm   : rows of a row-major field: contiguous 64 KB gather + store
//   copy      : flat 16 B vector copy (HBM reference)
#include "../paper_2303_12529_b200/csrc/engine.cuh"
#include <cstdio>
#include <vector>
using C = float2;
constexpr int N = 2048, NK = 48, S = 4, R = 4, NT = 512;
constexpr size_t FS = (size_t)N * N;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const C* __restrict__ src, C* __restrict__ dst, int nitems) {
  extern __shared__ __align__(16) unsigned char smraw[];
  C* buf[2] = {reinterpret_cast<C*>(smraw), reinterpret_cast<C*>(smraw) + 8192};
  const eng::Lay L{N, 2};
  const int per = (MODE == 0 || MODE == 9) ? N / S : N / R;  // items per field
  auto prefetch = [&](int q, C* b) {
    const int f = q / per, it = q % per;
    const C* s = src + (size_t)f * FS;
    if (MODE == 0) eng::gather_rect<8>(b, s, L, 0, 11, it * S, 2);
    else if (MODE == 9) eng::gather_rect<8>(b, s, eng::Lay{N, 3}, 0, 11, it * S, 2);
    else if (MODE == 3 || MODE == 5) eng::gather_rect<8>(b, s, eng::Lay{N, 11}, it * R, 2, 0, 11);
    else if (MODE == 7) eng::gather_rect<8>(b, s, eng::Lay{N, 3}, it * R, 2, 0, 11);
    else if (MODE == 8) eng::gather_rect<8>(b, s, eng::Lay{N, 4}, it * R, 2, 0, 11);
    else eng::gather_rect<8>(b, s, L, it * R, 2, 0, 11);
  };
  int q = blockIdx.x, par = 0;
  if (q >= nitems) return;
  prefetch(q, buf[0]);
  eng::cp_commit();
  while (true) {
    const int nq = q + gridDim.x;
    if (nq < nitems) prefetch(nq, buf[par ^ 1]);
    eng::cp_commit();
    eng::cp_wait<1>();
    __syncthreads();
    const C* b = buf[par];
    const int f = q / per, it = q % per;
    C* d = dst + (size_t)f * FS;
    if (MODE == 0) {
      for (int e = threadIdx.x; e < 8192; e += NT) d[L.at(e >> 2, it * S + (e & 3))] = b[e];
    } else if (MODE == 9) {
      const eng::Lay L8{N, 3};
      for (int e = threadIdx.x; e < 8192; e += NT) d[L8.at(e >> 2, it * S + (e & 3))] = b[e];
    } else if (MODE == 1) {
      // F2-like: thread owns idx = j + r*256 of row seq (last radix-8 stage mapping)
      for (int i = 0; i < 2; ++i) {
        const int bb = threadIdx.x + i * NT, j = bb & 255, seq = bb >> 8;
        for (int r = 0; r < 8; ++r) { const int idx = j + r * 256; d[L.at(it * R + seq, idx)] = b[seq * N + idx]; }
      }
    } else if (MODE == 6) {
      if (b[threadIdx.x].x == 12345.f) d[threadIdx.x] = b[0];
    } else if (MODE == 2 || MODE == 5) {
      // 16 B vector stores: chunk of tile t = 4 rows x 4 cols = 128 B = 8 x 16 B
      for (int p = threadIdx.x; p < 4096; p += NT) {
        const int t = p >> 3, rem = p & 7, r = rem >> 1, c = (rem & 1) * 2;
        const float4 v = *reinterpret_cast<const float4*>(&b[r * N + t * 4 + c]);
        *reinterpret_cast<float4*>(&d[L.at(it * R + r, t * 4 + c)]) = v;
      }
    } else {
      for (int e = threadIdx.x * 2; e < 8192; e += NT * 2)
        *reinterpret_cast<float4*>(&d[(size_t)(it * R) * N + e]) = *reinterpret_cast<const float4*>(&b[e]);
    }
    __syncthreads();
    if (nq >= nitems) break;
    q = nq;
    par ^= 1;
  }
}

__global__ void kcopy(const float4* __restrict__ s, float4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = s[i];
}

int main() {
  C *a, *b;
  cudaMalloc(&a, FS * NK * sizeof(C));
  cudaMalloc(&b, FS * NK * sizeof(C));
  cudaMemset(a, 0, FS * NK * sizeof(C));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t smem = 2 * 8192 * sizeof(C);
  const char* names[] = {"cols", "rows_stg", "rows_v16", "rows_rm", "ctR_rmW", "rmR_ctW", "ctR_only", "ct8R_rmW", "ct16R_rmW", "cols4_ct8"};
  void (*kerns[])(const C*, C*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
  auto run = [&](int mode) {
    auto kern = kerns[mode];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int nitems = NK * (N / 4);
    for (int rep = 0; rep < 2; ++rep) kern<<<148, NT, smem>>>(a, b, nitems);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) kern<<<148, NT, smem>>>(a, b, nitems);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-10s %8.3f ms  %7.1f GB/s (read+write)\n", names[mode], ms, 2.0 * FS * NK * sizeof(C) / ms / 1e6);
  };
  for (int m = 0; m < 10; ++m) run(m);
  const size_t n16 = FS * NK * sizeof(C) / 16;
  for (int rep = 0; rep < 2; ++rep) kcopy<<<148 * 8, 512>>>((const float4*)a, (float4*)b, n16);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; ++rep) kcopy<<<148 * 8, 512>>>((const float4*)a, (float4*)b, n16);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  printf("%-10s %8.3f ms  %7.1f GB/s (read+write)\n", "copy", ms, 2.0 * FS * NK * sizeof(C) / ms / 1e6);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
