// Microbenchmark: achievable HBM bandwidth of column-strip access patterns
// (NB contiguous complex64 per row, 2048 rows) vs contiguous rows, for the
// FFT column-pass design.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int H = 2048, W = 2048;

template <int NB, int THREADS>
__global__ void __launch_bounds__(THREADS) copy_cols(const float2* __restrict__ src, float2* __restrict__ dst) {
  // CTA owns columns [c0, c0+NB) x all rows; thread t handles (row, col) = (t / NB + k*THREADS/NB, t % NB)
  const int c0 = blockIdx.x * NB;
  const int col = threadIdx.x % NB;
  const int r0 = threadIdx.x / NB;
  constexpr int RSTEP = THREADS / NB;
  constexpr int PER = H / RSTEP;
  float2 v[PER > 16 ? 16 : PER];
#pragma unroll 1
  for (int base = 0; base < PER; base += 16) {
#pragma unroll
    for (int k = 0; k < 16 && base + k < PER; ++k) v[k] = src[(size_t)(r0 + (base + k) * RSTEP) * W + c0 + col];
#pragma unroll
    for (int k = 0; k < 16 && base + k < PER; ++k) dst[(size_t)(r0 + (base + k) * RSTEP) * W + c0 + col] = v[k];
  }
}

__global__ void copy_flat(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

template <class F> float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const size_t n = (size_t)H * W;
  float2 *a, *b;
  cudaMalloc(&a, n * 8 * 4);  // 4 buffers' worth to defeat L2 reuse across reps
  cudaMalloc(&b, n * 8 * 4);
  cudaMemset(a, 0, n * 32);
  const double bytes = 2.0 * n * 8;
  int rot = 0;
  auto buf = [&](float2* p) { return p + (size_t)(rot % 4) * n; };
  float ms = timeit([&] { copy_flat<<<148 * 8, 256>>>((const float4*)buf(a), (float4*)buf(b), n / 2); ++rot; });
  printf("flat copy            %8.2f us  %8.1f GB/s\n", ms * 1e3, bytes / ms / 1e6);
#define RUN(NBv, T)                                                                                   \
  ms = timeit([&] { copy_cols<NBv, T><<<W / NBv, T>>>(buf(a), buf(b)); ++rot; });                       \
  printf("cols NB=%2d T=%4d     %8.2f us  %8.1f GB/s\n", NBv, T, ms * 1e3, bytes / ms / 1e6);
  RUN(2, 256) RUN(4, 256) RUN(4, 512) RUN(8, 256) RUN(8, 512) RUN(16, 256) RUN(16, 512) RUN(32, 512)
  cudaDeviceSynchronize();
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
