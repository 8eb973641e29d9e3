// Arithmetic peaks on this B200 (SURVEY §8(d) asks for FP32 and FP64 beside
// the driver's HBM / bf16 figures): independent FMA chains per thread, all SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peak_flops peak_flops.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void __launch_bounds__(256) fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == (T)-1) out[0] = x0;
}

template <typename T>
void run(const char* name, int sms) {
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int blocks = sms * 8, iters = 4096;
  fma_loop<T><<<blocks, 256>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, 256>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
  printf("%s FMA: %8.2f TFLOP/s\n", name, flops / (ms * 1e9));
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<float>("fp32", sms);
  run<double>("fp64", sms);
  return 0;
}
