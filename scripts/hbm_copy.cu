// Achievable HBM streaming on this B200 (context for the roofline denominator):
// (1) grid-stride 16-byte vector copy, (2) TMA bulk copy global -> shared ->
// global through a 3-slot mbarrier ring per CTA (the spectral passes' data path
// without the transform).  Reports GB/s as (read + write bytes) / time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_copy hbm_copy.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void copy_vec(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(512, 1) copy_tma(const char* a, char* b, size_t chunks, unsigned chunk) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 3 * (size_t)chunk);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  size_t it = blockIdx.x;
  unsigned q = 0;
  auto load = [&](size_t c, int slot) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[slot])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(sm + (size_t)slot * chunk)),
                 "l"(a + c * chunk), "r"(chunk), "r"(sa(&bar[slot]))
                 : "memory");
  };
  if (it < chunks) load(it, 0);
  if (it + gridDim.x < chunks) load(it + gridDim.x, 1);
  for (; it < chunks; it += gridDim.x, ++q) {
    const int slot = q % 3;
    const size_t nx = it + 2 * (size_t)gridDim.x;
    if (nx < chunks) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot (q+2)%3 held the store of step q-1
      load(nx, (q + 2) % 3);
    }
    unsigned ok = 0, par = (q / 3) & 1;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(sa(&bar[slot])), "r"(par)
                   : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + it * chunk),
                 "r"(sa(sm + (size_t)slot * chunk)), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)4 << 30;  // 4 GiB each way: far beyond L2
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int blocks : {sms * 4, sms * 8, sms * 16}) {
    copy_vec<<<blocks, 512>>>((const float4*)a, (float4*)b, bytes / 16);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copy_vec<<<blocks, 512>>>((const float4*)a, (float4*)b, bytes / 16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("vec16 copy  %5d blocks: %7.1f GB/s (read+write)\n", blocks, 2.0 * bytes * 5 / (ms * 1e6));
  }
  for (unsigned chunk : {32768u, 65536u}) {
    const size_t smem = 3 * (size_t)chunk + 64;
    cudaFuncSetAttribute(copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    copy_tma<<<sms, 512, smem>>>(a, b, bytes / chunk, chunk);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copy_tma<<<sms, 512, smem>>>(a, b, bytes / chunk, chunk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("TMA bulk ring, %2u KB chunks, 1 CTA/SM: %7.1f GB/s (read+write)  %s\n", chunk / 1024,
           2.0 * bytes * 5 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
