// Distributed shared memory throughput on B200 (context for the tall-grid
// cluster passes): 4-CTA clusters, 512 threads, each CTA moves `kBytes` per
// round to its peers with st.shared::cluster.v4 (push) or pulls them with
// ld.shared::cluster.v4, with a cluster barrier per round; plus the same
// volume through local shared memory.  Reports per-SM GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kBytes = 64 * 1024;
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned map(const void* p, unsigned r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(sa(p)), "r"(r));
  return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE>  // 0 push remote, 1 pull remote, 2 local copy
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 1) k(int rounds, float* sink) {
  extern __shared__ __align__(16) float4 buf[];  // src [kBytes] + dst [kBytes]
  float4* src = buf;
  float4* dst = buf + kBytes / 16;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < kBytes / 16; i += blockDim.x) src[i] = make_float4(i, rank, 0, 0);
  csync();
  unsigned dbase[4], sbase[4];
  for (int c = 0; c < 4; ++c) {
    dbase[c] = map(dst, c);
    sbase[c] = map(src, c);
  }
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
#pragma unroll 4
    for (int i = threadIdx.x; i < kBytes / 16; i += blockDim.x) {
      const unsigned peer = (rank + 1 + (i & 3)) & 3;  // spread over the other CTAs (and self)
      if (MODE == 0) {
        const float4 v = src[i];
        const unsigned a = dbase[peer] + i * 16;
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
      } else if (MODE == 1) {
        float4 v;
        const unsigned a = sbase[peer] + i * 16;
        asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
                     : "memory");
        dst[i] = v;
      } else {
        dst[i] = src[(i + 1) % (kBytes / 16)];
      }
    }
    csync();
    acc += dst[threadIdx.x].x;
  }
  if (acc == -1.f) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 2000, grid = (sms / 4) * 4;
  const char* names[3] = {"push st.shared::cluster.v4 ", "pull ld.shared::cluster.v4 ", "local shared copy          "};
  for (int mode = 0; mode < 3; ++mode) {
    auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kBytes);
    kern<<<grid, 512, 2 * kBytes>>>(10, sink);
    cudaEventRecord(e0);
    kern<<<grid, 512, 2 * kBytes>>>(rounds, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us_round = ms * 1e3 / rounds;
    printf("%s %6.2f us per 64 KB round per CTA -> %6.1f GB/s per SM (incl. one cluster barrier)  %s\n", names[mode],
           us_round, kBytes / (us_round * 1e3), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
