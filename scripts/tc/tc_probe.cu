// Probe of the tcgen05 building blocks (tc_common.cuh): D[128 x N] = A[128 x K] B[N x K]^T
// in kind::tf32 with small-integer operands (exact in tf32), K-major no-swizzle
// layouts, K = 64 (8 MMAs accumulating), N = 64, and a negated-B variant.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

constexpr int M = 128, N = 64, K = 64;

__global__ void k_probe(const float* A, const float* B, float* D, int neg) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sA = reinterpret_cast<float*>(sm);                  // 128 x 64 = 32 KB
  float* sB = reinterpret_cast<float*>(sm + M * K * 4);      // 64 x 64 = 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int i = t; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(sA) + tc::kmaj_off(r, k, K)) = A[i];
  }
  for (int i = t; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(reinterpret_cast<char*>(sB) + tc::kmaj_off(r, k, K)) = B[i];
  }
  if (t < 32) tc::tmem_alloc<64>(&tbase);
  if (t == 0) tc::mbar_init(&bar, 1);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc::tc_before();
  __syncthreads();
  tc::tc_after();
  const uint32_t d = tbase;
  if (t == 0) {
    const uint32_t idesc = tc::idesc_tf32(M, N, false, neg != 0);
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t da = tc::smem_desc(tc::smem_u32(sA) + kk * 256, 128, (K / 4) * 128);
      const uint64_t db = tc::smem_desc(tc::smem_u32(sB) + kk * 256, 128, (K / 4) * 128);
      tc::mma_tf32(d, da, db, idesc, kk > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_after();
  const int warp = t >> 5, lane = t & 31;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(d + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) D[row * N + c0 + i] = v[i];
  }
  tc::tc_before();
  __syncthreads();
  if (t < 32) tc::tmem_free<64>(d);
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 13 - 6);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (M * K + N * K) * 4;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad_total = 0;
  for (int neg = 0; neg < 2; ++neg) {
    cudaMemset(dD, 0, D.size() * 4);
    k_probe<<<1, 128, smem>>>(dA, dB, dD, neg);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
        if (neg) s = -s;
        if (D[i * N + j] != (float)s) {
          if (bad < 5) printf("neg=%d D[%d][%d] = %g, want %g\n", neg, i, j, D[i * N + j], s);
          ++bad;
        }
      }
    printf("probe neg=%d: %d mismatches of %d\n", neg, bad, M * N);
    bad_total += bad;
  }
  return bad_total != 0;
}
