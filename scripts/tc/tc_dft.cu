// Tensor-core DFT experiment for the F1 column pass:
// the 2048-point inverse transform of one 4-column tile as a four-step
// DFT whose two stages are tcgen05.mma kind::tf32 GEMMs with error-
// compensated split-TF32 operands (x = hi + lo, three products per real
// GEMM: hi*hi + lo*hi + hi*lo), accumulators in TMEM read back with
// tcgen05.ld, the twiddle multiply between the stages on the CUDA cores.
//
//   n = 64 n1 + n2, f = f1 + 32 f2 (N1 = 32, N2 = 64):
//   stage 1  Y[(c, f1)][n2] = sum_f2 X[(c, f1)][f2] F64[n2][f2]   M=128 N=64 K=64
//   twiddle  Y'           = Y * w^(f1 n2),  w = e^(2 pi i / 2048)
//   stage 2  T[(c, n2)][n1] = sum_f1 Y'[(c, n2)][f1] F32[n1][f1]  2 x (M=128 N=32 K=32)
//   output   t_c[64 n1 + n2] = T[(c, n2)][n1]
//
// Complex products are four real GEMMs (negation through the instruction
// descriptor).  Operands are staged in shared memory in the canonical
// K-major no-swizzle layout; the hi and lo halves of the data are staged one
// after the other (64 KB), the DFT matrices' hi and lo halves stay resident.
//
// COMPUTE-ONLY, like profiles/r01_compute_only_passes.txt for the CUDA-core
// engine: every item transforms the same resident input tile and nothing
// streams from / to HBM (the first items are written out for the accuracy
// check); the F1 workload is 512 tiles x 48 kernels = 24576 items.
//
//   ./tc_dft [items] [split: 3 | 1]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kSmIn = 2048 * 4 * 8;         // input tile [row][4] complex64
constexpr int kSmF64 = 4 * 64 * 64 * 4;     // F64 re/im x hi/lo
constexpr int kSmF32 = 4 * 32 * 32 * 4;     // F32 re/im x hi/lo
constexpr int kSmSt = 2 * 128 * 64 * 4;     // staging: re, im arrays (stage 1: 128 x 64; stage 2: 256 x 32)
constexpr int kSmTw = (32 + 64) * 8;        // twiddle factor tables
constexpr int kSmem = kSmIn + kSmF64 + kSmF32 + kSmSt + kSmTw + 64;

struct Smem {
  float2* in;
  float* f64;  // [4][64x64]: re_hi, re_lo, im_hi, im_lo
  float* f32;  // [4][32x32]
  float* st;   // [2][...]: re, im
  float2* ta;  // e^(2 pi i a / 32), a < 32
  float2* tb;  // e^(2 pi i b / 2048), b < 64
};

__device__ __forceinline__ float* at(float* base, uint32_t off) {
  return reinterpret_cast<float*>(reinterpret_cast<char*>(base) + off);
}

__device__ __forceinline__ float2 twiddle(const Smem& s, int e) {  // w^e, e < 2048
  const float2 a = s.ta[e >> 6], b = s.tb[e & 63];
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int SPLIT>
__device__ void mma_stage1(uint32_t tm, const Smem& s, bool hi_phase) {
  // D1r (cols 0..63) and D1i (cols 64..127) += X * F64^T, one data half
  const uint32_t st = tc::smem_u32(s.st), f = tc::smem_u32(s.f64);
  const uint32_t xr = st, xi = st + 128 * 64 * 4;
  const uint32_t frh = f, frl = f + 16384, fih = f + 32768, fil = f + 49152;
  const uint32_t id = tc::idesc_tf32(128, 64), idn = tc::idesc_tf32(128, 64, false, true);
  auto gemm = [&](uint32_t d, uint32_t a, uint32_t b, uint32_t idsc, bool first) {
    for (int kk = 0; kk < 8; ++kk)
      tc::mma_tf32(d, tc::smem_desc(a + kk * 256, 128, 2048), tc::smem_desc(b + kk * 256, 128, 2048), idsc,
                   !(first && kk == 0));
  };
  if (hi_phase) {
    gemm(tm + 0, xr, frh, id, true);
    gemm(tm + 0, xi, fih, idn, false);
    gemm(tm + 64, xr, fih, id, true);
    gemm(tm + 64, xi, frh, id, false);
    if (SPLIT == 3) {
      gemm(tm + 0, xr, frl, id, false);
      gemm(tm + 0, xi, fil, idn, false);
      gemm(tm + 64, xr, fil, id, false);
      gemm(tm + 64, xi, frl, id, false);
    }
  } else {
    gemm(tm + 0, xr, frh, id, false);
    gemm(tm + 0, xi, fih, idn, false);
    gemm(tm + 64, xr, fih, id, false);
    gemm(tm + 64, xi, frh, id, false);
  }
}

template <int SPLIT>
__device__ void mma_stage2(uint32_t tm, const Smem& s, bool hi_phase) {
  // per half h: D2r (cols 128 + 64 h ..+32), D2i (..+32..64) += Y' * F32^T
  const uint32_t st = tc::smem_u32(s.st), f = tc::smem_u32(s.f32);
  const uint32_t frh = f, frl = f + 4096, fih = f + 8192, fil = f + 12288;
  const uint32_t id = tc::idesc_tf32(128, 32), idn = tc::idesc_tf32(128, 32, false, true);
  for (int h = 0; h < 2; ++h) {
    const uint32_t yr = st + h * 16384, yi = st + 32768 + h * 16384;
    const uint32_t dr = tm + 128 + 64 * h, di = dr + 32;
    auto gemm = [&](uint32_t d, uint32_t a, uint32_t b, uint32_t idsc, bool first) {
      for (int kk = 0; kk < 4; ++kk)
        tc::mma_tf32(d, tc::smem_desc(a + kk * 256, 128, 1024), tc::smem_desc(b + kk * 256, 128, 1024), idsc,
                     !(first && kk == 0));
    };
    if (hi_phase) {
      gemm(dr, yr, frh, id, true);
      gemm(dr, yi, fih, idn, false);
      gemm(di, yr, fih, id, true);
      gemm(di, yi, frh, id, false);
      if (SPLIT == 3) {
        gemm(dr, yr, frl, id, false);
        gemm(dr, yi, fil, idn, false);
        gemm(di, yr, fil, id, false);
        gemm(di, yi, frl, id, false);
      }
    } else {
      gemm(dr, yr, frh, id, false);
      gemm(dr, yi, fih, idn, false);
      gemm(di, yr, fih, id, false);
      gemm(di, yi, frh, id, false);
    }
  }
}

// MMA_ONLY: the same MMA sequence and completion waits per item with no
// CUDA-core staging, twiddles or TMEM read-back -- the tensor-core floor of
// this formulation (results are garbage; timing only).
template <int SPLIT, bool MMA_ONLY = false>
__global__ void __launch_bounds__(kThreads, 1) k_tc_dft(const float2* __restrict__ tile, int items, float2* out,
                                                        int nout, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  Smem s;
  s.in = reinterpret_cast<float2*>(sm);
  s.f64 = reinterpret_cast<float*>(sm + kSmIn);
  s.f32 = reinterpret_cast<float*>(sm + kSmIn + kSmF64);
  s.st = reinterpret_cast<float*>(sm + kSmIn + kSmF64 + kSmF32);
  s.ta = reinterpret_cast<float2*>(sm + kSmIn + kSmF64 + kSmF32 + kSmSt);
  s.tb = s.ta + 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kSmIn + kSmF64 + kSmF32 + kSmSt + kSmTw);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 2);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // resident operands: the input tile, the DFT matrices (split), the twiddle tables
  for (int i = t; i < 2048 * 4; i += kThreads) s.in[i] = tile[i];
  for (int i = t; i < 64 * 64; i += kThreads) {
    const int n = i >> 6, k = i & 63;
    double sv, cv;
    sincospi(2.0 * (double)((n * k) & 63) / 64.0, &sv, &cv);
    float h, l;
    const uint32_t o = tc::kmaj_off(n, k, 64);
    tc::split_tf32((float)cv, h, l);
    *at(s.f64, o) = h;
    *at(s.f64 + 4096, o) = l;
    tc::split_tf32((float)sv, h, l);
    *at(s.f64 + 8192, o) = h;
    *at(s.f64 + 12288, o) = l;
  }
  for (int i = t; i < 32 * 32; i += kThreads) {
    const int n = i >> 5, k = i & 31;
    double sv, cv;
    sincospi(2.0 * (double)((n * k) & 31) / 32.0, &sv, &cv);
    float h, l;
    const uint32_t o = tc::kmaj_off(n, k, 32);
    tc::split_tf32((float)cv, h, l);
    *at(s.f32, o) = h;
    *at(s.f32 + 1024, o) = l;
    tc::split_tf32((float)sv, h, l);
    *at(s.f32 + 2048, o) = h;
    *at(s.f32 + 3072, o) = l;
  }
  if (t < 32) {
    double sv, cv;
    sincospi(2.0 * t / 32.0, &sv, &cv);
    s.ta[t] = make_float2((float)cv, (float)sv);
  }
  if (t < 64) {
    double sv, cv;
    sincospi(2.0 * t / 2048.0, &sv, &cv);
    s.tb[t] = make_float2((float)cv, (float)sv);
  }
  if (warp == 0) tc::tmem_alloc<256>(tbase);
  if (t == 0) tc::mbar_init(bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  tc::fence_async_smem();
  tc::tc_before();
  __syncthreads();
  tc::tc_after();
  const uint32_t tm = *tbase;
  const uint32_t lane_q = (uint32_t)((warp & 3) * 32) << 16;  // this warp's TMEM lane quarter
  uint32_t phase = 0;
  float acc = 0.f;
  auto sync_mma = [&]() {  // operands written -> MMAs issued -> completed
    tc::fence_async_smem();
    tc::tc_before();
    __syncthreads();
    tc::tc_after();
  };
  auto wait_mma = [&]() {
    if (t == 0) tc::mma_commit(bar);
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    tc::tc_after();
  };
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    // ---- stage 1 operands: X[(c, f1)][f2], row b = t & 127, f2 half = t >> 7
    const int b = t & 127, c = b >> 5, f1 = b & 31, f2h = (t >> 7) * 32;
    if (MMA_ONLY) {
      for (int ph = 0; ph < (SPLIT == 3 ? 2 : 1); ++ph) {
        if (t == 0) mma_stage1<SPLIT>(tm, s, ph == 0);
        wait_mma();
      }
      for (int ph = 0; ph < (SPLIT == 3 ? 2 : 1); ++ph) {
        if (t == 0) mma_stage2<SPLIT>(tm, s, ph == 0);
        wait_mma();
      }
      continue;
    }
    for (int ph = 0; ph < (SPLIT == 3 ? 2 : 1); ++ph) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int f2 = f2h + j;
        const float2 x = s.in[(f1 + 32 * f2) * 4 + c];
        float rh, rl, ih, il;
        tc::split_tf32(x.x, rh, rl);
        tc::split_tf32(x.y, ih, il);
        const uint32_t o = tc::kmaj_off(b, f2, 64);
        *at(s.st, o) = ph ? rl : (SPLIT == 3 ? rh : x.x);
        *at(s.st + 128 * 64, o) = ph ? il : (SPLIT == 3 ? ih : x.y);
      }
      sync_mma();
      if (t == 0) mma_stage1<SPLIT>(tm, s, ph == 0);
      wait_mma();
    }
    // ---- twiddle + stage 2 operands: Y'[(c, n2)][f1]; warp w and w + 4 split n2
    {
      const int row = (warp & 3) * 32 + lane;  // = b of stage 1: (c, f1)
      const int cc = row >> 5, ff = row & 31, n2h = (warp >> 2) * 32;
      for (int ph = 0; ph < (SPLIT == 3 ? 2 : 1); ++ph) {
        for (int q = 0; q < 2; ++q) {
          float yr[16], yi[16];
          const int n20 = n2h + 16 * q;
          tc::tmem_ld16(tm + lane_q + n20, yr);
          tc::tmem_ld16(tm + lane_q + 64 + n20, yi);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n2 = n20 + j;
            const float2 w = twiddle(s, ff * n2);
            const float vr = yr[j] * w.x - yi[j] * w.y, vi = yr[j] * w.y + yi[j] * w.x;
            float rh, rl, ih, il;
            tc::split_tf32(vr, rh, rl);
            tc::split_tf32(vi, ih, il);
            const uint32_t o = tc::kmaj_off(cc * 64 + n2, ff, 32);
            *at(s.st, o) = ph ? rl : (SPLIT == 3 ? rh : vr);
            *at(s.st + 256 * 32, o) = ph ? il : (SPLIT == 3 ? ih : vi);
          }
        }
        sync_mma();
        if (t == 0) mma_stage2<SPLIT>(tm, s, ph == 0);
        wait_mma();
      }
    }
    // ---- epilogue: T[(c, n2)][n1] -> t_c[64 n1 + n2]; warps 0-3 take half 0, 4-7 half 1
    {
      const int h = warp >> 2, row = (warp & 3) * 32 + lane;  // TMEM lane = row within the half
      const int r = 128 * h + row, cc = r >> 6, n2 = r & 63;
      float vr[16], vi[16];
      for (int q = 0; q < 2; ++q) {
        tc::tmem_ld16(tm + lane_q + 128 + 64 * h + 16 * q, vr);
        tc::tmem_ld16(tm + lane_q + 128 + 64 * h + 32 + 16 * q, vi);
        if (it < nout) {
          for (int j = 0; j < 16; ++j)
            out[(size_t)it * 8192 + cc * 2048 + 64 * (16 * q + j) + n2] = make_float2(vr[j], vi[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc += vr[j] + vi[j];
        }
      }
    }
    tc::tc_before();
    __syncthreads();
    tc::tc_after();
  }
  if (acc == 12345.f) sink[blockIdx.x] = acc;  // keep the epilogue live
  tc::tc_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free<256>(tm);
}

}  // namespace

int main(int argc, char** argv) {
  const int items = argc > 1 ? atoi(argv[1]) : 24576;
  const int split = argc > 2 ? atoi(argv[2]) : 3;
  const bool mma_only = argc > 3 && atoi(argv[3]) == 1;
  std::vector<float2> tile(2048 * 4);
  srand(7);
  for (auto& v : tile) v = make_float2(2.f * rand() / RAND_MAX - 1.f, 2.f * rand() / RAND_MAX - 1.f);
  float2 *dtile, *dout;
  float* sink;
  const int nout = 2;
  cudaMalloc(&dtile, tile.size() * 8);
  cudaMalloc(&dout, (size_t)nout * 8192 * 8);
  cudaMalloc(&sink, 1024 * 4);
  cudaMemcpy(dtile, tile.data(), tile.size() * 8, cudaMemcpyHostToDevice);
  auto kern = mma_only ? (split == 3 ? k_tc_dft<3, true> : k_tc_dft<1, true>) : (split == 3 ? k_tc_dft<3> : k_tc_dft<1>);
  cudaFuncSetAttribute(k_tc_dft<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaFuncSetAttribute(k_tc_dft<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaFuncSetAttribute(k_tc_dft<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  cudaFuncSetAttribute(k_tc_dft<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  (split == 3 ? k_tc_dft<3> : k_tc_dft<1>)<<<sms, kThreads, kSmem>>>(dtile, nout, dout, nout, sink);  // accuracy
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float2> out((size_t)nout * 8192);
  cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost);
  // reference: double-precision inverse DFT (unnormalised) of each column
  double maxerr = 0, maxref = 0;
  for (int c = 0; c < 4; ++c) {
    std::vector<double> xr(2048), xi(2048);
    for (int f = 0; f < 2048; ++f) { xr[f] = tile[f * 4 + c].x; xi[f] = tile[f * 4 + c].y; }
    for (int n = 0; n < 2048; ++n) {
      double sr = 0, si = 0;
      for (int f = 0; f < 2048; ++f) {
        const double a = 2.0 * M_PI * (double)((long)f * n % 2048) / 2048.0;
        sr += xr[f] * cos(a) - xi[f] * sin(a);
        si += xr[f] * sin(a) + xi[f] * cos(a);
      }
      for (int it = 0; it < nout; ++it) {
        const float2 g = out[(size_t)it * 8192 + c * 2048 + n];
        maxerr = fmax(maxerr, fmax(fabs(g.x - sr), fabs(g.y - si)));
      }
      maxref = fmax(maxref, fmax(fabs(sr), fabs(si)));
    }
  }
  printf("split=%d accuracy: max |err| / max |ref| = %.3e (CUDA-core complex64 FFT engine: ~1e-7)\n", split,
         maxerr / maxref);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<sms, kThreads, kSmem>>>(dtile, items, dout, 0, sink);  // warm-up
  cudaEventRecord(e0);
  kern<<<sms, kThreads, kSmem>>>(dtile, items, dout, 0, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = (double)items * (split == 3 ? 18.87e6 : 6.29e6);
  printf("%s split=%d items=%d (F1 workload = 24576: 512 tiles x 48 kernels): %.1f us, %.1f TFLOP/s tf32 MMA, "
         "%.3f us per tile-kernel per SM\n", mma_only ? "MMA-only" : "full", split, items, ms * 1e3, flop / (ms * 1e-3) / 1e12,
         ms * 1e3 * sms / items);
  return 0;
}
