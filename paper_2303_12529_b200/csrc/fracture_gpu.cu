// Greedy rectangle fracturing / shot count on the device, replacing
// fracture + _largest_rect (metrics.py:55-108).
//
// Reference semantics (metrics.py:90-104): repeatedly take the largest-area
// all-ones rectangle -- ties topmost, then leftmost, then (the row-major
// sweep meets it first) the smallest bottom row -- and clear it.
//
// Device formulation.  Heights h(y, x) = length of the run of lit pixels in
// column x ending at row y (metrics.py:67-68).  For a bottom row y the
// candidates of the reference's histogram-stack sweep (metrics.py:69-86) are
// dominated by the maximal rectangles: for every column x, height h(x),
// spanning (L(x), R(x)) = the nearest columns with a strictly smaller height
// on each side.  Any other popped candidate of the same height is strictly
// narrower, and equal (area, top, left) within one row means the same
// rectangle, so the row's best under the (area desc, top asc, left asc)
// order is the best maximal rectangle.  Clearing a rectangle with bottom row
// rb changes heights only in its columns: 0 inside it and
// h' = min(h, y - rb) below it -- a pointwise rule, no column scan.
//
// One thread-block cluster (16 CTAs, or 8 where 16 do not fit) runs the
// whole greedy loop: CTA c owns the box rows y = c (mod cluster size) with
// their uint16 heights and row bests in shared memory (interleaved rows
// spread a tall rectangle's re-sweeps over every CTA).  Per round every CTA
// applies the clear to its rows, re-sweeps its changed rows (one warp per
// row: run-length segments by ballot, nearest smaller segments by pointer
// jumping), reduces its row bests, pushes its best into every CTA's
// double-buffered slots over distributed shared memory, and after one
// cluster barrier every warp takes the same global best from its own slots.
// Candidates are 64-bit keys whose unsigned order is the reference's.  Boxes
// too large for the cluster's shared memory (or with a side over 4096), and
// runs that exceed the round budget, finish on the host algorithm
// (fracture.cu) from the current mask -- greedy is memoryless, so the result
// is unchanged.
//
// Measured (B200, the configs[1] solve's final mask, 982 x 974 box, 240
// rectangles; ncu kernel times): bounding box 8 us + heights 17 us + the
// cluster loop 972 us = 1.0 ms on the device, against 3.4-3.9 ms for the host
// algorithm (scripts/fracture_probe.py).  Rows with at most 32 run-length
// segments find their nearest smaller segments by warp shuffles; longer
// rows by pointer jumping in shared memory.
#include <cooperative_groups.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lsopc_b200.h"
#include "common.cuh"

namespace cg = cooperative_groups;

void lsb_set_error(const std::string& m);  // plan.cu: lsopc_last_error()

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRounds = 1 << 16;
constexpr size_t kSmemCap = 227 * 1024;

// A candidate rectangle packed into one 64-bit key whose unsigned order is
// the reference's preference (metrics.py:80-84 plus the row-major first-met
// rule): area (bits 36..63), then smaller top, smaller left, smaller bottom
// row (12 bits each, stored as 4095 - value).  Box sides <= 4096.
using Key = unsigned long long;
constexpr int kKeyMaxSide = 4096;

__device__ __forceinline__ Key make_key(int area, int top, int left, int y) {
  return ((Key)area << 36) | ((Key)(4095 - top) << 24) | ((Key)(4095 - left) << 12) | (Key)(4095 - y);
}
__device__ __forceinline__ int key_area(Key k) { return (int)(k >> 36); }
__device__ __forceinline__ int key_top(Key k) { return 4095 - (int)((k >> 24) & 4095); }
__device__ __forceinline__ int key_left(Key k) { return 4095 - (int)((k >> 12) & 4095); }
__device__ __forceinline__ int key_y(Key k) { return 4095 - (int)(k & 4095); }

__device__ __forceinline__ Key warp_max_key(Key k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Key t = __shfl_xor_sync(0xffffffffu, k, o);
    k = t > k ? t : k;
  }
  return k;
}

struct Box {
  int y0, y1, x0, x1;  // lit bounding box (inclusive); y1 < 0: empty
};

struct Status {
  unsigned long long count;  // rectangles found on the device
  int state;                 // 0 done, 1 round budget exhausted (remaining mask written), 2 box does not fit
  int pad;
};

// bounding box of the lit pixels (atomic min / max: order independent)
__global__ void k_bbox(int H, int W, const uint8_t* __restrict__ m, Box* box) {
  int y0 = H, y1 = -1, x0 = W, x1 = -1;
  const size_t n = (size_t)H * W;
  const RowSplit rs = row_split(W);
  auto lit = [&](size_t i) {
    const int y = (int)row_of(rs, i), x = (int)col_of(rs, i);
    y0 = min(y0, y); y1 = max(y1, y); x0 = min(x0, x); x1 = max(x1, x);
  };
  if (W % 16 == 0 && reinterpret_cast<uintptr_t>(m) % 16 == 0) {
    // 16 pixels of one row per load; only a non-zero chunk is inspected
    const uint4* m16 = reinterpret_cast<const uint4*>(m);
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n / 16; q += (size_t)gridDim.x * blockDim.x) {
      const uint4 v = m16[q];
      if (!(v.x | v.y | v.z | v.w)) continue;
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      int first = -1, last = -1;
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if ((w[b >> 2] >> (8 * (b & 3))) & 0xffu) {
          if (first < 0) first = b;
          last = b;
        }
      lit(16 * q + first);
      lit(16 * q + last);
    }
  } else {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      if (m[i]) lit(i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
    y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
    x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
  }
  if ((threadIdx.x & 31) == 0 && y1 >= 0) {
    atomicMin(&box->y0, y0); atomicMax(&box->y1, y1);
    atomicMin(&box->x0, x0); atomicMax(&box->x1, x1);
  }
}

// column run heights over the box (metrics.py:67-68), uint16, box-row-major.
// A block covers 32 columns x 32 row segments: each thread scans its
// segment from a zero carry, then one thread per column chains the carries
// (the height at each segment's last row) and the threads add the carry to
// their segment's leading run.
__global__ void __launch_bounds__(1024) k_heights(int W, const uint8_t* __restrict__ m, const Box* box,
                                                  uint16_t* hts) {
  __shared__ int tail[32][33], lead[32][33], carry[32][33];
  const Box b = *box;
  if (b.y1 < 0) return;
  const int Wb = b.x1 - b.x0 + 1, Hb = b.y1 - b.y0 + 1;
  const int cx = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + cx;
  const int seg = (Hb + 31) / 32;
  const int y0 = sg * seg, y1 = min(Hb, y0 + seg);
  int h = 0, run0 = 0;
  bool leading = true;
  if (x < Wb) {
    const uint8_t* col = m + (size_t)b.y0 * W + b.x0 + x;
    for (int y = y0; y < y1; ++y) {
      const bool lit = col[(size_t)y * W] != 0;
      h = lit ? h + 1 : 0;
      if (leading && lit) ++run0;
      else leading = false;
      hts[(size_t)y * Wb + x] = (uint16_t)h;
    }
  }
  tail[sg][cx] = h;
  lead[sg][cx] = leading && y1 > y0 ? -1 : run0;  // -1: the whole segment is lit
  __syncthreads();
  if (sg == 0) {
    int c = 0;
    for (int k = 0; k < 32; ++k) {
      carry[k][cx] = c;
      c = lead[k][cx] < 0 ? c + tail[k][cx] : tail[k][cx];
    }
  }
  __syncthreads();
  const int c = carry[sg][cx];
  if (x < Wb && c > 0) {
    const int n = lead[sg][cx] < 0 ? y1 - y0 : lead[sg][cx];
    for (int y = y0; y < y0 + n; ++y) hts[(size_t)y * Wb + x] += (uint16_t)c;
  }
}

// Best maximal rectangle with bottom row Y over the heights hr[0, W) (one
// warp).  The row is run-length encoded into segments of equal height
// (ballot + popc over 32-column strips); every segment's maximal rectangle
// spans from the nearest segment of strictly smaller height on its left to
// the nearest on its right.  Those neighbours come from synchronous pointer
// jumping (L(i) <- L(L(i)) while h(L(i)) >= h(i), likewise R), O(log n)
// warp passes even for staircase profiles; updates in place are safe because
// every intermediate L / R keeps its invariant (all segments strictly
// between hold a height >= its own).  Scratch (warp-private shared memory):
// st, sh, Ls, Rs, each W + 1 shorts.
__device__ Key sweep_row(const uint16_t* hr, int W, int Y, short* st, short* sh, short* Ls, short* Rs) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nseg = 0;
  // two columns per lane per 64-column strip: one 32-bit load of a height
  // pair (rows are 16-byte aligned), the left neighbour of the pair from the
  // previous lane (or the previous strip's last column)
  const uint32_t* hr2 = reinterpret_cast<const uint32_t*>(hr);
  int carry = -1;  // height of the column left of the strip (-1: none)
#pragma unroll 2
  for (int base = 0; base < W; base += 64) {
    const int x0 = base + 2 * lane;
    const uint32_t pr = x0 < W ? hr2[x0 >> 1] : 0u;
    const int v0 = (int)(pr & 0xffffu), v1 = x0 + 1 < W ? (int)(pr >> 16) : 0;
    int left = __shfl_up_sync(0xffffffffu, v1, 1);
    if (lane == 0) left = carry;
    carry = __shfl_sync(0xffffffffu, v1, 31);
    const bool b0 = x0 < W && left != v0;      // x0 == 0 has left == -1
    const bool b1 = x0 + 1 < W && v0 != v1;
    const unsigned bal0 = __ballot_sync(0xffffffffu, b0), bal1 = __ballot_sync(0xffffffffu, b1);
    const int before = nseg + __popc(bal0 & lt) + __popc(bal1 & lt);
    if (b0) {
      st[before] = (short)x0;
      sh[before] = (short)v0;
    }
    if (b1) {
      st[before + b0] = (short)(x0 + 1);
      sh[before + b0] = (short)v1;
    }
    nseg += __popc(bal0) + __popc(bal1);
  }
  if (lane == 0) st[nseg] = (short)W;
  __syncwarp();
  if (nseg <= 32) {
    // one segment per lane: the nearest strictly smaller segment on each
    // side by shuffles at growing distance (no shared-memory round trips)
    const int h = lane < nseg ? sh[lane] : 0;
    int l = -1, r = nseg;
    bool lf = lane >= nseg, rf = lane >= nseg;
    for (int k = 1; k < nseg; ++k) {
      const int hl = __shfl_up_sync(0xffffffffu, h, k), hr_ = __shfl_down_sync(0xffffffffu, h, k);
      if (!lf) {
        if (lane < k) lf = true;  // no candidate left of it: l stays -1
        else if (hl < h) { l = lane - k; lf = true; }
      }
      if (!rf) {
        if (lane + k >= nseg) rf = true;  // none right of it: r stays nseg
        else if (hr_ < h) { r = lane + k; rf = true; }
      }
      if (__all_sync(0xffffffffu, lf && rf)) break;
    }
    Key best = 0;
    if (lane < nseg && h > 0) {
      const int left = l >= 0 ? st[l + 1] : 0;
      const int right = r < nseg ? st[r] : W;
      best = make_key(h * (right - left), Y - h + 1, left, Y);
    }
    __syncwarp();
    return warp_max_key(best);
  }
  for (int i = lane; i < nseg; i += 32) {
    Ls[i] = (short)(i - 1);
    Rs[i] = (short)(i + 1);
  }
  __syncwarp();
  for (;;) {
    bool ch = false;
    for (int i = lane; i < nseg; i += 32) {
      const int h = sh[i];
      const int l = Ls[i], r = Rs[i];
      if (l >= 0 && sh[l] >= h) {
        Ls[i] = Ls[l];
        ch = true;
      }
      if (r < nseg && sh[r] >= h) {
        Rs[i] = Rs[r];
        ch = true;
      }
    }
    if (!__any_sync(0xffffffffu, ch)) break;
    __syncwarp();
  }
  __syncwarp();
  Key best = 0;
  for (int i = lane; i < nseg; i += 32) {
    const int h = sh[i];
    if (h == 0) continue;
    const int l = Ls[i], r = Rs[i];
    const int left = l >= 0 ? st[l + 1] : 0;
    const int right = r < nseg ? st[r] : W;
    const Key c = make_key(h * (right - left), Y - h + 1, left, Y);
    best = c > best ? c : best;
  }
  __syncwarp();
  return warp_max_key(best);
}

struct FracArgs {
  const Box* box;
  const uint16_t* hts;     // box heights (k_heights)
  int32_t* rects;          // [cap][4] (x, y, w, h) in grid coordinates
  unsigned long long cap;
  Status* status;
  uint8_t* remain;         // box-sized mask of what is left when the round budget runs out
  int max_rounds;
  long long* prof;         // FRAC_PROF builds: per-phase clock totals of CTA 0
};

#ifdef FRAC_PROF
#define PROF_MARK(i)                                                  \
  do {                                                                \
    if (a.prof && rank == 0 && tid == 0) {                            \
      const long long t_ = clock64();                                 \
      a.prof[i] += t_ - t_prev;                                       \
      t_prev = t_;                                                    \
    }                                                                 \
  } while (0)
#else
#define PROF_MARK(i) do { } while (0)
#endif

__global__ void __launch_bounds__(kThreads, 1) k_fracture_cluster(FracArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const Box b = *a.box;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.y1 < 0) {
    if (rank == 0 && tid == 0) { a.status->count = 0; a.status->state = 0; }
    return;
  }
  const int Hb = b.y1 - b.y0 + 1, Wb = b.x1 - b.x0 + 1;
  const int nloc = (Hb - rank + CL - 1) / CL;     // rows y = rank + CL * r
  const int nmax = (Hb + CL - 1) / CL;
  const int wpad = (Wb + 7) & ~7;
  // layout: slots[2][16] Key | rowbest[nmax] Key | list[nmax] int | nchg[2] int (+2 pad) |
  //         heights[nmax][wpad] u16 | sweep scratch [nsw][4][wpad + 8] short (nsw sweeping warps)
  Key* slots = reinterpret_cast<Key*>(smem);
  Key* rowbest = slots + 2 * 16;
  int* list = reinterpret_cast<int*>(rowbest + nmax);  // changed rows
  int* nchg = list + nmax;  // [2]: changed-row counters by round parity
  uint16_t* hts = reinterpret_cast<uint16_t*>(nchg + 4);
  unsigned char* scratch = reinterpret_cast<unsigned char*>(hts + (size_t)nmax * wpad);
  const size_t used = (size_t)(scratch - smem);
  const size_t wsc = (size_t)(wpad + 8) * 2;  // one scratch array of a sweeping warp, bytes
  const int nsw = used >= kSmemCap ? 0 : (int)min((size_t)kWarps, (kSmemCap - used) / (4 * wsc));
  if (nsw < 4 || Wb > kKeyMaxSide || Hb > kKeyMaxSide) {  // uniform over the cluster: the box does not fit
    if (rank == 0 && tid == 0) { a.status->count = 0; a.status->state = 2; }
    return;
  }
  short* sw_st = reinterpret_cast<short*>(scratch + (size_t)warp * 4 * wsc);
  short* sw_sh = sw_st + wsc / 2;
  short* sw_L = sw_sh + wsc / 2;
  short* sw_R = sw_L + wsc / 2;
  // load own rows, sweep them
  for (int r = 0; r < nloc; ++r) {
    const uint16_t* src = a.hts + (size_t)(rank + CL * r) * Wb;
    for (int x = tid; x < Wb; x += kThreads) hts[(size_t)r * wpad + x] = src[x];
  }
  __syncthreads();
  if (warp < nsw) {
    for (int r = warp; r < nloc; r += nsw) {
      const Key c = sweep_row(hts + (size_t)r * wpad, Wb, rank + CL * r, sw_st, sw_sh, sw_L, sw_R);
      if (lane == 0) rowbest[r] = c;
    }
  }
  __syncthreads();
  unsigned long long count = 0;
  int par = 0, rounds = 0;
  Key G;
  if (tid == 0) nchg[0] = nchg[1] = 0;
#ifdef FRAC_PROF
  long long t_prev = clock64();
#endif
  for (;;) {
    // warp 0: CTA best -> every CTA's slot row (remote stores before the
    // barrier); after it every warp reads its own CTA's slots and takes the
    // same global best
    if (warp == 0) {
      Key c = 0;
      for (int r = lane; r < nloc; r += 32) c = rowbest[r] > c ? rowbest[r] : c;
      c = warp_max_key(c);
      if (lane < CL) *cluster.map_shared_rank(&slots[par * 16 + rank], lane) = c;
      if (lane == 0) nchg[par] = 0;  // this round's changed-row counter (read after the next __syncthreads)
    }
    PROF_MARK(0);
    cluster.sync();
    PROF_MARK(1);
    G = warp_max_key(lane < CL ? slots[par * 16 + lane] : 0);
    PROF_MARK(2);
    if (G == 0 || rounds == a.max_rounds) break;
    ++rounds;
    const int gy = key_y(G), gtop = key_top(G), gleft = key_left(G);
    const int gh = gy - gtop + 1, gw = key_area(G) / gh;
    if (rank == 0 && tid == 0 && count < a.cap) {
      int32_t* o = a.rects + 4 * count;
      o[0] = gleft + b.x0; o[1] = gtop + b.y0; o[2] = gw; o[3] = gh;
    }
    ++count;
    // clear: 0 inside the rectangle, min(h, y - rb) below it (own rows only);
    // a warp per row, changed rows appended to this round's list
    const int rfirst = gtop <= rank ? 0 : (gtop - rank + CL - 1) / CL;
    for (int r = rfirst + warp; r < nloc; r += kWarps) {
      const int Y = rank + CL * r;
      uint16_t* row = hts + (size_t)r * wpad;
      bool ch = false;
      // column pairs (32-bit words; rows are 16-byte aligned), the ends masked
      const int xe = gleft + gw;
      for (int x = (gleft & ~1) + 2 * lane; x < xe; x += 64) {
        uint32_t* p = reinterpret_cast<uint32_t*>(row + x);
        const uint32_t w = *p;
        const int h0 = (int)(w & 0xffffu), h1 = (int)(w >> 16);
        const int n0 = x >= gleft ? (Y <= gy ? 0 : min(h0, Y - gy)) : h0;
        const int n1 = x + 1 < xe ? (Y <= gy ? 0 : min(h1, Y - gy)) : h1;
        if (n0 != h0 || n1 != h1) {
          *p = (uint32_t)n0 | ((uint32_t)n1 << 16);
          ch = true;
        }
      }
      if (__any_sync(0xffffffffu, ch) && lane == 0) list[atomicAdd(&nchg[par], 1)] = r;
    }
    __syncthreads();
    const int n = nchg[par];
    PROF_MARK(4);
#ifdef FRAC_PROF
    if (a.prof && rank == 0 && tid == 0) { a.prof[6] += n; a.prof[7] = max(a.prof[7], (long long)n); }
#endif
#ifdef FRAC_NOSWEEP
    if (false) {
#else
    if (warp < nsw) {
#endif
      for (int i = warp; i < n; i += nsw) {
        const int r = list[i];
        const Key cr = sweep_row(hts + (size_t)r * wpad, Wb, rank + CL * r, sw_st, sw_sh, sw_L, sw_R);
        if (lane == 0) rowbest[r] = cr;
      }
    }
    __syncthreads();
    PROF_MARK(5);
    par ^= 1;
  }
  if (rank == 0 && tid == 0) {
    a.status->count = count;
    a.status->state = G == 0 ? 0 : 1;
  }
  if (G != 0) {  // hand the rest to the host: remaining mask of own rows
    for (int r = 0; r < nloc; ++r)
      for (int x = tid; x < Wb; x += kThreads)
        a.remain[(size_t)(rank + CL * r) * Wb + x] = hts[(size_t)r * wpad + x] != 0;
  }
  cluster.sync();  // no CTA exits while its shared slots may still be read
}

struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
      cap = bytes;
    }
    return p;
  }
};

int fail(const char* what, cudaError_t e) {
  lsb_set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return LSOPC_ECUDA;
}

int cluster_size() {
  static int cl = 0;
  if (cl) return cl;
  cudaFuncSetAttribute(k_fracture_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemCap);
  cudaFuncSetAttribute(k_fracture_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {16, 8, 4}) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemCap;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_fracture_cluster, &cfg) == cudaSuccess && n > 0) {
      cl = c;
      break;
    }
    cudaGetLastError();
  }
  return cl;
}

}  // namespace

extern "C" int lsopc_fracture(int H, int W, const uint8_t* mask_host, int32_t* rects, size_t cap, size_t* count);

// fracture / shot_count of a device mask (metrics.py:55-108): the greedy loop
// on one thread-block cluster (above); rectangles (x, y, w, h) to host memory.
extern "C" int lsopc_fracture_dev(int H, int W, const uint8_t* mask_dev, int32_t* rects_host, size_t cap,
                                  size_t* count, void* stream) {
  if (H < 0 || W < 0 || !count) return LSOPC_EINVAL;
  *count = 0;
  if ((size_t)H * W == 0) return LSOPC_OK;
  if (H > 65535 || W > 65535) return LSOPC_EINVAL;  // uint16 heights
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  thread_local Scratch sh, sr, sx;  // heights + remaining mask, rects, box/status
  const size_t n = (size_t)H * W;
  const size_t dcap = cap < (size_t)kMaxRounds ? cap : (size_t)kMaxRounds;
  char* hx = static_cast<char*>(sx.get(sizeof(Box) + sizeof(Status) + 8 * sizeof(long long)));
  uint16_t* hts = static_cast<uint16_t*>(sh.get(n * 3));  // heights (2 B) + remaining mask (1 B)
  int32_t* dr = static_cast<int32_t*>(sr.get((dcap ? dcap : 1) * 16));
  if (!hx || !hts || !dr) return fail("cudaMalloc", cudaErrorMemoryAllocation);
  Box* box = reinterpret_cast<Box*>(hx);
  Status* st = reinterpret_cast<Status*>(hx + sizeof(Box));
  uint8_t* remain = reinterpret_cast<uint8_t*>(hts + n);
  const Box init{H, -1, W, -1};
  cudaError_t e;
  if ((e = cudaMemcpyAsync(box, &init, sizeof(Box), cudaMemcpyHostToDevice, s))) return fail("memcpy", e);
  k_bbox<<<148 * 4, 256, 0, s>>>(H, W, mask_dev, box);
  k_heights<<<(W + 31) / 32, 1024, 0, s>>>(W, mask_dev, box, hts);
  const int cl = cluster_size();
  Status hs{0, 2, 0};
  Box hb{};
  if (cl) {
    // LSOPC_B200_FRACTURE_ROUNDS (tests): a smaller round budget exercises the host continuation
    const char* rb = std::getenv("LSOPC_B200_FRACTURE_ROUNDS");
    const int rounds = rb ? std::atoi(rb) : kMaxRounds;
    long long* prof = nullptr;
#ifdef FRAC_PROF
    prof = reinterpret_cast<long long*>(hx + sizeof(Box) + sizeof(Status));
    cudaMemsetAsync(prof, 0, 8 * sizeof(long long), s);
#endif
    FracArgs a{box, hts, dr, (unsigned long long)dcap, st, remain, rounds, prof};
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemCap;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if ((e = cudaLaunchKernelEx(&cfg, k_fracture_cluster, a))) return fail("fracture kernel", e);
    if ((e = cudaMemcpyAsync(&hs, st, sizeof(Status), cudaMemcpyDeviceToHost, s))) return fail("memcpy", e);
  }
  if ((e = cudaMemcpyAsync(&hb, box, sizeof(Box), cudaMemcpyDeviceToHost, s))) return fail("memcpy", e);
  if ((e = cudaStreamSynchronize(s))) return fail("fracture", e);
#ifdef FRAC_PROF
  {
    long long hp[8];
    cudaMemcpy(hp, hx + sizeof(Box) + sizeof(Status), sizeof(hp), cudaMemcpyDeviceToHost);
    fprintf(stderr, "FRAC_PROF rounds %llu: reduce %lld sync %lld pick %lld clear %lld compact %lld sweep %lld "
            "(cycles, CTA 0); changed rows %lld, max %lld\n", (unsigned long long)hs.count, hp[0], hp[1], hp[2],
            hp[3], hp[4], hp[5], hp[6], hp[7]);
  }
#endif
  if (hb.y1 < 0) return LSOPC_OK;
  size_t k = (size_t)hs.count;
  if (rects_host && k) {
    const size_t nc = k < cap ? k : cap;
    if ((e = cudaMemcpy(rects_host, dr, nc * 16, cudaMemcpyDeviceToHost))) return fail("memcpy", e);
  }
  if (hs.state != 0) {
    // host continuation: the whole box (it does not fit the cluster) or what
    // the round budget left; greedy from the current mask gives the same rest
    const int Hb = hb.y1 - hb.y0 + 1, Wb = hb.x1 - hb.x0 + 1;
    std::vector<uint8_t> m((size_t)Hb * Wb);
    if (hs.state == 2) {
      if ((e = cudaMemcpy2D(m.data(), Wb, mask_dev + (size_t)hb.y0 * W + hb.x0, W, Wb, Hb,
                            cudaMemcpyDeviceToHost)))
        return fail("memcpy", e);
      k = 0;
    } else if ((e = cudaMemcpy(m.data(), remain, m.size(), cudaMemcpyDeviceToHost))) {
      return fail("memcpy", e);
    }
    size_t more = 0;
    int rc = lsopc_fracture(Hb, Wb, m.data(), nullptr, 0, &more);
    if (rc) return rc;
    if (rects_host && k < cap) {
      std::vector<int32_t> r(4 * (more ? more : 1));
      rc = lsopc_fracture(Hb, Wb, m.data(), r.data(), more, &more);
      if (rc) return rc;
      for (size_t i = 0; i < more && k + i < cap; ++i) {
        int32_t* o = rects_host + 4 * (k + i);
        o[0] = r[4 * i] + hb.x0; o[1] = r[4 * i + 1] + hb.y0; o[2] = r[4 * i + 2]; o[3] = r[4 * i + 3];
      }
    }
    k += more;
  }
  *count = k;
  return LSOPC_OK;
}

