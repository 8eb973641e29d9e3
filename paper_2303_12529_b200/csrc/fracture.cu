// Greedy rectangle fracturing / shot count (host code), replacing
// fracture + _largest_rect (metrics.py:55-108).
//
// Reference semantics: repeatedly take the largest-area all-ones rectangle,
// ties broken topmost then leftmost (the first candidate met by a row-major
// histogram-stack sweep), and clear it.  The reference re-sweeps the whole
// mask every round (O(shots * H * W)).  Here the sweep result is cached per
// bottom row: clearing a rectangle only changes the column heights of its
// columns from its top row down to where each column run ends, so only those
// rows are re-swept.  Scanning the cached row bests in row order with the
// reference's strict comparison returns exactly the reference's pick.
#include "../../include/lsopc_b200.h"

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace {

struct Cand {
  long long area = 0;
  int x = 0, y = 0, w = 0, h = 0;
};

// metrics.py:80-84 ordering: larger area, then smaller top, then smaller left
inline bool better(const Cand& c, const Cand& best) {
  return c.area > best.area || (c.area == best.area && (c.y < best.y || (c.y == best.y && c.x < best.x)));
}

// histogram-stack sweep of columns [a, b) of one bottom row, all heights > 0
// inside (metrics.py:67-86 restricted to one run: no rectangle crosses a
// zero-height column, and within a row two candidates with equal
// (area, top, left) are the same rectangle, so sweeping runs separately and
// keeping the strict `better` order returns the reference's pick)
void sweep_run(const int* heights, int a, int b, int y, int* stack, Cand& best) {
  int top = -1;
  for (int x = a; x <= b; ++x) {
    const int cur = x < b ? heights[x] : 0;
    while (top >= 0 && heights[stack[top]] > cur) {
      const int hh = heights[stack[top]];
      --top;
      const int left = top >= 0 ? stack[top] + 1 : a;
      Cand c;
      c.area = (long long)hh * (x - left);
      c.x = left;
      c.y = y - hh + 1;
      c.w = x - left;
      c.h = hh;
      if (better(c, best)) best = c;
    }
    stack[++top] = x;
  }
}

// sweep of columns [x0, W) of one bottom row: heights > 0 exactly where the
// row's mask byte is 1; zero runs are skipped 8 bytes at a time
Cand sweep_row(const int* heights, const uint8_t* mrow, int W, int y, std::vector<int>& stack, int x0 = 0) {
  Cand best;
  int x = x0;
  while (x < W) {
    while (x + 8 <= W) {
      uint64_t w8;
      std::memcpy(&w8, mrow + x, 8);
      if (w8) break;
      x += 8;
    }
    while (x < W && !mrow[x]) ++x;
    if (x >= W) break;
    int b = x;
    while (b < W && mrow[b]) ++b;
    sweep_run(heights, x, b, y, stack.data(), best);
    x = b;
  }
  return best;
}

}  // namespace

extern "C" int lsopc_fracture(int H0, int W0, const uint8_t* mask_host, int32_t* rects, size_t cap,
                              size_t* count) {
  if (H0 < 0 || W0 < 0 || !count) return LSOPC_EINVAL;
  // Work on the bounding box of the lit pixels: every rectangle lies inside
  // it and the (area, top, left) order is translation invariant, so the
  // rectangles are the reference's, offset by the box corner.
  int y0 = H0, y1 = -1, x0 = W0, x1 = -1;
  for (int y = 0; y < H0; ++y) {
    const uint8_t* r = mask_host + (size_t)y * W0;
    int x = 0, first = -1, last = -1;
    for (; x + 8 <= W0; x += 8) {
      uint64_t w8;
      std::memcpy(&w8, r + x, 8);
      if (w8) {
        if (first < 0) first = x;
        last = x + 7;
      }
    }
    for (; x < W0; ++x)
      if (r[x]) {
        if (first < 0) first = x;
        last = x;
      }
    if (first < 0) continue;
    while (!r[first]) ++first;
    while (!r[last]) --last;
    if (y0 == H0) y0 = y;
    y1 = y;
    x0 = first < x0 ? first : x0;
    x1 = last > x1 ? last : x1;
  }
  if (y1 < 0) {
    *count = 0;
    return LSOPC_OK;
  }
  const int H = y1 - y0 + 1, W = x1 - x0 + 1;
  const uint8_t* const mask_box = mask_host + (size_t)y0 * W0 + x0;  // row stride W0
  thread_local std::vector<uint8_t> tls_m;
  thread_local std::vector<int> tls_hts;
  tls_m.resize((size_t)H * W);
  tls_hts.resize((size_t)H * W);
  uint8_t* const m = tls_m.data();  // raw pointers: no TLS or vector reloads in the loops
  int* const hts = tls_hts.data();
  // mask bytes and column run heights in one row-major pass (vectorisable:
  // no dependence along a row), each row swept while it is still in cache
  std::vector<int> stack(W + 1);
  std::vector<Cand> rowbest(H);
  for (int y = 0; y < H; ++y) {
    const uint8_t* __restrict__ src = mask_box + (size_t)y * W0;
    uint8_t* __restrict__ mr = m + (size_t)y * W;
    int* __restrict__ hr = hts + (size_t)y * W;
    if (y == 0) {
      for (int x = 0; x < W; ++x) {
        const int v = src[x] != 0;
        mr[x] = (uint8_t)v;
        hr[x] = v;
      }
    } else {
      const int* __restrict__ up = hr - W;
      for (int x = 0; x < W; ++x) {
        const int v = src[x] != 0;
        mr[x] = (uint8_t)v;
        hr[x] = v ? up[x] + 1 : 0;
      }
    }
    rowbest[y] = sweep_row(hr, mr, W, y, stack);
  }
  size_t k = 0;
  while (true) {
    Cand best;
    for (int y = 0; y < H; ++y)
      if (better(rowbest[y], best)) best = rowbest[y];
    if (best.area == 0) break;
    if (rects && k < cap) {
      rects[4 * k] = best.x + x0;
      rects[4 * k + 1] = best.y + y0;
      rects[4 * k + 2] = best.w;
      rects[4 * k + 3] = best.h;
    }
    ++k;
    for (int yy = best.y; yy < best.y + best.h; ++yy) std::memset(&m[(size_t)yy * W + best.x], 0, best.w);
    // refresh the heights of the cleared columns from the rectangle's top row down
    int ymax = best.y + best.h - 1;
    for (int x = best.x; x < best.x + best.w; ++x) {
      for (int y = best.y; y < H; ++y) {
        size_t p = (size_t)y * W + x;
        int nh = m[p] ? (y > 0 ? hts[p - W] : 0) + 1 : 0;
        if (y >= best.y + best.h && nh == hts[p]) break;
        hts[p] = nh;
        if (y > ymax) ymax = y;
      }
    }
    // Re-sweep the affected rows.  Only runs meeting the cleared columns
    // changed (their heights, or their extent where the rectangle split them):
    // all lie inside [a, b), the cleared columns widened to the nearest zero
    // pixel on each side.  A row whose cached best lies outside [a, b) keeps
    // it as the best of its unchanged runs, so only [a, b) is swept and the
    // better of the two kept; otherwise the whole row is swept again.
    for (int y = best.y; y <= ymax; ++y) {
      const uint8_t* mr = &m[(size_t)y * W];
      const int* hr = &hts[(size_t)y * W];
      int a = best.x, b = best.x + best.w;
      while (a > 0 && mr[a - 1]) --a;
      while (b < W && mr[b]) ++b;
      const Cand old = rowbest[y];
      if (old.area > 0 && (old.x >= b || old.x + old.w <= a)) {
        const Cand c = sweep_row(hr, mr, b, y, stack, a);
        rowbest[y] = better(c, old) ? c : old;
      } else {
        rowbest[y] = sweep_row(hr, mr, W, y, stack);
      }
    }
  }
  *count = k;
  return LSOPC_OK;
}
