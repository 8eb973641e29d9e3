// C ABI (include/lsopc_b200.h): plans, device spectra, the operator entry
// points, and the on-device DSO loop driver (optimizer.py:204-284).
#include "internal.h"
#include "internal_ls.h"
#include "../../include/lsopc_b200.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

using namespace lsb;

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(LSOPC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ck_launch(const char* what) { ck(cudaGetLastError(), what); }

template <class F> int guarded(F&& f) {
  try {
    f();
    return LSOPC_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LSOPC_EINVAL;
  }
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) cudaFree(p);
    p = nullptr;
    ck(cudaMalloc(&p, bytes), "cudaMalloc");
    cap = bytes;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace

// error text for lsopc_last_error() from the other translation units
void lsb_set_error(const std::string& m) { g_err = m; }

struct lsopc_plan {
  Grid g{};
  // idle sessions kept for reuse by the next lsopc_session_create with the
  // same kernel sets and config: their buffers and captured graphs survive
  // (cudaMalloc/cudaFree and graph instantiation cost more than a 2048^2 solve)
  std::vector<lsopc_session*> pool;
  // T: per-kernel work fields (T_k / U_k) of the spectral passes, grown to the
  // largest (focus + defocus) kernel count used on this plan.
  // A: per-kernel row-major fields A_k (F2 -> A1).
  DevBuf tw, tw64, mhat, scratch, scratch2, T, A, V0, V1, If, Id, wf, wd, partials, scal, hard, tsdf_i, tsdf_f;
  // small grids: kernel-group partials of I and V and their tickets (spectral.cuh choose_lgg)
  DevBuf Ipart, Vpart, tick;
  ~lsopc_plan() {
    for (DevBuf* b : {&tw, &tw64, &mhat, &scratch, &scratch2, &T, &A, &V0, &V1, &If, &Id, &wf, &wd, &partials,
                      &scal, &hard, &tsdf_i, &tsdf_f, &Ipart, &Vpart, &tick})
      b->release();
  }
  // bumped whenever T or A is reallocated: CUDA graphs captured before that
  // hold the old pointers and must be re-captured (lsopc_session::gen)
  unsigned long long gen = 0;
  size_t n() const { return g.n(); }
  void ensure_T(int nk_total) {
    const size_t bytes = (size_t)nk_total * n() * g.csize();
    if (bytes > T.cap || bytes > A.cap) ++gen;
    T.ensure(bytes);
    A.ensure(bytes);
  }
};

void lsb_purge_pool(lsopc_plan* p, const lsopc_kset* ks);

struct lsopc_kset {
  lsopc_plan* plan = nullptr;
  int nk = 0, K = 0;
  DevBuf spec;
  DevBuf G;  // tensor-core F1: the taps' row DFT (f1_tc.cu), when the plan and the set allow it
  std::vector<double> w;
  ~lsopc_kset() {
    spec.release();
    G.release();
  }
};

namespace {

void check_plan(const lsopc_plan* p) {
  if (!p) throw Error(LSOPC_EINVAL, "null plan");
}
void check_kset(const lsopc_plan* p, const lsopc_kset* k) {
  if (!k || k->plan != p) throw Error(LSOPC_EINVAL, "kernel set does not belong to this plan");
}

double reduce_to_host(int op, size_t n, const double* a, const double* b, const uint8_t* a8, const uint8_t* b8,
                      lsopc_plan* plan, cudaStream_t s, int W = 0, Tile t = Tile{0, 0, 0, 0}) {
  thread_local DevBuf tmp;  // plan-less calls: per-thread partials, kept across calls
  double* part;
  double* out;
  if (plan) {
    part = plan->partials.as<double>();
    out = plan->scal.as<double>();
  } else {
    tmp.ensure((ls_blocks() + 8) * sizeof(double));
    part = tmp.as<double>();
    out = part + ls_blocks();
  }
  launch_reduce(op, n, a, b, a8, b8, part, out, s, W, t.ix0, t.ix1, t.iy0, t.iy1);
  ck_launch("reduce");
  double h = 0.0;
  ck(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, s), "memcpy");
  ck(cudaStreamSynchronize(s), "sync");
  return h;
}

// SpecSet views of one or two kernel sets on the plan's work buffers
SpecSet spec_set(lsopc_plan* p, const lsopc_kset* ks, int which, size_t T_off_kernels) {
  SpecSet s{};
  s.nk = ks->nk;
  s.w = ks->w.data();
  s.spec = ks->spec.p;
  s.T = static_cast<char*>(p->T.p) + T_off_kernels * p->n() * p->g.csize();
  s.A = static_cast<char*>(p->A.p) + T_off_kernels * p->n() * p->g.csize();
  s.I = which == 0 ? p->If.p : p->Id.p;
  s.gate = which == 0 ? p->wf.p : p->wd.p;
  s.V = which == 0 ? p->V0.p : p->V1.p;
  s.Ipart = p->Ipart.p;
  s.Vpart = p->Vpart.p;
  s.tick = p->tick.as<unsigned>();
  s.G = ks->G.p;
  s.K = ks->K;
  return s;
}

// the mask's transform and F1 of nsets sets: the tensor-core F1 reads the
// mask pass's row transform (scratch), the FFT F1 its full 2-D transform
void mask_and_f1(lsopc_plan* p, const SpecSet* sets, int nsets, const uint8_t* mu8, const double* mf,
                 const double* phi, StopFlag stop, cudaStream_t s) {
  const bool tc = use_tc_f1(p->g, sets, nsets);
  launch_mask_fft(p->g, mu8, mf, phi, p->mhat.p, p->scratch.p, stop, s, !tc);
  launch_f1(p->g, p->mhat.p, sets, nsets, stop, s, p->scratch.p);
}

// forward of one set (I into If) or of focus + defocus (If, Id) from a mask
// (exactly one of mu8 / mf / phi non-null)
void forward(lsopc_plan* p, const lsopc_kset* f, const lsopc_kset* d, StopFlag stop, cudaStream_t s,
             const uint8_t* mu8, const double* mf, const double* phi, double* a0_c128 = nullptr) {
  p->ensure_T(f->nk + (d ? d->nk : 0));
  SpecSet sets[2] = {spec_set(p, f, 0, 0), d ? spec_set(p, d, 1, f->nk) : SpecSet{}};
  mask_and_f1(p, sets, d ? 2 : 1, mu8, mf, phi, stop, s);
  launch_f2(p->g, sets, d ? 2 : 1, a0_c128, stop, s);
  ck_launch("forward");
}

}  // namespace

// ============================================================================

extern "C" {

const char* lsopc_last_error(void) { return g_err.c_str(); }
int lsopc_abi_version(void) { return 1; }

int lsopc_plan_create(int H, int W, int precision, lsopc_plan** out) {
  return guarded([&] {
    if (!out) throw Error(LSOPC_EINVAL, "null output");
    if (!pow2(H) || !pow2(W) || H < 4 || W < 4 || H > 8192 || W > 8192 || (size_t)H * W < 16)
      throw Error(LSOPC_EINVAL, "grid " + std::to_string(W) + "x" + std::to_string(H) +
                                    " unsupported: sides must be powers of two in [4, 8192]");
    if (precision != LSOPC_FP32 && precision != LSOPC_FP64) throw Error(LSOPC_EINVAL, "bad precision");
    // tall-grid split: 8192-point columns as four 2048-point planes, while a
    // row item still holds the four rows (one per plane) it combines
    const bool tma_off = [] {
      const char* e = std::getenv("LSOPC_B200_NO_TMA");
      return e && e[0] == '1';
    }();
    const char* nv = std::getenv("LSOPC_B200_NO_VSPLIT");
    const int row_item = precision == LSOPC_FP64 ? 4096 : 8192;  // elements per row item
    const bool vsplit = !(nv && nv[0] == '1') && !tma_off && H == 8192 && W >= 256 && W * 4 <= row_item;
    if (precision == LSOPC_FP64 && (W > 4096 || (H > 4096 && !vsplit)))
      throw Error(LSOPC_EINVAL, "the FP64 tier supports sides up to 4096, and 8192 x W grids with 256 <= W <= "
                                "1024; use the FP32 tier for larger grids");
    auto* p = new lsopc_plan();
    try {
      p->g.H = H;
      p->g.W = W;
      p->g.lgH = ilog2(H);
      p->g.lgW = ilog2(W);
      p->g.prec = precision;
      p->g.vsplit = vsplit ? 1 : 0;
      p->g.tcf1 = tcf1_plan_ok(H, W, p->g.prec, p->g.vsplit) ? 1 : 0;
      const int nmax = H > W ? H : W;
      p->g.lgnmax = ilog2(nmax);
      std::vector<double> t64(2 * nmax);
      std::vector<float> t32(2 * nmax);
      for (int j = 0; j < nmax; ++j) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)nmax;
        t64[2 * j] = (double)cosl(a);
        t64[2 * j + 1] = (double)sinl(a);
        t32[2 * j] = (float)cosl(a);
        t32[2 * j + 1] = (float)sinl(a);
      }
      p->tw64.ensure(t64.size() * sizeof(double));
      ck(cudaMemcpy(p->tw64.p, t64.data(), t64.size() * sizeof(double), cudaMemcpyHostToDevice), "memcpy");
      if (precision == LSOPC_FP64) {
        p->g.tw = p->tw64.p;
      } else {
        p->tw.ensure(t32.size() * sizeof(float));
        ck(cudaMemcpy(p->tw.p, t32.data(), t32.size() * sizeof(float), cudaMemcpyHostToDevice), "memcpy");
        p->g.tw = p->tw.p;
      }
      p->g.tw64 = p->tw64.p;
      const size_t n = p->n();
      p->mhat.ensure(n * p->g.csize());
      p->scratch.ensure(n * 16);
      p->scratch2.ensure(n * 16);
      p->V0.ensure(n * p->g.csize());
      p->V1.ensure(n * p->g.csize());
      p->If.ensure(n * p->g.rsize());
      p->Id.ensure(n * p->g.rsize());
      p->wf.ensure(n * p->g.rsize());
      p->wd.ensure(n * p->g.rsize());
      size_t np = (size_t)std::max(std::max(reduce_blocks(), ls_blocks()), H) * 4 + 64;
      p->partials.ensure(np * sizeof(double));
      if (n <= ((size_t)1 << 18)) {  // few items per pass: kernel groups (<= 8) fill the SMs
        p->Ipart.ensure(8 * 2 * n * p->g.rsize());
        p->Vpart.ensure(8 * 2 * n * p->g.csize());
        p->tick.ensure(4 * (size_t)std::max(H, W) * sizeof(unsigned));
        ck(cudaMemset(p->tick.p, 0, 4 * (size_t)std::max(H, W) * sizeof(unsigned)), "memset");
      }
      p->scal.ensure(64 * sizeof(double));
      p->hard.ensure(3 * n);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int lsopc_plan_destroy(lsopc_plan* plan) {
  return guarded([&] {
    cudaDeviceSynchronize();
    if (plan) lsb_purge_pool(plan, nullptr);
    delete plan;
  });
}

int lsopc_kset_create(lsopc_plan* plan, int n_k, int K, const double* coeffs_host, const double* weights_host,
                      void* stream, lsopc_kset** out) {
  return guarded([&] {
    check_plan(plan);
    if (n_k < 1 || K < 1) throw Error(LSOPC_EINVAL, "kernel set must contain at least one kernel");
    if (K > plan->g.H || K > plan->g.W)
      throw Error(LSOPC_EINVAL, "kernel side " + std::to_string(K) + " exceeds grid " + std::to_string(plan->g.W) +
                                    "x" + std::to_string(plan->g.H));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* ks = new lsopc_kset();
    try {
      ks->plan = plan;
      ks->nk = n_k;
      ks->K = K;
      ks->w.assign(weights_host, weights_host + n_k);
      ks->spec.ensure((size_t)n_k * plan->n() * plan->g.csize());
      DevBuf coeffs;
      const size_t cb = (size_t)n_k * K * K * 2 * sizeof(double);
      coeffs.ensure(cb);
      ck(cudaMemcpyAsync(coeffs.p, coeffs_host, cb, cudaMemcpyHostToDevice, s), "memcpy");
      launch_kernel_spectra(plan->g, n_k, K, coeffs.as<double>(), ks->spec.p, plan->scratch.p, plan->scratch2.p, s);
      ck_launch("kernel spectra");
      if (plan->g.tcf1 && tcf1_kset_ok(n_k, K)) {
        ks->G.ensure((size_t)plan->g.W * K * n_k * 8);
        launch_tap_rows(plan->g, n_k, K, coeffs.as<double>(), ks->G.p, s);
        ck_launch("tap rows");
      }
      ck(cudaStreamSynchronize(s), "sync");
      coeffs.release();
    } catch (...) {
      delete ks;
      throw;
    }
    *out = ks;
  });
}

int lsopc_kset_download(const lsopc_kset* ks, double* out, void* stream) {
  return guarded([&] {
    if (!ks) throw Error(LSOPC_EINVAL, "null kernel set");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = ks->plan->n();
    Grid g = ks->plan->g;
    for (int k = 0; k < ks->nk; ++k) {
      launch_spec_to_c128(g, static_cast<const char*>(ks->spec.p) + (size_t)k * n * g.csize(), out + (size_t)k * n * 2, s);
      ck_launch("download");
    }
  });
}

int lsopc_kset_destroy(lsopc_kset* ks) {
  return guarded([&] {
    cudaDeviceSynchronize();
    if (ks && ks->plan) lsb_purge_pool(ks->plan, ks);
    delete ks;
  });
}

int lsopc_aerial_intensity(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev, double dose,
                           double* out_dev, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_kset(plan, ks);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    forward(plan, ks, nullptr, nullptr, s, nullptr, mask_dev, nullptr);
    launch_scale_intensity(plan->g, plan->If.p, dose, out_dev, s);
    ck_launch("scale intensity");
  });
}

int lsopc_print_corners(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus,
                        const double* mask_dev, double i_th, double sigma_z, int binarize, void* nom, void* inner,
                        void* outer, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_kset(plan, focus);
    check_kset(plan, defocus);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    forward(plan, focus, defocus, nullptr, s, nullptr, mask_dev, nullptr);
    ResistParams rp{i_th, sigma_z, 0.0, 0.0};
    if (binarize)
      launch_resist(plan->g, plan->If.p, plan->Id.p, nullptr, nullptr, rp, nullptr, nullptr, nullptr, nullptr,
                    nullptr, static_cast<uint8_t*>(nom), static_cast<uint8_t*>(inner), static_cast<uint8_t*>(outer),
                    nullptr, nullptr, s);
    else
      launch_resist(plan->g, plan->If.p, plan->Id.p, nullptr, nullptr, rp, nullptr, nullptr,
                    static_cast<double*>(nom), static_cast<double*>(inner), static_cast<double*>(outer), nullptr,
                    nullptr, nullptr, nullptr, nullptr, s);
    ck_launch("resist");
  });
}

int lsopc_socs_gradient(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev, const double* z_dev,
                        const double* zt_dev, double sigma_z, double dose, double* out_dev, void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_kset(plan, ks);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = plan->n();
    forward(plan, ks, nullptr, nullptr, s, nullptr, mask_dev, nullptr);
    launch_gate(plan->g, z_dev, zt_dev, 1.0, plan->wf.p, s);
    ck_launch("gate");
    SpecSet set = spec_set(plan, ks, 0, 0);
    launch_adjoint(plan->g, &set, 1, nullptr, s);
    ck_launch("adjoint");
    launch_adjoint_finish(plan->g, plan->V0.p, nullptr, 4.0 * sigma_z * dose / (double)n, out_dev, nullptr,
                          nullptr, nullptr, s);
    ck_launch("adjoint finish");
  });
}

int lsopc_convolve(lsopc_plan* plan, const lsopc_kset* ks, const double* mask_dev, double* out_c128_dev,
                   void* stream) {
  return guarded([&] {
    check_plan(plan);
    check_kset(plan, ks);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    forward(plan, ks, nullptr, nullptr, s, nullptr, mask_dev, nullptr, out_c128_dev);
  });
}

int lsopc_geometry_gradient(int H, int W, const double* phi, double* gx, double* gy, double* gxx, double* gyy,
                            double* gxy, double* mag, void* stream) {
  return guarded([&] {
    if (H < 1 || W < 1) throw Error(LSOPC_EINVAL, "empty field");
    launch_geometry(H, W, phi, gx, gy, gxx, gyy, gxy, mag, static_cast<cudaStream_t>(stream));
    ck_launch("geometry");
  });
}

int lsopc_curvature(int H, int W, const double* phi, const double* m, double weight, double* out, void* stream) {
  return guarded([&] {
    if (H < 1 || W < 1) throw Error(LSOPC_EINVAL, "empty field");
    launch_curvature(H, W, phi, m, weight, out, static_cast<cudaStream_t>(stream));
    ck_launch("curvature");
  });
}

int lsopc_tsdf(int H, int W, const uint8_t* mask, double d_upper, double d_lower, double* phi, void* stream) {
  return guarded([&] {
    if (H < 1 || W < 1) throw Error(LSOPC_EINVAL, "empty mask");
    if (!(d_lower < 0.0 && 0.0 < d_upper))
      throw Error(LSOPC_EINVAL, "truncation bounds must satisfy D_l < 0 < D_u");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n = (size_t)H * W;
    double diff = reduce_to_host(RD_COUNTNEQ8, n, nullptr, nullptr, mask, nullptr, nullptr, s);
    if (diff == 0.0 || diff == (double)n) throw Error(LSOPC_EDEGENERATE, "mask is uniform: no boundary exists");
    // scratch kept per calling thread: a cudaMalloc / cudaFree pair per call
    // (cudaFree synchronises the device) cost more than the transform
    thread_local DevBuf si, sf;
    si.ensure(tsdf_scratch_i32(H, W) * sizeof(int));
    sf.ensure(tsdf_scratch_f64(H, W) * sizeof(double));
    launch_tsdf(H, W, mask, d_upper, d_lower, phi, si.as<int>(), sf.as<double>(), s);
    ck_launch("tsdf");
    ck(cudaStreamSynchronize(s), "sync");
  });
}

int lsopc_elementwise(int op, size_t n, const double* a, const double* b, double p0, double p1, double p2,
                      double* out, uint8_t* out8, void* stream) {
  return guarded([&] {
    if (op < EW_MASK || op > EW_HYPOT) throw Error(LSOPC_EINVAL, "unknown elementwise op");
    if (n == 0) return;
    launch_elementwise(op, n, a, b, p0, p1, p2, out, out8, static_cast<cudaStream_t>(stream));
    ck_launch("elementwise");
  });
}

int lsopc_reduce(int op, size_t n, const double* a, const double* b, const uint8_t* a8, const uint8_t* b8,
                 double* out_host, void* stream) {
  return guarded([&] {
    if (op < RD_SUMSQDIFF || op > RD_COUNTNEQ) throw Error(LSOPC_EINVAL, "unknown reduction");
    if (n == 0) {
      *out_host = 0.0;
      return;
    }
    *out_host = reduce_to_host(op, n, a, b, a8, b8, nullptr, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"

// ============================================================================
// DSO loop session

struct lsopc_session {
  lsopc_plan* plan = nullptr;
  const lsopc_kset* focus = nullptr;
  const lsopc_kset* defocus = nullptr;
  lsopc_config cfg{};
  cudaStream_t s = nullptr;
  DevBuf target, phi, best, v[2], d[2], u, mask, mod, hist, state, part_ls, part_up, dots, gm;
  DevBuf rein;  // opt-in reinitialisation: reduce partials, lit count, gate flag
  int it = 0;  // iterations enqueued
  bool have_mod = false;
  // strip of an oversized tile (lsopc_session_set_tile): interior / stencil columns
  bool tiled = false;
  Tile tile{};
  DevBuf scalars;  // 8 doubles exchanged with the other ranks between phases
  // one DSO iteration captured as a CUDA graph per buffer parity (it & 1)
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  unsigned long long gen = 0;  // plan->gen when the graphs were captured
  int* hflag = nullptr;  // pinned host copies of DevState::stopped (async polling)
  cudaEvent_t ev[2] = {nullptr, nullptr};
  void drop_graphs() {
    for (auto& g : graph) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
  }
  ~lsopc_session() {
    drop_graphs();
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (hflag) cudaFreeHost(hflag);
    for (DevBuf* b : {&target, &phi, &best, &v[0], &v[1], &d[0], &d[1], &u, &mask, &mod, &hist, &state, &part_ls,
                      &part_up, &dots, &gm, &scalars, &rein})
      b->release();
  }
  DevState* st() const { return state.as<DevState>(); }
};

namespace {

constexpr size_t kPoolCap = 4;

bool same_key(const lsopc_session* ss, const lsopc_kset* f, const lsopc_kset* d, const lsopc_config& c,
              bool have_mod) {
  return ss->focus == f && ss->defocus == d && ss->have_mod == have_mod &&
         std::memcmp(&ss->cfg, &c, sizeof(c)) == 0;
}

lsopc_session* take_pooled(lsopc_plan* p, const lsopc_kset* f, const lsopc_kset* d, const lsopc_config& c,
                           bool have_mod) {
  for (size_t i = 0; i < p->pool.size(); ++i) {
    if (same_key(p->pool[i], f, d, c, have_mod)) {
      lsopc_session* ss = p->pool[i];
      p->pool.erase(p->pool.begin() + i);
      return ss;
    }
  }
  return nullptr;
}

void give_to_pool(lsopc_session* ss) {
  lsopc_plan* p = ss->plan;
  p->pool.insert(p->pool.begin(), ss);
  while (p->pool.size() > kPoolCap) {
    delete p->pool.back();
    p->pool.pop_back();
  }
}

// drop pooled sessions that reference a kernel set (before it is freed), or all
void purge_pool(lsopc_plan* p, const lsopc_kset* ks) {
  for (size_t i = 0; i < p->pool.size();) {
    if (!ks || p->pool[i]->focus == ks || p->pool[i]->defocus == ks) {
      delete p->pool[i];
      p->pool.erase(p->pool.begin() + i);
    } else {
      ++i;
    }
  }
}

}  // namespace

void lsb_purge_pool(lsopc_plan* p, const lsopc_kset* ks) { purge_pool(p, ks); }

namespace {

// Pass boundaries inside one iteration, for per-pass CUDA-event timing.
enum { PS_MASK = 0, PS_F1, PS_F2, PS_RESIST, PS_A1, PS_A2, PS_A3, PS_LS, PS_N };

// One iteration on buffers of parity `par`; every iteration-dependent
// decision (restart, record index, stop) reads the device state, so the same
// launch sequence serves every iteration of that parity (graph capture).
void enqueue_iteration(lsopc_session* ss, int par, cudaStream_t s, cudaEvent_t* ev = nullptr) {
  lsopc_plan* p = ss->plan;
  const Grid& g = p->g;
  const size_t n = g.n();
  const int it = par;
  DevState* st = ss->st();
  StopFlag stop = &st->stopped;
  const lsopc_config& c = ss->cfg;
  double* v = ss->v[it & 1].as<double>();
  double* vprev = ss->v[(it + 1) & 1].as<double>();
  double* d = ss->d[it & 1].as<double>();
  double* dprev = ss->d[(it + 1) & 1].as<double>();
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
  };
  SpecSet sets[2] = {spec_set(p, ss->focus, 0, 0), spec_set(p, ss->defocus, 1, ss->focus->nk)};

  // forward: M^ -> T_k -> I_f, I_d -> resist, losses, gates
  mark(0);
  const bool tc = use_tc_f1(g, sets, 2);
  launch_mask_fft(g, ss->mask.as<uint8_t>(), nullptr, nullptr, p->mhat.p, p->scratch.p, stop, s, !tc);
  mark(1);
  launch_f1(g, p->mhat.p, sets, 2, stop, s, p->scratch.p);
  mark(2);
  launch_f2(g, sets, 2, nullptr, stop, s);
  mark(3);
  ResistParams rp{c.i_th, c.sigma_z, c.alpha, c.beta};
  LoopCfg lc{c.alpha, c.beta, c.stop_rel_tol, c.stop_patience};
  // each control step (loss/best/patience, CG beta, CFL step, record) runs in
  // the last block of the kernel producing its partials (control.cuh)
  const LoopTail tail{st, ss->hist.as<double>(), lc, c.eta, c.cg_restart_every};
  launch_resist(g, p->If.p, p->Id.p, ss->target.as<uint8_t>(), nullptr, rp, p->wf.p, p->wd.p, nullptr, nullptr,
                nullptr, nullptr, nullptr, nullptr, p->partials.as<double>(), stop, s, 0, 0, &tail);
  launch_copy_best(n, ss->phi.as<double>(), ss->best.as<double>(), st, s);
  mark(4);
  // adjoint: U_k, then one frequency-domain accumulator per set and one inverse
  launch_a1(g, sets, 2, stop, s);
  mark(5);
  launch_a2(g, sets, 2, stop, s);
  mark(6);
  launch_adjoint_finish(g, p->V0.p, p->V1.p, 4.0 * c.sigma_z / (double)n, v, vprev, ss->dots.as<double>(), stop, s,
                        0, 0, &tail);
  mark(7);
  // level-set step
  launch_ls_velocity(g.H, g.W, ss->phi.as<double>(), v, dprev, ss->have_mod ? ss->mod.as<double>() : nullptr,
                     c.curvature_weight, c.use_curvature, st, d, ss->u.as<double>(),
                     c.update_form ? ss->gm.as<double>() : nullptr, ss->part_ls.as<double>(), full_tile(g.W), s,
                     &tail, c.grad_scheme == 1);
  launch_ls_update(g.H, g.W, ss->phi.as<double>(), ss->u.as<double>(), c.update_form ? ss->gm.as<double>() : nullptr,
                   c.d_lower, c.d_upper, st, ss->mask.as<uint8_t>(),
                   ss->part_up.as<double>(), full_tile(g.W), s, &tail);
  if (c.reinit_every > 0) {  // opt-in: phi <- TSDF(mask) after every reinit_every-th iteration
    double* rp = ss->rein.as<double>();
    int* skip = reinterpret_cast<int*>(rp + ls_blocks() + 1);
    launch_reduce(RD_COUNTNEQ8, n, nullptr, nullptr, ss->mask.as<uint8_t>(), nullptr, rp, rp + ls_blocks(), s);
    launch_reinit_gate(st, rp + ls_blocks(), (double)n, c.reinit_every, skip, s);
    launch_tsdf(g.H, g.W, ss->mask.as<uint8_t>(), c.d_upper, c.d_lower, ss->phi.as<double>(), p->tsdf_i.as<int>(),
                p->tsdf_f.as<double>(), s, skip);
  }
  mark(8);
  ck_launch("dso iteration");
}

// One phase of a strip iteration (lsopc_session_phase).  Each phase ends
// with this rank's partial scalars in ss->scalars; the caller combines them
// across ranks (sum / max) before the next phase consumes them.
void enqueue_phase(lsopc_session* ss, int phase, cudaStream_t s) {
  lsopc_plan* p = ss->plan;
  const Grid& g = p->g;
  const size_t n = g.n();
  DevState* st = ss->st();
  StopFlag stop = &st->stopped;
  const lsopc_config& c = ss->cfg;
  const int par = ss->it & 1;
  double* v = ss->v[par].as<double>();
  double* vprev = ss->v[par ^ 1].as<double>();
  double* d = ss->d[par].as<double>();
  double* dprev = ss->d[par ^ 1].as<double>();
  double* sc = ss->scalars.as<double>();
  const Tile& t = ss->tile;
  SpecSet sets[2] = {spec_set(p, ss->focus, 0, 0), spec_set(p, ss->defocus, 1, ss->focus->nk)};
  switch (phase) {
    case 0: {  // forward from phi (the halo columns were refreshed by the caller) -> sum losses
      mask_and_f1(p, sets, 2, nullptr, nullptr, ss->phi.as<double>(), stop, s);
      launch_f2(g, sets, 2, nullptr, stop, s);
      ResistParams rp{c.i_th, c.sigma_z, c.alpha, c.beta};
      launch_resist(g, p->If.p, p->Id.p, ss->target.as<uint8_t>(), nullptr, rp, p->wf.p, p->wd.p, nullptr,
                    nullptr, nullptr, nullptr, nullptr, nullptr, p->partials.as<double>(), stop, s, t.ix0, t.ix1,
                    nullptr, t.iy0, t.iy1);
      launch_reduce_partials(p->partials.as<double>(), reduce_blocks(), 4, 0, sc, s);
    } break;
    case 1:    // stop rule on the global losses; adjoint -> sum PR dots
    case 6: {  // 6: the stop rule alone (after phase 5)
      LoopCfg lc{c.alpha, c.beta, c.stop_rel_tol, c.stop_patience};
      launch_after_forward(sc, 1, lc, st, ss->hist.as<double>(), s);
      launch_copy_best(n, ss->phi.as<double>(), ss->best.as<double>(), st, s);
      if (phase == 6) break;
    }
      [[fallthrough]];
    case 5: {  // 5: the adjoint alone, straight after phase 0 (it reads only the forward's fields)
      launch_a1(g, sets, 2, stop, s);
      launch_a2(g, sets, 2, stop, s);
      const int nd = launch_adjoint_finish(g, p->V0.p, p->V1.p, 4.0 * c.sigma_z / (double)n, v, vprev,
                                           ss->dots.as<double>(), stop, s, t.ix0, t.ix1, nullptr, t.iy0, t.iy1);
      launch_reduce_partials(ss->dots.as<double>(), nd, 2, 0, sc + 2, s);
    } break;
    case 2: {  // CG on the global dots; level-set velocity -> max |v_total|, max |grad phi|
      launch_after_grad(sc + 2, 1, c.cg_restart_every, st, s);
      launch_ls_velocity(g.H, g.W, ss->phi.as<double>(), v, dprev, ss->have_mod ? ss->mod.as<double>() : nullptr,
                         c.curvature_weight, c.use_curvature, st, d, ss->u.as<double>(),
                         c.update_form ? ss->gm.as<double>() : nullptr, ss->part_ls.as<double>(), t, s, nullptr,
                         c.grad_scheme == 1);
      launch_reduce_partials(ss->part_ls.as<double>(), ls_blocks(), 2, 1, sc + 4, s);
    } break;
    case 3: {  // CFL step on the global max; interior update -> max step
      launch_after_velocity(sc + 4, 1, c.eta, st, ss->hist.as<double>(), s);
      launch_ls_update(g.H, g.W, ss->phi.as<double>(), ss->u.as<double>(),
                       c.update_form ? ss->gm.as<double>() : nullptr, c.d_lower, c.d_upper, st,
                       ss->mask.as<uint8_t>(), ss->part_up.as<double>(), t, s);
      launch_reduce_partials(ss->part_up.as<double>(), ls_blocks(), 1, 1, sc + 6, s);
    } break;
    default:  // record on the global max step
      launch_after_update(sc + 6, 1, st, ss->hist.as<double>(), s);
      break;
  }
  ck_launch("dso phase");
}

// Capture one DSO iteration per buffer parity as a CUDA graph (on a private
// stream: the caller's may be the legacy stream).  The graphs bake in the
// plan's T / A pointers, so they are tied to the plan's buffer generation.
void capture_graphs(lsopc_session* ss) {
  ss->drop_graphs();
  const char* ng = std::getenv("LSOPC_B200_NO_GRAPH");
  if (ng && ng[0] == '1') return;
  cudaStream_t cs;
  ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
  for (int par = 0; par < 2; ++par) {
    cudaGraph_t gr;
    ck(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed), "capture");
    enqueue_iteration(ss, par, cs);
    ck(cudaStreamEndCapture(cs, &gr), "capture end");
    ck(cudaGraphInstantiate(&ss->graph[par], gr, 0), "graph instantiate");
    cudaGraphDestroy(gr);
  }
  cudaStreamDestroy(cs);
  ss->gen = ss->plan->gen;
}

// graphs of a session whose plan buffers moved since capture are re-captured
void refresh_graphs(lsopc_session* ss) {
  if (ss->gen != ss->plan->gen && (ss->graph[0] || ss->graph[1])) capture_graphs(ss);
}

}  // namespace

extern "C" {

int lsopc_session_create(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus,
                         const uint8_t* target_dev, const double* phi0_dev, const double* mod_dev,
                         const lsopc_config* cfg, void* stream, lsopc_session** out) {
  return guarded([&] {
    check_plan(plan);
    check_kset(plan, focus);
    check_kset(plan, defocus);
    if (!cfg || !out) throw Error(LSOPC_EINVAL, "null argument");
    if (cfg->max_iters < 0) throw Error(LSOPC_EINVAL, "max_iters must be >= 0");
    if (cfg->cg_restart_every < 1) throw Error(LSOPC_EINVAL, "cg_restart_every must be >= 1");
    if (cfg->grad_scheme != 0 && cfg->grad_scheme != 1) throw Error(LSOPC_EINVAL, "grad_scheme must be 0 or 1");
    if (cfg->reinit_every < 0) throw Error(LSOPC_EINVAL, "reinit_every must be >= 0");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Grid& g = plan->g;
    const size_t n = g.n();
    lsopc_session* ss = take_pooled(plan, focus, defocus, *cfg, mod_dev != nullptr);
    const bool fresh = ss == nullptr;
    if (fresh) ss = new lsopc_session();
    try {
      ss->plan = plan;
      ss->focus = focus;
      ss->defocus = defocus;
      ss->cfg = *cfg;
      ss->s = s;
      ss->it = 0;
      ss->have_mod = mod_dev != nullptr;
      ss->tiled = false;  // a pooled strip session comes back as a whole-grid one
      ss->tile = Tile{};
      plan->ensure_T(focus->nk + defocus->nk);
      if (fresh) {
        ss->target.ensure(n);
        ss->phi.ensure(n * 8);
        ss->best.ensure(n * 8);
        for (int i = 0; i < 2; ++i) {
          ss->v[i].ensure(n * 8);
          ss->d[i].ensure(n * 8);
        }
        ss->u.ensure(n * 8);
        if (cfg->update_form) ss->gm.ensure(n * 8);
        ss->mask.ensure(n);
        ss->hist.ensure((size_t)(cfg->max_iters + 1) * 7 * sizeof(double));
        ss->state.ensure(sizeof(DevState));
        ss->part_ls.ensure((size_t)ls_blocks() * 2 * sizeof(double));
        ss->part_up.ensure((size_t)ls_blocks() * sizeof(double));
        ss->dots.ensure((size_t)(finish_max_blocks() + 1) * 2 * sizeof(double));
        if (mod_dev) ss->mod.ensure(n * 8);
        if (cfg->reinit_every > 0) ss->rein.ensure(((size_t)ls_blocks() + 2) * sizeof(double));
      }
      if (cfg->reinit_every > 0) {
        plan->tsdf_i.ensure(tsdf_scratch_i32(g.H, g.W) * sizeof(int));
        plan->tsdf_f.ensure(tsdf_scratch_f64(g.H, g.W) * sizeof(double));
      }
      ck(cudaMemcpyAsync(ss->target.p, target_dev, n, cudaMemcpyDeviceToDevice, s), "memcpy");
      launch_binarize_u8(n, ss->target.as<uint8_t>(), s);  // any non-zero byte is lit (optimizer.py:197)
      // optimizer.py:197-201: uniform target -> DegenerateInputError
      if (!cfg->skip_target_check) {
        double lit = reduce_to_host(RD_COUNTNEQ8, n, nullptr, nullptr, ss->target.as<uint8_t>(), nullptr, plan, s);
        if (lit == 0.0 || lit == (double)n) throw Error(LSOPC_EDEGENERATE, "target layout is uniform");
      }
      if (phi0_dev) {
        ck(cudaMemcpyAsync(ss->phi.p, phi0_dev, n * 8, cudaMemcpyDeviceToDevice, s), "memcpy");
      } else {
        plan->tsdf_i.ensure(tsdf_scratch_i32(g.H, g.W) * sizeof(int));
        plan->tsdf_f.ensure(tsdf_scratch_f64(g.H, g.W) * sizeof(double));
        launch_tsdf(g.H, g.W, ss->target.as<uint8_t>(), cfg->d_upper, cfg->d_lower, ss->phi.as<double>(),
                    plan->tsdf_i.as<int>(), plan->tsdf_f.as<double>(), s);
        ck_launch("tsdf");
      }
      if (mod_dev) ck(cudaMemcpyAsync(ss->mod.p, mod_dev, n * 8, cudaMemcpyDeviceToDevice, s), "memcpy");
      ck(cudaMemcpyAsync(ss->best.p, ss->phi.p, n * 8, cudaMemcpyDeviceToDevice, s), "memcpy");
      launch_elementwise(EW_MASK, n, ss->phi.as<double>(), nullptr, 0, 0, 0, nullptr, ss->mask.as<uint8_t>(), s);
      DevState h{};
      h.best = std::numeric_limits<double>::infinity();
      h.nonfinite_it = -1;
      ck(cudaMemcpyAsync(ss->state.p, &h, sizeof(h), cudaMemcpyHostToDevice, s), "memcpy");
      for (int i = 0; i < 2; ++i) ck(cudaMemsetAsync(ss->v[i].p, 0, n * 8, s), "memset");
      ck(cudaStreamSynchronize(s), "sync");
      if (fresh) capture_graphs(ss);
      else refresh_graphs(ss);  // a pooled session whose plan buffers were reallocated
      if (fresh) {
        ck(cudaHostAlloc(&ss->hflag, 2 * sizeof(int), cudaHostAllocDefault), "host alloc");
        for (auto& e : ss->ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      }
    } catch (...) {
      delete ss;
      throw;
    }
    *out = ss;
  });
}

int lsopc_session_enqueue(lsopc_session* ss, int n) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    refresh_graphs(ss);  // another call on this plan may have grown T / A meanwhile
    for (int i = 0; i < n && ss->it < ss->cfg.max_iters; ++i) {
      if (ss->graph[ss->it & 1]) ck(cudaGraphLaunch(ss->graph[ss->it & 1], ss->s), "graph launch");
      else enqueue_iteration(ss, ss->it & 1, ss->s);
      ++ss->it;
    }
  });
}

int lsopc_session_poll(lsopc_session* ss, int* stopped, int* iters_enqueued) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    DevState h{};
    ck(cudaMemcpyAsync(&h, ss->state.p, sizeof(h), cudaMemcpyDeviceToHost, ss->s), "memcpy");
    ck(cudaStreamSynchronize(ss->s), "sync");
    if (stopped) *stopped = h.stopped;
    if (iters_enqueued) *iters_enqueued = ss->it;
  });
}

int lsopc_session_finish(lsopc_session* ss, double* best_phi_dev, uint8_t* final_mask_dev, double* history_host,
                         lsopc_result* res) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    lsopc_plan* p = ss->plan;
    const Grid& g = p->g;
    const size_t n = g.n();
    cudaStream_t s = ss->s;
    DevState h{};
    ck(cudaMemcpyAsync(&h, ss->state.p, sizeof(h), cudaMemcpyDeviceToHost, s), "memcpy");
    ck(cudaStreamSynchronize(s), "sync");
    if (h.nonfinite_it >= 0)
      throw Error(LSOPC_ENUMERIC, "non-finite loss at iteration " + std::to_string(h.nonfinite_it));
    if (history_host && h.nhist > 0)
      ck(cudaMemcpy(history_host, ss->hist.p, (size_t)h.nhist * 7 * sizeof(double), cudaMemcpyDeviceToHost),
         "memcpy");
    // optimizer.py:271-277: best phi -> mask -> hard corners -> L2 / PVB.  The
    // forward that found the best iterate already counted its hard prints
    // (same mask bytes, same kernels: bit-identical intensities), so a
    // whole-grid session takes those counts; strips and sessions without an
    // iteration run the final forward.
    uint8_t* fm = final_mask_dev ? final_mask_dev : ss->mask.as<uint8_t>();
    launch_elementwise(EW_MASK, n, ss->best.as<double>(), nullptr, 0, 0, 0, nullptr, fm, s);
    double l2, pvb;
    if (!ss->tiled && h.have_counts) {
      l2 = h.best_l2;
      pvb = h.best_pvb;
    } else {
      forward(p, ss->focus, ss->defocus, nullptr, s, fm, nullptr, nullptr);
      uint8_t* hn = p->hard.as<uint8_t>();
      ResistParams rp{ss->cfg.i_th, ss->cfg.sigma_z, 0.0, 0.0};
      launch_resist(g, p->If.p, p->Id.p, nullptr, nullptr, rp, nullptr, nullptr, nullptr, nullptr, nullptr, hn,
                    hn + n, hn + 2 * n, nullptr, nullptr, s);
      ck_launch("final prints");
      const int cw = ss->tiled ? g.W : 0;  // strip: count the interior columns only
      l2 = reduce_to_host(RD_COUNTNEQ8, n, nullptr, nullptr, hn, ss->target.as<uint8_t>(), p, s, cw, ss->tile);
      pvb = reduce_to_host(RD_COUNTNEQ8, n, nullptr, nullptr, hn + n, hn + 2 * n, p, s, cw, ss->tile);
    }
    if (best_phi_dev) ck(cudaMemcpyAsync(best_phi_dev, ss->best.p, n * 8, cudaMemcpyDeviceToDevice, s), "memcpy");
    ck(cudaStreamSynchronize(s), "sync");
    if (res) {
      res->iters = h.nhist;
      res->l2 = (int)l2;
      res->pvband = (int)pvb;
      res->nonfinite_iter = h.nonfinite_it;
    }
  });
}

int lsopc_session_phi(lsopc_session* ss, double* phi_dev) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    ck(cudaMemcpyAsync(phi_dev, ss->phi.p, ss->plan->n() * 8, cudaMemcpyDeviceToDevice, ss->s), "memcpy");
  });
}

int lsopc_session_losses(lsopc_session* ss, double* l_ilt, double* l_pvb, double* l_dso) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    lsopc_plan* p = ss->plan;
    const Grid& g = p->g;
    const lsopc_config& c = ss->cfg;
    cudaStream_t s = ss->s;
    SpecSet sets[2] = {spec_set(p, ss->focus, 0, 0), spec_set(p, ss->defocus, 1, ss->focus->nk)};
    // _forward_losses on mask_from_phi(phi) (optimizer.py:172-177, 334-336); not gated by the stop flag
    mask_and_f1(p, sets, 2, nullptr, nullptr, ss->phi.as<double>(), nullptr, s);
    launch_f2(g, sets, 2, nullptr, nullptr, s);
    ResistParams rp{c.i_th, c.sigma_z, c.alpha, c.beta};
    ss->scalars.ensure(8 * sizeof(double));
    double* sc = ss->scalars.as<double>();
    launch_resist(g, p->If.p, p->Id.p, ss->target.as<uint8_t>(), nullptr, rp, nullptr, nullptr, nullptr, nullptr,
                  nullptr, nullptr, nullptr, nullptr, p->partials.as<double>(), nullptr, s);
    launch_reduce_partials(p->partials.as<double>(), reduce_blocks(), 4, 0, sc, s);
    double h[2];
    ck(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, s), "memcpy");
    ck(cudaStreamSynchronize(s), "sync");
    if (l_ilt) *l_ilt = h[0];
    if (l_pvb) *l_pvb = h[1];
    if (l_dso) *l_dso = c.alpha * h[0] + c.beta * h[1];
  });
}

int lsopc_session_destroy(lsopc_session* ss) {
  return guarded([&] {
    if (!ss) return;
    ck(cudaStreamSynchronize(ss->s), "sync");
    give_to_pool(ss);
  });
}

int lsopc_dsn_init(size_t n, const float* phi_raw_dev, const float* m_raw_dev, double d_lower, double d_upper,
                   double epsilon, double* phi0_dev, double* m_dev, void* stream) {
  return guarded([&] {
    if (!(d_lower < 0.0 && 0.0 < d_upper)) throw Error(LSOPC_EINVAL, "truncation bounds must satisfy D_l < 0 < D_u");
    if (!(epsilon > 0.0)) throw Error(LSOPC_EINVAL, "epsilon must be positive");
    if (n == 0) return;
    launch_dsn_init(n, phi_raw_dev, m_raw_dev, d_lower, d_upper, epsilon, phi0_dev, m_dev,
                    static_cast<cudaStream_t>(stream));
    ck_launch("dsn init");
  });
}

int lsopc_session_set_window(lsopc_session* ss, int ix0, int ix1, int xlo, int xhi, int iy0, int iy1, int ylo,
                             int yhi) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    const int W = ss->plan->g.W, H = ss->plan->g.H;
    if (!(0 <= ix0 && ix0 < ix1 && ix1 <= W && 0 <= xlo && xlo <= ix0 && ix1 <= xhi && xhi <= W))
      throw Error(LSOPC_EINVAL, "bad strip geometry (columns)");
    if (!(0 <= iy0 && iy0 < iy1 && iy1 <= H && 0 <= ylo && ylo <= iy0 && iy1 <= yhi && yhi <= H))
      throw Error(LSOPC_EINVAL, "bad strip geometry (rows)");
    if (ss->it) throw Error(LSOPC_EINVAL, "set the strip before the first iteration");
    if (ss->cfg.reinit_every > 0) throw Error(LSOPC_EINVAL, "reinitialisation needs the whole grid (not a strip)");
    ss->tiled = true;
    ss->tile = Tile{ix0, ix1, xlo, xhi, iy0, iy1, ylo, yhi};
    ss->scalars.ensure(8 * sizeof(double));
    ck(cudaMemsetAsync(ss->scalars.p, 0, 8 * sizeof(double), ss->s), "memset");
  });
}

int lsopc_session_phase(lsopc_session* ss, int phase) {
  return guarded([&] {
    if (!ss || !ss->tiled) throw Error(LSOPC_EINVAL, "phases need a strip session (lsopc_session_set_tile)");
    if (phase < 0 || phase > 6) throw Error(LSOPC_EINVAL, "phase must be 0..6");
    if (phase == 0 && ss->it >= ss->cfg.max_iters) throw Error(LSOPC_EINVAL, "max_iters reached");
    enqueue_phase(ss, phase, ss->s);
    if (phase == 4) ++ss->it;
  });
}

int lsopc_session_set_tile(lsopc_session* ss, int ix0, int ix1, int xlo, int xhi) {
  if (!ss) return lsopc_session_set_window(ss, ix0, ix1, xlo, xhi, 0, 1, 0, 1);
  const int H = ss->plan->g.H;
  return lsopc_session_set_window(ss, ix0, ix1, xlo, xhi, 0, H, 0, H);
}

double* lsopc_session_scalars(lsopc_session* ss) { return ss ? ss->scalars.as<double>() : nullptr; }
double* lsopc_session_phi_ptr(lsopc_session* ss) { return ss ? ss->phi.as<double>() : nullptr; }
int* lsopc_session_state_flag(lsopc_session* ss) { return ss ? &ss->st()->stopped : nullptr; }

int lsopc_session_time_passes(lsopc_session* ss, int reps, double* ms_out) {
  return guarded([&] {
    if (!ss) throw Error(LSOPC_EINVAL, "null session");
    if (reps < 1) throw Error(LSOPC_EINVAL, "reps must be >= 1");
    cudaEvent_t ev[PS_N + 1];
    for (auto& e : ev) ck(cudaEventCreate(&e), "event");
    double acc[PS_N] = {0};
    for (int r = 0; r < reps && ss->it < ss->cfg.max_iters; ++r) {
      enqueue_iteration(ss, ss->it & 1, ss->s, ev);
      ++ss->it;
      ck(cudaEventSynchronize(ev[PS_N]), "sync");
      for (int i = 0; i < PS_N; ++i) {
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]), "elapsed");
        acc[i] += ms;
      }
    }
    for (int i = 0; i < PS_N; ++i) ms_out[i] = acc[i] / reps;
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int lsopc_session_launches_per_iter(const lsopc_session* ss) {
  if (!ss) return 0;
  // mask rows+cols 2, F1 1, F2 1, resist (+ loss control) 1, copy_best 1, A1 1, A2 1,
  // A3 (+ CG control) 1, velocity (+ CFL control) 1, update (+ record) 1;
  // opt-in reinitialisation: lit count 2, gate 1, TSDF 3
  return 2 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + (ss->cfg.reinit_every > 0 ? 6 : 0);
}

int lsopc_optimize(lsopc_plan* plan, const lsopc_kset* focus, const lsopc_kset* defocus, const uint8_t* target_dev,
                   const double* phi0_dev, const double* mod_dev, const lsopc_config* cfg, double* best_phi_dev,
                   uint8_t* final_mask_dev, double* history_host, lsopc_result* result, void* stream) {
  lsopc_session* ss = nullptr;
  int rc = lsopc_session_create(plan, focus, defocus, target_dev, phi0_dev, mod_dev, cfg, stream, &ss);
  if (rc) return rc;
  // Keep one chunk queued ahead: enqueue chunk k+1, then wait for chunk k and
  // read its stop flag (copied to pinned memory behind it).  Once the device
  // stop rule fires, every later kernel exits at entry, so over-enqueueing
  // costs at most one chunk of empty launches.
  const int chunk = 4;
  auto enqueue_chunk = [&](int slot) -> int {
    int r = lsopc_session_enqueue(ss, chunk);
    if (r) return r;
    r = guarded([&] {
      ck(cudaMemcpyAsync(&ss->hflag[slot], &ss->st()->stopped, sizeof(int), cudaMemcpyDeviceToHost, ss->s),
         "memcpy");
      ck(cudaEventRecord(ss->ev[slot], ss->s), "event");
    });
    return r;
  };
  rc = enqueue_chunk(0);
  for (int k = 0; !rc; ++k) {
    const bool more = ss->it < cfg->max_iters;
    if (more && (rc = enqueue_chunk((k + 1) & 1))) break;
    rc = guarded([&] { ck(cudaEventSynchronize(ss->ev[k & 1]), "sync"); });
    if (rc || ss->hflag[k & 1] || !more) break;
  }
  if (!rc) rc = lsopc_session_finish(ss, best_phi_dev, final_mask_dev, history_host, result);
  std::string keep = g_err;
  lsopc_session_destroy(ss);
  g_err = keep;
  return rc;
}


}  // extern "C"
