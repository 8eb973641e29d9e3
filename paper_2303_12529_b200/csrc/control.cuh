// Loop control of the DSO iteration (optimizer.py:238-269) as device bodies:
// fixed-order reductions of per-block partials plus the scalar state updates.
// They run either as single-block kernels (levelset.cu: strip phases, where a
// collective sits in between) or as the fused tail of the producing kernel,
// executed by the producer's last block to finish (fence + ticket), which
// saves a launch per control step in the single-GPU graph.
#pragma once
#include "common.cuh"
#include "internal_ls.h"

namespace lsb {

// fixed-order reduction of nb partials (NV per block) by one block; L2 loads
// (partials were written by other SMs in the same kernel when fused)
template <int NV, bool MAX>
LS_D void reduce_partials(const double* part, int nb, double (&out)[NV], double* red) {
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double p = __ldcg(part + NV * b + j);
      acc[j] = MAX ? nmax(acc[j], p) : acc[j] + p;
    }
  }
  if (MAX) block_max<NV>(acc, red);
  else block_sum<NV>(acc, red);
#pragma unroll
  for (int j = 0; j < NV; ++j) out[j] = acc[j];
}

// true in every thread of the block that finishes last; the ticket is
// re-armed by that block (release_ticket) for the next launch / graph replay.
// red: the caller's shared reduction scratch (no static shared memory here,
// so kernels keep their full dynamic allowance)
LS_D bool last_block(unsigned* ticket, double* red) {
  unsigned* flag = reinterpret_cast<unsigned*>(red);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *flag = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  const bool last = *flag != 0;
  __syncthreads();
  if (last) __threadfence();
  return last;
}
LS_D void release_ticket(unsigned* ticket) {
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0;
}

// optimizer.py:238-251: loss, best iterate, patience.  part: 4 partials per
// block (losses, then the hard-print L2 / PVB counts of the same forward)
LS_D void after_forward_body(const double* part, int nb, const LoopCfg& c, DevState* st, double* hist,
                             double* red) {
  if (st->stopped) return;
  double l[4];  // L_ilt, L_pvb, hard-print L2 count, hard-print PVB count
  reduce_partials<4, false>(part, nb, l, red);
  if (threadIdx.x != 0) return;
  const double l_ilt = l[0], l_pvb = l[1];
  const double l_dso = c.alpha * l_ilt + c.beta * l_pvb;
  st->l_ilt = l_ilt;
  st->l_pvb = l_pvb;
  st->l_dso = l_dso;
  st->improved = 0;
  if (!isfinite(l_dso)) {
    st->nonfinite_it = st->it;
    st->stopped = 1;
    return;
  }
  double rel;
  if (l_dso < st->best) {
    rel = isfinite(st->best) ? (st->best - l_dso) / st->best : CUDART_INF;
    st->best = l_dso;
    st->improved = 1;
    st->best_l2 = l[2];
    st->best_pvb = l[3];
    st->have_counts = 1;
  } else {
    rel = 0.0;
  }
  st->streak = rel < c.stop_rel_tol ? st->streak + 1 : 0;
  if (st->streak >= c.stop_patience) {
    double* h = hist + 7 * st->nhist;
    h[0] = l_ilt; h[1] = l_pvb; h[2] = l_dso; h[3] = 0.0; h[4] = 0.0; h[5] = 0.0; h[6] = 0.0;
    st->nhist += 1;
    st->stopped = 1;
  }
}

// optimizer.py:154-169,253: Polak-Ribiere beta with restart
LS_D void after_grad_body(const double* dots, int nb, int restart_every, DevState* st, double* red) {
  if (st->stopped) return;
  const int restart = st->it == 0 || st->it % restart_every == 0;
  double s[2] = {0.0, 0.0};
  if (!restart) reduce_partials<2, false>(dots, nb, s, red);
  if (threadIdx.x != 0) return;
  st->use_beta = 0;
  st->beta = 0.0;
  if (restart || s[1] == 0.0) return;
  double b = s[0] / s[1];
  if (b <= 0.0) return;
  st->beta = b;
  st->use_beta = 1;
}

// optimizer.py:143-151,257-261: dt = eta / max|v_total|
LS_D void after_velocity_body(const double* part, int nb, double eta, DevState* st, double* hist, double* red) {
  if (st->stopped) return;
  double m[2];
  reduce_partials<2, true>(part, nb, m, red);
  if (threadIdx.x != 0) return;
  st->vmax = m[0];
  st->gmax = m[1];
  if (m[0] == 0.0) {
    double* h = hist + 7 * st->nhist;
    h[0] = st->l_ilt; h[1] = st->l_pvb; h[2] = st->l_dso; h[3] = 0.0; h[4] = 0.0; h[5] = 0.0; h[6] = m[1];
    st->nhist += 1;
    st->stopped = 1;
    return;
  }
  st->dt = eta / m[0];
}

// optimizer.py:262-265: history record of a completed step
LS_D void after_update_body(const double* part, int nb, DevState* st, double* hist, double* red) {
  if (st->stopped) return;
  double m[1];
  reduce_partials<1, true>(part, nb, m, red);
  if (threadIdx.x != 0) return;
  double* h = hist + 7 * st->nhist;
  h[0] = st->l_ilt; h[1] = st->l_pvb; h[2] = st->l_dso; h[3] = st->dt; h[4] = st->vmax; h[5] = m[0];
  h[6] = st->gmax;
  st->nhist += 1;
  st->it += 1;
}

}  // namespace lsb
