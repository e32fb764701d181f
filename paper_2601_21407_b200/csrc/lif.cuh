// lif.cuh -- the LIF baseline of the reference (dynamics.py:227-244, :532-538;
// adjoint.py:197-227), the paper's comparison neuron:
//   k_lif_forward   T steps per launch, V in registers, V trace + spikes out
//   k_lif_backward  the per-step adjoint with the surrogate reset factor
// Operation order follows the reference (v + k (i - v); d_v_pre = g_v_out
// ((1 - s) + (v_reset - v_pre) sg) + g_spike sg), so the float64 build
// matches NumPy (compiled with -fmad=false).
#pragma once

#include "hh_host.cuh"

namespace hhb {
namespace lif {

template <typename T>
__global__ void k_lif_forward(int64_t n, int64_t steps, T k, T theta, T v_reset, const T* v_in, const T* i_ext,
                              int64_t i_st, int64_t i_sn, T* v_out, uint8_t* spk_out, T* v_fin) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  T v = v_in[j];
  for (int64_t t = 0; t < steps; ++t) {
    const T cur = i_ext[t * i_st + j * i_sn];
    const T vn = add_(v, mul_(k, sub_(cur, v)));
    const bool s = vn >= theta;
    v = s ? v_reset : vn;
    if (v_out) v_out[t * n + j] = v;
    if (spk_out) spk_out[t * n + j] = s ? 1 : 0;
  }
  v_fin[j] = v;
}

template <typename T>
__global__ void k_lif_backward(int64_t n, T k, T theta, T v_reset, DevSur<T> sur, const T* v, const T* i_ext,
                               int64_t i_sn, const T* g_v_out, const T* g_spike, T* d_v_in, T* d_i,
                               long long* bad) {
  const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const T vp = add_(v[j], mul_(k, sub_(i_ext[j * i_sn], v[j])));
  const T s = vp >= theta ? T(1) : T(0);
  const T sg = surrogate(sur, sub_(vp, theta));
  const T gs = g_spike ? g_spike[j] : T(0);
  const T dvp = add_(mul_(g_v_out[j], add_(sub_(T(1), s), mul_(sub_(v_reset, vp), sg))), mul_(gs, sg));
  const T dv = mul_(dvp, sub_(T(1), k));
  d_v_in[j] = dv;
  d_i[j] = mul_(dvp, k);
  if (!finite_(dv)) atomicMax(bad, 0LL);
}

}  // namespace lif
}  // namespace hhb
