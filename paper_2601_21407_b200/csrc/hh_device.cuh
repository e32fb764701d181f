// hh_device.cuh -- per-neuron Hodgkin-Huxley step math for sm_100a.
//
// One header is shared by the forward kernel, the backward kernel's segment
// recompute and its adjoint step, so all three round identically (checkpoint
// invariance is bit-exact).  Every floating operation goes through the
// explicit-rounding helpers below, which stops the compiler from contracting
// differently in different kernels.
//
// Two arithmetic flavours, selected by the scalar type:
//   float  -- the throughput build.  exp via MUFU ex2.approx with the
//             -log2(e)/b factor folded on the host, reciprocals via MUFU
//             rcp.approx, rate_scale folded into `a`, the linoid's removable
//             singularity handled by its Bernoulli series for |x/b| < 1
//             (exact to ~2e-8 there, instead of the 1-exp cancellation of
//             dynamics.py:62-65 that fp32 cannot afford).
//   double -- the parity build.  The reference's operation order
//             (dynamics.py:409-440, :476-524; adjoint.py:122-188): true
//             divisions, libdevice exp, the LINOID_EPS=1e-7 branch, scale
//             applied after the rate.  This TU is compiled with -fmad=false
//             so no FMA contraction either, like NumPy.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hhb200.h"

namespace hhb {

constexpr int kMaxGates = HHB_MAX_GATES;
constexpr int kMaxLeak = HHB_MAX_CHANNELS;
// partial-sum slots of the parameter-gradient reduction:
// [0] c_m, [1 + g] channel ending at gate g, [1 + kMaxGates + j] j-th leak channel
constexpr int kSlots = 1 + kMaxGates + kMaxLeak;

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ float ex2_(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ bool finite_(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite_(double x) { return isfinite(x); }

// ---------------------------------------------------------------- tables
// Device copy of hhb_params_t, precomputed per flavour; passed BY VALUE as a
// kernel parameter, so every field is a constant-bank operand.
template <typename T>
struct DevRate {
  int kind;
  T a;      // float: a*rate_scale; double: a
  T v0;
  T b;
  T inv_b;  // 1/b
  T k2;     // float: -log2(e)/b
  T ab;     // float: a*b*scale  (linoid value at the singularity)
};

template <typename T>
struct DevGate {
  DevRate<T> al, be;
  int k;          // exponent
  int first;      // first gate of its channel
  int last;       // last gate of its channel
  int channel;    // owning channel index
  int leak_lo;    // double flavour: leak channels declared after this
  int leak_hi;    //   channel (and before the next gated one), added in order
  T g, e;         // owning channel g_max, e_rev
};

template <typename T>
struct DevTable {
  int ng;
  int nleak;
  int nch;
  int has_scale;
  int leak_head;   // double flavour: leak channels declared before the first gated one
  T scale;
  T dt;
  T dt_cm;         // dt / c_m (host fp64, rounded to T)
  T theta;
  T neg_dt;        // -dt
  T ndl;           // float: -dt*log2(e)
  T leak_g_sum;    // float: sum of leak g
  T leak_ge_sum;   // float: sum of leak g*E
  T cm_coef;       // -(dt / c_m^2)
  T ndt_cm;        // -(dt / c_m)
  T leak_g[kMaxLeak];
  T leak_e[kMaxLeak];
  int leak_ch[kMaxLeak];
  DevGate<T> gate[kMaxGates];
};

template <typename T>
struct DevSur {
  int kind;   // 0 sigmoid-derivative, 1 rectangular
  T w;        // width
  T inv_w;
  T k2;       // float: -log2(e)/w
  T half_inv_w;
};

// ---------------------------------------------------------------- rates
// value of one rate at potential v (RateFn.__call__, dynamics.py:56-65)
__device__ __forceinline__ float rate_val(const DevRate<float>& r, float v) {
  const float x = sub_(v, r.v0);
  const float e = ex2_(mul_(x, r.k2));            // exp(-x/b)
  if (r.kind == HHB_RATE_EXP) return mul_(r.a, e);
  if (r.kind == HHB_RATE_SIGMOID) return mul_(r.a, rcp_(add_(1.0f, e)));
  const float u = mul_(x, r.inv_b);
  const float w = mul_(u, u);
  // u/(1-exp(-u)) = 1 + u/2 + u^2/12 - u^4/720 + u^6/30240 - u^8/1209600
  float f = fma_(w, -8.267195767195767e-07f, 3.3068783068783070e-05f);
  f = fma_(w, f, -1.3888888888888889e-03f);
  f = fma_(w, f, 8.3333333333333333e-02f);
  f = fma_(w, f, fma_(u, 0.5f, 1.0f));
  const float series = mul_(r.ab, f);
  const float direct = mul_(mul_(r.a, x), rcp_(sub_(1.0f, e)));
  return (fabsf(u) < 1.0f) ? series : direct;
}

__device__ __forceinline__ double rate_val(const DevRate<double>& r, double v) {
  const double x = sub_(v, r.v0);
  const double e = exp(-x / r.b);                 // np.negative, np.divide, np.exp
  if (r.kind == HHB_RATE_EXP) return mul_(e, r.a);
  if (r.kind == HHB_RATE_SIGMOID) return r.a / add_(e, 1.0);
  const double den = sub_(1.0, e);
  if (fabs(den) < 1e-7) return mul_(r.a, r.b);    // LINOID_EPS branch
  return mul_(x, r.a) / den;
}

// value and slope (RateFn.__call__ + RateFn.deriv, dynamics.py:56-79)
__device__ __forceinline__ void rate_val_slope(const DevRate<float>& r, float v, float& val,
                                               float& slope) {
  const float x = sub_(v, r.v0);
  const float e = ex2_(mul_(x, r.k2));
  if (r.kind == HHB_RATE_EXP) {
    val = mul_(r.a, e);
    slope = mul_(-r.inv_b, val);
    return;
  }
  if (r.kind == HHB_RATE_SIGMOID) {
    const float s = rcp_(add_(1.0f, e));
    val = mul_(r.a, s);
    slope = mul_(mul_(val, r.inv_b), sub_(1.0f, s));
    return;
  }
  const float u = mul_(x, r.inv_b);
  const float w = mul_(u, u);
  float f = fma_(w, -8.267195767195767e-07f, 3.3068783068783070e-05f);
  f = fma_(w, f, -1.3888888888888889e-03f);
  f = fma_(w, f, 8.3333333333333333e-02f);
  f = fma_(w, f, fma_(u, 0.5f, 1.0f));
  // f'(u) = 1/2 + u/6 - u^3/180 + u^5/5040 - u^7/151200 + u^9/4790016
  float d = fma_(w, 2.0876756987868099e-07f, -6.6137566137566138e-06f);
  d = fma_(w, d, 1.9841269841269841e-04f);
  d = fma_(w, d, -5.5555555555555556e-03f);
  d = fma_(w, d, 1.6666666666666667e-01f);
  d = fma_(u, d, 0.5f);
  const float den = sub_(1.0f, e);
  const float rd = rcp_(den);
  const bool small = fabsf(u) < 1.0f;
  val = small ? mul_(r.ab, f) : mul_(mul_(r.a, x), rd);
  // a*(den - u*e)/den^2 ; r.a already carries rate_scale
  slope = small ? mul_(r.a, d)
                : mul_(mul_(r.a, sub_(den, mul_(u, e))), mul_(rd, rd));
}

__device__ __forceinline__ void rate_val_slope(const DevRate<double>& r, double v, double& val,
                                               double& slope) {
  const double x = sub_(v, r.v0);
  const double e = exp(-x / r.b);
  if (r.kind == HHB_RATE_EXP) {
    val = mul_(e, r.a);
    slope = mul_(-(r.a / r.b), e);
    return;
  }
  if (r.kind == HHB_RATE_SIGMOID) {
    val = r.a / add_(e, 1.0);
    const double s = 1.0 / add_(1.0, e);
    slope = mul_(mul_(r.a / r.b, s), sub_(1.0, s));
    return;
  }
  const double den = sub_(1.0, e);
  if (fabs(den) < 1e-7) {
    val = mul_(r.a, r.b);
    slope = mul_(0.5, r.a);
    return;
  }
  val = mul_(x, r.a) / den;
  slope = mul_(r.a, sub_(den, mul_(x, e) / r.b)) / mul_(den, den);
}

// ---------------------------------------------------------------- pieces
template <typename T>
__device__ __forceinline__ T ipow_(T p, int k) {  // int_pow, dynamics.py:349-357
  if (k == 0) return T(1);
  T out = p;
  for (int i = 1; i < k; ++i) out = mul_(out, p);
  return out;
}

template <typename T>
__device__ __forceinline__ T scaled(const DevTable<T>& tb, T x) {
  if constexpr (sizeof(T) == 8) {
    return tb.has_scale ? mul_(x, tb.scale) : x;
  } else {
    return x;  // folded into a on the host
  }
}

// exponential-Euler gate update (dynamics.py:492-508)
__device__ __forceinline__ float gate_update(const DevTable<float>& tb, float p, float a, float b) {
  const float s = add_(a, b);
  const float pinf = mul_(a, rcp_(s));
  const float dec = ex2_(mul_(s, tb.ndl));
  const float pn = fma_(sub_(p, pinf), dec, pinf);
  return (s == 0.0f) ? p : pn;
}
__device__ __forceinline__ double gate_update(const DevTable<double>& tb, double p, double a,
                                              double b) {
  double s = add_(a, b);
  const bool zero = (s == 0.0);
  const double sd = zero ? 1.0 : s;
  const double pinf = a / sd;
  const double dec = exp(mul_(zero ? 0.0 : s, tb.neg_dt));
  const double pn = add_(mul_(sub_(p, pinf), dec), pinf);
  return zero ? p : pn;
}

// Ionic current of the channels without gates.  float: all leaks folded into
// one FMA.  double: the leaks declared before the first gated channel, in
// declaration order (the rest are added after their predecessor, see
// leak_after), so I_ion is summed in the reference's channel order
// (dynamics.py:476-516; the first add onto 0.0 is exact).
__device__ __forceinline__ float leak_current(const DevTable<float>& tb, float v) {
  return fma_(tb.leak_g_sum, v, -tb.leak_ge_sum);
}
__device__ __forceinline__ double leak_current(const DevTable<double>& tb, double v) {
  double ion = 0.0;
  for (int j = 0; j < tb.leak_head; ++j) ion = add_(ion, mul_(sub_(v, tb.leak_e[j]), tb.leak_g[j]));
  return ion;
}
__device__ __forceinline__ float leak_after(const DevTable<float>&, const DevGate<float>&, float,
                                            float ion) {
  return ion;
}
__device__ __forceinline__ double leak_after(const DevTable<double>& tb, const DevGate<double>& G,
                                             double v, double ion) {
  for (int j = G.leak_lo; j < G.leak_hi; ++j)
    ion = add_(ion, mul_(sub_(v, tb.leak_e[j]), tb.leak_g[j]));
  return ion;
}
__device__ __forceinline__ float channel_term(float g, float e, float eta, float v) {
  return mul_(mul_(eta, g), sub_(v, e));
}
__device__ __forceinline__ double channel_term(double g, double e, double eta, double v) {
  return mul_(mul_(eta, g), sub_(v, e));
}
template <typename T>
__device__ __forceinline__ T membrane(const DevTable<T>& tb, T v, T cur, T ion) {
  if constexpr (sizeof(T) == 4) {
    return fma_(sub_(cur, ion), tb.dt_cm, v);
  } else {
    return add_(v, mul_(sub_(cur, ion), tb.dt_cm));
  }
}

// ---------------------------------------------------------------- forward
// One fused step for one neuron (hh_step, dynamics.py:472-528).  Gates and the
// ionic sum read the pre-update V and gates.  p[] is updated in place; the
// new potential is returned.
template <typename T, int NG>
__device__ __forceinline__ T step_forward(const DevTable<T>& tb, T v, T (&p)[NG > 0 ? NG : 1],
                                          T cur) {
  T ion = leak_current(tb, v);
  T eta = T(1);
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const DevGate<T>& G = tb.gate[g];
    const T pk = ipow_(p[g], G.k);
    eta = G.first ? pk : mul_(eta, pk);
    const T a = scaled(tb, rate_val(G.al, v));
    const T b = scaled(tb, rate_val(G.be, v));
    p[g] = gate_update(tb, p[g], a, b);
    if (G.last) ion = leak_after(tb, G, v, add_(ion, channel_term(G.g, G.e, eta, v)));
  }
  return membrane(tb, v, cur, ion);
}

// ---------------------------------------------------------------- surrogate
__device__ __forceinline__ float surrogate(const DevSur<float>& s, float u) {
  if (s.kind == HHB_SUR_RECTANGULAR) return (fabsf(u) <= s.w) ? s.half_inv_w : 0.0f;
  const float q = rcp_(add_(1.0f, ex2_(mul_(u, s.k2))));
  return mul_(mul_(q, sub_(1.0f, q)), s.inv_w);
}
__device__ __forceinline__ double surrogate(const DevSur<double>& s, double u) {
  if (s.kind == HHB_SUR_RECTANGULAR) return (fabs(u) <= s.w) ? 0.5 / s.w : 0.0;
  const double q = 1.0 / add_(1.0, exp(-u / s.w));
  return mul_(q, sub_(1.0, q)) / s.w;
}

// ---------------------------------------------------------------- backward
// Adjoint of step_forward for one neuron (hh_step_backward, adjoint.py:116-188).
//   in : v, p (the step's input state), cur, d_v = dL/dV' (seed already added),
//        d_p = dL/dp', d_spike
//   out: d_v = dL/dV, d_p = dL/dp, return dL/di
//   acc: += per-slot parameter-gradient sums (scaled by constants at the end)
template <typename T, int NG>
__device__ __forceinline__ T step_backward(const DevTable<T>& tb, const DevSur<T>& sur, T v,
                                           const T (&p)[NG > 0 ? NG : 1], T cur, T& d_v,
                                           T (&d_p)[NG > 0 ? NG : 1], T d_spike, bool has_spike,
                                           double (&acc)[kSlots]) {
  // recompute eta per gate-channel, ionic current, V'
  T pk[NG > 0 ? NG : 1];
  T pre[NG > 0 ? NG : 1];    // product of pk of earlier gates in the same channel
  T eta_end[NG > 0 ? NG : 1];
  T ion = leak_current(tb, v);
  T gsum;
  if constexpr (sizeof(T) == 4) {
    gsum = tb.leak_g_sum;
  } else {
    gsum = 0.0;
    for (int j = 0; j < tb.nleak; ++j) gsum = add_(gsum, tb.leak_g[j]);
  }
  T eta = T(1);
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const DevGate<T>& G = tb.gate[g];
    pk[g] = ipow_(p[g], G.k);
    pre[g] = G.first ? T(1) : eta;
    eta = G.first ? pk[g] : mul_(eta, pk[g]);
    eta_end[g] = eta;
    if (G.last) {
      ion = leak_after(tb, G, v, add_(ion, channel_term(G.g, G.e, eta, v)));
      gsum = add_(gsum, mul_(G.g, eta));
    }
  }
  const T vn = membrane(tb, v, cur, ion);

  T g_vp = d_v;
  if (has_spike) g_vp = add_(g_vp, mul_(d_spike, surrogate(sur, sub_(vn, tb.theta))));
  const T d_i = mul_(g_vp, tb.dt_cm);

  acc[0] += double(mul_(g_vp, sub_(cur, ion)));
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const DevGate<T>& G = tb.gate[g];
    if (G.last) acc[1 + g] += double(mul_(mul_(g_vp, eta_end[g]), sub_(v, G.e)));
  }
#pragma unroll
  for (int j = 0; j < kMaxLeak; ++j)  // compile-time slot index keeps acc[] in registers
    if (j < tb.nleak) acc[1 + kMaxGates + j] += double(mul_(g_vp, sub_(v, tb.leak_e[j])));

  T dv_in = mul_(g_vp, sub_(T(1), mul_(tb.dt_cm, gsum)));

  // suffix products of pk within each channel (for d eta / d p)
  T suf[NG > 0 ? NG : 1];
  T run = T(1);
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    const DevGate<T>& G = tb.gate[g];
    suf[g] = G.last ? T(1) : run;
    run = G.last ? pk[g] : mul_(run, pk[g]);
  }

#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const DevGate<T>& G = tb.gate[g];
    T a, b, da, db;
    rate_val_slope(G.al, v, a, da);
    rate_val_slope(G.be, v, b, db);
    a = scaled(tb, a);
    b = scaled(tb, b);
    da = scaled(tb, da);
    db = scaled(tb, db);
    const T s = add_(a, b);
    const T up = d_p[g];
    T dp;
    if constexpr (sizeof(T) == 4) {
      const float rs = rcp_(s);
      const float e = ex2_(mul_(s, tb.ndl));
      const float pinf = mul_(a, rs);
      const float dpinf = mul_(sub_(mul_(da, b), mul_(a, db)), mul_(rs, rs));
      const float term = fma_(dpinf, sub_(1.0f, e),
                              mul_(sub_(p[g], pinf), mul_(mul_(tb.neg_dt, add_(da, db)), e)));
      const bool pos = s > 0.0f;
      dv_in = pos ? fma_(up, term, dv_in) : dv_in;
      dp = pos ? mul_(up, e) : up;
    } else {
      const bool pos = s > 0.0;
      const double ss = pos ? s : 1.0;
      const double e = exp(mul_(-tb.dt, s));
      const double pinf = pos ? a / ss : p[g];
      dp = mul_(up, pos ? e : 1.0);
      const double dpinf = pos ? sub_(mul_(da, b), mul_(a, db)) / mul_(ss, ss) : 0.0;
      const double dedv = mul_(mul_(-tb.dt, add_(da, db)), e);
      const double term = pos ? add_(mul_(dpinf, sub_(1.0, e)), mul_(sub_(p[g], pinf), dedv)) : 0.0;
      dv_in = add_(dv_in, mul_(up, term));
    }
    if (G.k > 0) {
      // d eta / d p = k p^(k-1) * prod(other gates of the channel)
      T der = mul_(T(G.k), ipow_(p[g], G.k - 1));
      der = mul_(der, mul_(pre[g], suf[g]));
      dp = add_(dp, mul_(mul_(mul_(mul_(g_vp, tb.ndt_cm), G.g), sub_(v, G.e)), der));
    }
    d_p[g] = dp;
  }
  d_v = dv_in;
  return d_i;
}

}  // namespace hhb
