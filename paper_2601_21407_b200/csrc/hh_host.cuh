// hh_host.cuh -- host-side packing of the C-ABI tables into the per-flavour
// device tables, launch geometry, and the launcher templates that the two
// flavour TUs (hh_f32.cu, hh_f64.cu) instantiate.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hh_kernels.cuh"

namespace hhb {

void set_error(const std::string& msg);  // capi.cu, thread-local

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

inline int cuda_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HHB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HHB_OK;
}

constexpr double kLog2e = 1.4426950408889634;
constexpr int kNumSMs = 148;

// ConfigurationError checks of dynamics.py:50-54, :106-108, :140-142, :178-188
// plus the structural invariants of the flattened table.
inline int check_params(const hhb_params_t* P) {
  if (P == nullptr) return fail(HHB_EINVAL, "params is NULL");
  if (P->n_gates < 0 || P->n_gates > HHB_MAX_GATES)
    return fail(HHB_EINVAL, "n_gates out of range [0, 8]");
  if (P->n_channels < 0 || P->n_channels > HHB_MAX_CHANNELS)
    return fail(HHB_EINVAL, "n_channels out of range [0, 8]");
  if (!(P->c_m > 0)) return fail(HHB_EINVAL, "c_m must be > 0");
  if (!(P->dt > 0)) return fail(HHB_EINVAL, "dt must be > 0");
  if (!(P->rate_scale > 0)) return fail(HHB_EINVAL, "rate_scale must be > 0");
  int next = 0;
  for (int c = 0; c < P->n_channels; ++c) {
    const hhb_channel_t& C = P->channels[c];
    if (!(C.g_max >= 0)) return fail(HHB_EINVAL, "channel g_max must be >= 0");
    if (C.gate_begin != next || C.gate_count < 0)
      return fail(HHB_EINVAL, "channel gate ranges must be contiguous in declaration order");
    next += C.gate_count;
  }
  if (next != P->n_gates) return fail(HHB_EINVAL, "channel gate counts do not sum to n_gates");
  for (int c = 0; c < P->n_channels; ++c) {
    const hhb_channel_t& C = P->channels[c];
    for (int g = C.gate_begin; g < C.gate_begin + C.gate_count; ++g)
      if (P->gates[g].channel != c) return fail(HHB_EINVAL, "gate channel index mismatch");
  }
  for (int g = 0; g < P->n_gates; ++g) {
    const hhb_gate_t& G = P->gates[g];
    if (G.exponent < 0) return fail(HHB_EINVAL, "gate exponent must be a non-negative integer");
    for (const hhb_rate_t* r : {&G.alpha, &G.beta}) {
      if (r->kind < 0 || r->kind > 2) return fail(HHB_EINVAL, "unknown rate kind");
      if (r->b == 0.0) return fail(HHB_EINVAL, "rate slope parameter b must be nonzero");
    }
  }
  return HHB_OK;
}

template <typename T>
inline DevRate<T> pack_rate(const hhb_rate_t& r, double scale) {
  DevRate<T> d{};
  d.kind = r.kind;
  d.v0 = T(r.v0);
  d.b = T(r.b);
  d.inv_b = T(1.0 / r.b);
  if constexpr (sizeof(T) == 4) {
    d.a = T(r.a * scale);
    d.k2 = T(-kLog2e / r.b);
    d.ab = T(r.a * r.b * scale);
  } else {
    d.a = r.a;
    d.k2 = -kLog2e / r.b;
    d.ab = r.a * r.b;
  }
  return d;
}

template <typename T>
inline DevTable<T> pack_table(const hhb_params_t* P) {
  DevTable<T> tb{};
  tb.ng = P->n_gates;
  tb.nch = P->n_channels;
  tb.has_scale = P->rate_scale != 1.0;
  tb.scale = T(P->rate_scale);
  tb.dt = T(P->dt);
  tb.dt_cm = T(P->dt / P->c_m);
  tb.theta = T(P->v_theta);
  tb.neg_dt = T(-P->dt);
  tb.ndl = T(-P->dt * kLog2e);
  tb.cm_coef = T(-(P->dt / (P->c_m * P->c_m)));
  tb.ndt_cm = T(-(P->dt / P->c_m));
  double gsum = 0.0, gesum = 0.0;
  int nleak = 0;
  int last_gated_gate = -1;  // last gate of the most recent gated channel
  for (int c = 0; c < P->n_channels; ++c) {
    const hhb_channel_t& C = P->channels[c];
    if (C.gate_count == 0) {
      tb.leak_g[nleak] = T(C.g_max);
      tb.leak_e[nleak] = T(C.e_rev);
      tb.leak_ch[nleak] = c;
      gsum += C.g_max;
      gesum += C.g_max * C.e_rev;
      if (last_gated_gate < 0) {
        tb.leak_head = nleak + 1;
      } else {
        tb.gate[last_gated_gate].leak_hi = nleak + 1;
      }
      ++nleak;
      continue;
    }
    for (int g = C.gate_begin; g < C.gate_begin + C.gate_count; ++g) {
      const hhb_gate_t& G = P->gates[g];
      DevGate<T>& D = tb.gate[g];
      D.al = pack_rate<T>(G.alpha, P->rate_scale);
      D.be = pack_rate<T>(G.beta, P->rate_scale);
      D.k = G.exponent;
      D.first = (g == C.gate_begin);
      D.last = (g == C.gate_begin + C.gate_count - 1);
      D.channel = c;
      D.g = T(C.g_max);
      D.e = T(C.e_rev);
      D.leak_lo = nleak;
      D.leak_hi = nleak;
    }
    last_gated_gate = C.gate_begin + C.gate_count - 1;
  }
  tb.nleak = nleak;
  tb.leak_g_sum = T(gsum);
  tb.leak_ge_sum = T(gesum);
  return tb;
}

template <typename T>
inline DevSur<T> pack_sur(const hhb_surrogate_t* s) {
  DevSur<T> d{};
  d.kind = s->kind;
  d.w = T(s->width);
  d.inv_w = T(1.0 / s->width);
  d.k2 = T(-kLog2e / s->width);
  d.half_inv_w = T(0.5 / s->width);
  return d;
}

template <typename T>
inline PoissonTab<T> poisson_table(double lam, double amp) {
  PoissonTab<T> tb{};
  tb.amp = T(amp);
  double pk = std::exp(-lam), cdf = pk;
  int k = 0;
  for (; k < 48; ++k) {
    tb.cdf[k] = T(cdf);
    if (cdf >= 1.0 - 1.16e-10) break;
    pk *= lam / double(k + 1);
    cdf += pk;
  }
  tb.size = k < 48 ? k + 1 : 48;
  return tb;
}

inline int fwd_block(int64_t threads) {
  if (threads >= int64_t(kNumSMs) * kFwdThreads) return kFwdThreads;
  int64_t per = (threads + kNumSMs - 1) / kNumSMs;
  per = ((per + 31) / 32) * 32;
  if (per < 32) per = 32;
  if (per > kFwdThreads) per = kFwdThreads;
  return int(per);
}

inline int64_t bwd_blocks(int64_t n) { return (n + kBwdThreads - 1) / kBwdThreads; }

inline int grid_1d(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 65535LL * 16) b = 65535LL * 16;
  if (b < 1) b = 1;
  return int(b);
}

// ------------------------------------------------------------ launchers
template <typename T, int VEC, bool POIS>
int launch_forward_vec(const DevTable<T>& tb, const FwdArgs<T>& a, const PoissonTab<T>& ptab,
                       cudaStream_t st) {
  const int64_t threads = (a.n + VEC - 1) / VEC;
  const int tpb = fwd_block(threads);
  const int64_t blocks = (threads + tpb - 1) / tpb;
  if (blocks > 0x7fffffffLL) return fail(HHB_EINVAL, "too many neurons for one launch");
  switch (tb.ng) {
#define HHB_CASE(NG) \
  case NG:           \
    k_forward<T, NG, VEC, POIS><<<unsigned(blocks), tpb, 0, st>>>(tb, a, ptab); \
    break;
    HHB_CASE(0) HHB_CASE(1) HHB_CASE(2) HHB_CASE(3) HHB_CASE(4)
    HHB_CASE(5) HHB_CASE(6) HHB_CASE(7) HHB_CASE(8)
#undef HHB_CASE
    default:
      return fail(HHB_ENOTSUP, "n_gates > 8");
  }
  return cuda_check("k_forward launch");
}

template <typename T>
int launch_backward(const DevTable<T>& tb, const DevSur<T>& sur, const BwdArgs<T>& a,
                    double* d_params, cudaStream_t st) {
  const int64_t blocks = bwd_blocks(a.n);
  if (blocks > 0x7fffffffLL) return fail(HHB_EINVAL, "too many neurons for one launch");
  switch (tb.ng) {
#define HHB_CASE(NG) \
  case NG:           \
    k_backward<T, NG><<<unsigned(blocks), kBwdThreads, 0, st>>>(tb, sur, a); \
    break;
    HHB_CASE(0) HHB_CASE(1) HHB_CASE(2) HHB_CASE(3) HHB_CASE(4)
    HHB_CASE(5) HHB_CASE(6) HHB_CASE(7) HHB_CASE(8)
#undef HHB_CASE
    default:
      return fail(HHB_ENOTSUP, "n_gates > 8");
  }
  int rc = cuda_check("k_backward launch");
  if (rc) return rc;
  launch_pdl(k_reduce<T>, dim3(kSlots), dim3(256), 0, st, tb, (const double*)a.partials, int64_t(blocks), d_params);
  return cuda_check("k_reduce launch");
}

template <typename T>
int launch_ionic(const DevTable<T>& tb, int64_t n, const T* v, const T* g, int64_t g_ld, T* out,
                 cudaStream_t st) {
  const int grid = grid_1d(n, 256);
  switch (tb.ng) {
#define HHB_CASE(NG) \
  case NG:           \
    k_ionic<T, NG><<<grid, 256, 0, st>>>(tb, n, v, g, g_ld, out); \
    break;
    HHB_CASE(0) HHB_CASE(1) HHB_CASE(2) HHB_CASE(3) HHB_CASE(4)
    HHB_CASE(5) HHB_CASE(6) HHB_CASE(7) HHB_CASE(8)
#undef HHB_CASE
    default:
      return fail(HHB_ENOTSUP, "n_gates > 8");
  }
  return cuda_check("k_ionic launch");
}

// Runtime-specialised float kernels (jit.cu).  Return false when the JIT is
// unavailable or disabled; the generic kernels then run.
bool jit_forward(const hhb_params_t* P, const FwdArgs<float>& a, const PoissonTab<float>* ptab, bool vec4,
                 cudaStream_t st, int& rc);
bool jit_backward(const hhb_params_t* P, const DevSur<float>& sur, const BwdArgs<float>& a, cudaStream_t st,
                  int& rc);
// host image of the JIT hh_net kernel's NetArgs (same member order and types)
struct CortexRunArgs {
  int64_t n, steps, t0, depth;
  long long* ring;
  float* psp;
  const double* lam;
  float decay, mu, sigma, w_scale;
  int mode, rec;
  unsigned long long seed;
  int64_t nbase;
  float* v;
  float* g;
  int64_t g_ld;
  uint32_t* bits;
  int64_t words;
  const int64_t* seg;
  int64_t tiles;
  const int* tgt;
  const int* w;
  const int* delay;
  int64_t* first_bad;
  unsigned* bar;                 // grid-barrier counter (one uint32 of device scratch)
  unsigned long long* timing;   // optional [steps][blocks][4] globaltimer stamps (profiling)
  int64_t reps, ld;              // replicas per launch; per-replica stride of v / psp / ring rows
  // thalamic drive (hhb_thalamic_t; th_off == nullptr: none) -- appended in the
  // order of NetArgs (jit.cu), which mirrors this struct field for field
  const int64_t* th_off;
  const float* th_w;
  int64_t th_base, th_on, th_end;
  uint32_t th_thr;
  uint64_t th_seed;
};
bool jit_cortex_run(const hhb_params_t* P, const CortexRunArgs& a, cudaStream_t st, int& rc);
const char* jit_status();
std::string jit_source(const hhb_params_t* P);
int jit_cubin(const hhb_params_t* P, int kind, std::vector<char>& cubin, std::string& log);

template <typename T>
inline bool try_jit_fwd(const hhb_params_t* P, const FwdArgs<T>& a, const PoissonTab<T>* ptab, bool vec4,
                        cudaStream_t st, int& rc) {
  if constexpr (sizeof(T) == 4) {
    return jit_forward(P, a, ptab, vec4, st, rc);
  } else {
    return false;
  }
}
template <typename T>
inline bool try_jit_bwd(const hhb_params_t* P, const DevSur<T>& s, const BwdArgs<T>& a, cudaStream_t st,
                        int& rc) {
  if constexpr (sizeof(T) == 4) {
    return jit_backward(P, s, a, st, rc);
  } else {
    return false;
  }
}

// Flavour entry points (one definition per TU: hh_f32.cu / hh_f64.cu).
template <typename T>
struct Flavour {
  // ptab != nullptr: the current is the fused Poisson stimulus (a.seed, a.nbase)
  static int forward(const hhb_params_t* P, const FwdArgs<T>& a, const PoissonTab<T>* ptab,
                     cudaStream_t st);
  static int backward(const hhb_params_t* P, const hhb_surrogate_t* S, const BwdArgs<T>& a,
                      double* d_params, cudaStream_t st);
  static int gate_rates(const hhb_gate_t* G, double scale, int64_t n, const T* v, T* al, T* be,
                        cudaStream_t st);
  static int rate_eval(const hhb_rate_t* R, int slope, int64_t n, const T* v, T* out,
                       cudaStream_t st);
  static int gate_step(int64_t n, const T* p, const T* al, const T* be, double dt, T* out,
                       cudaStream_t st);
  static int ionic(const hhb_params_t* P, int64_t n, const T* v, const T* g, int64_t g_ld, T* out,
                   cudaStream_t st);
  static int spike_detect(int64_t n, const T* vp, const T* vn, double theta, uint8_t* out,
                          cudaStream_t st);
  static int surrogate(const hhb_surrogate_t* S, int64_t n, const T* u, T* out, cudaStream_t st);
  static int poisson(int64_t n, int64_t steps, uint64_t seed, int64_t nbase, int64_t tbase,
                     double lam, double amp, T* out, int64_t ld, cudaStream_t st);
};

// Shared definitions, included once by each flavour TU with T fixed.
#define HHB_DEFINE_FLAVOUR(T, VECW)                                                              \
  template <>                                                                                    \
  int Flavour<T>::forward(const hhb_params_t* P, const FwdArgs<T>& a, const PoissonTab<T>* ptab,  \
                          cudaStream_t st) {                                                     \
    const DevTable<T> tb = pack_table<T>(P);                                                     \
    const bool pois = ptab != nullptr;                                                           \
    const PoissonTab<T> pt = pois ? *ptab : PoissonTab<T>{};                                     \
    const bool vec_ok =                                                                          \
        (a.n % (VECW) == 0) && (!pois || (VECW) != 4 || (a.nbase & 3) == 0) &&                   \
        (pois || ((a.i_sn == 1) && (a.i_st % (VECW) == 0) &&                                     \
                  (reinterpret_cast<uintptr_t>(a.i_ext) % (sizeof(T) * (VECW)) == 0))) &&        \
        (a.v_out == nullptr ||                                                                   \
         (a.v_ld % (VECW) == 0 && reinterpret_cast<uintptr_t>(a.v_out) % (sizeof(T) * (VECW)) == 0)) && \
        (a.ckpt == nullptr ||                                                                    \
         (a.ck_ld % (VECW) == 0 && reinterpret_cast<uintptr_t>(a.ckpt) % (sizeof(T) * (VECW)) == 0)); \
    const bool wide = vec_ok && a.n >= int64_t(kNumSMs) * 32 * (VECW);                            \
    int jrc = HHB_OK;                                                                            \
    if (try_jit_fwd<T>(P, a, ptab, wide && (VECW) == 4, st, jrc)) return jrc;                    \
    if (pois)                                                                                    \
      return wide ? launch_forward_vec<T, VECW, true>(tb, a, pt, st)                             \
                  : launch_forward_vec<T, 1, true>(tb, a, pt, st);                               \
    if (wide) return launch_forward_vec<T, VECW, false>(tb, a, pt, st);                          \
    return launch_forward_vec<T, 1, false>(tb, a, pt, st);                                       \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::backward(const hhb_params_t* P, const hhb_surrogate_t* S,                      \
                           const BwdArgs<T>& a, double* d_params, cudaStream_t st) {             \
    const DevTable<T> tb = pack_table<T>(P);                                                     \
    const DevSur<T> sur = pack_sur<T>(S);                                                        \
    int jrc = HHB_OK;                                                                            \
    if (try_jit_bwd<T>(P, sur, a, st, jrc)) {                                                    \
      if (jrc) return jrc;                                                                       \
      launch_pdl(k_reduce<T>, dim3(kSlots), dim3(256), 0, st, tb, (const double*)a.partials,        \
                 int64_t(bwd_blocks(a.n)), d_params);                                                \
      return cuda_check("k_reduce launch");                                                      \
    }                                                                                            \
    return launch_backward<T>(tb, sur, a, d_params, st);                                         \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::gate_rates(const hhb_gate_t* G, double scale, int64_t n, const T* v, T* al,    \
                             T* be, cudaStream_t st) {                                           \
    hhb_params_t P{};                                                                            \
    P.n_gates = 1;                                                                               \
    P.n_channels = 1;                                                                            \
    P.c_m = 1.0;                                                                                 \
    P.dt = 1.0;                                                                                  \
    P.rate_scale = scale;                                                                        \
    P.gates[0] = *G;                                                                             \
    P.gates[0].channel = 0;                                                                      \
    P.channels[0].gate_begin = 0;                                                                \
    P.channels[0].gate_count = 1;                                                                \
    k_rates<T><<<grid_1d(n, 256), 256, 0, st>>>(pack_table<T>(&P), n, v, al, be);               \
    return cuda_check("k_rates launch");                                                         \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::rate_eval(const hhb_rate_t* R, int slope, int64_t n, const T* v, T* out,       \
                            cudaStream_t st) {                                                   \
    k_rate_eval<T><<<grid_1d(n, 256), 256, 0, st>>>(pack_rate<T>(*R, 1.0), slope, n, v, out);   \
    return cuda_check("k_rate_eval launch");                                                     \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::gate_step(int64_t n, const T* p, const T* al, const T* be, double dt, T* out,  \
                            cudaStream_t st) {                                                   \
    k_gate_step<T><<<grid_1d(n, 256), 256, 0, st>>>(n, p, al, be, T(dt), out);                  \
    return cuda_check("k_gate_step launch");                                                     \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::ionic(const hhb_params_t* P, int64_t n, const T* v, const T* g, int64_t g_ld,  \
                        T* out, cudaStream_t st) {                                               \
    return launch_ionic<T>(pack_table<T>(P), n, v, g, g_ld, out, st);                            \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::spike_detect(int64_t n, const T* vp, const T* vn, double theta, uint8_t* out,  \
                               cudaStream_t st) {                                                \
    k_spike_detect<T><<<grid_1d(n, 256), 256, 0, st>>>(n, vp, vn, T(theta), out);               \
    return cuda_check("k_spike_detect launch");                                                  \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::surrogate(const hhb_surrogate_t* S, int64_t n, const T* u, T* out,             \
                            cudaStream_t st) {                                                   \
    k_surrogate<T><<<grid_1d(n, 256), 256, 0, st>>>(pack_sur<T>(S), n, u, out);                 \
    return cuda_check("k_surrogate launch");                                                     \
  }                                                                                              \
  template <>                                                                                    \
  int Flavour<T>::poisson(int64_t n, int64_t steps, uint64_t seed, int64_t nbase, int64_t tbase, \
                          double lam, double amp, T* out, int64_t ld, cudaStream_t st) {         \
    if (n <= 0 || steps <= 0) return HHB_OK;                                                     \
    const int64_t bx = ((n + 3) / 4 + 255) / 256;                                                \
    int64_t by = (int64_t(kNumSMs) * 8 + bx - 1) / bx;                                           \
    by = by < 1 ? 1 : (by > steps ? steps : (by > 65535 ? 65535 : by));                          \
    const dim3 grid{unsigned(bx), unsigned(by), 1u};                                             \
    k_poisson<T><<<grid, 256, 0, st>>>(n, steps, seed, nbase, tbase, poisson_table<T>(lam, amp),  \
                                       out, ld);                                                 \
    return cuda_check("k_poisson launch");                                                       \
  }

}  // namespace hhb
