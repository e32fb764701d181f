// capi.cu -- the extern "C" boundary declared in include/hhb200.h.
// Validates arguments, selects the arithmetic flavour and forwards to the
// launchers.  Nothing here allocates device memory or synchronises.
#include <cstring>
#include <string>

#include "hh_host.cuh"

namespace hhb {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

template <typename T>
struct FlavourOf;
template <>
struct FlavourOf<float> {
  using F = Flavour<float>;
};
template <>
struct FlavourOf<double> {
  using F = Flavour<double>;
};

static int check_dtype(int32_t dtype) {
  if (dtype != HHB_F32 && dtype != HHB_F64) return fail(HHB_EINVAL, "dtype must be HHB_F32 or HHB_F64");
  return HHB_OK;
}

template <typename T>
static int forward_t(const hhb_params_t* P, int64_t n, int64_t steps, const void* v_in,
                     const void* g_in, int64_t g_ld, void* v_fin, void* g_fin, const void* i_ext,
                     int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld, uint32_t* spk,
                     int64_t spk_ld, void* ckpt, int64_t ck_every, int64_t ck_ld,
                     int64_t step_base, int64_t* first_bad, cudaStream_t st, void* spk_val = nullptr,
                     int64_t spkv_ld = 0, const int64_t* step_base_dev = nullptr, double* sq_part = nullptr,
                     void* spk_bf = nullptr, int64_t spkb_ld = 0) {
  FwdArgs<T> a{};
  a.spk_bf = static_cast<uint16_t*>(spk_bf);
  a.spkb_ld = spkb_ld;
  a.sq_part = sq_part;
  a.step_dev = reinterpret_cast<const long long*>(step_base_dev);
  a.spk_val = static_cast<T*>(spk_val);
  a.spkv_ld = spkv_ld;
  a.n = n;
  a.steps = steps;
  a.v_in = static_cast<const T*>(v_in);
  a.g_in = static_cast<const T*>(g_in);
  a.g_ld = g_ld;
  a.v_fin = static_cast<T*>(v_fin);
  a.g_fin = static_cast<T*>(g_fin);
  a.i_ext = static_cast<const T*>(i_ext);
  a.i_st = i_st;
  a.i_sn = i_sn;
  a.v_out = static_cast<T*>(v_out);
  a.v_ld = v_ld;
  a.spk = spk;
  a.spk_ld = spk_ld;
  a.ckpt = static_cast<T*>(ckpt);
  a.ck_every = ck_every;
  a.ck_ld = ck_ld;
  a.step_base = step_base;
  a.first_bad = reinterpret_cast<long long*>(first_bad);
  return Flavour<T>::forward(P, a, nullptr, st);
}

template <typename T>
static int forward_poisson_t(const hhb_params_t* P, int64_t n, int64_t steps, const void* v_in,
                             const void* g_in, int64_t g_ld, void* v_fin, void* g_fin, uint64_t seed,
                             int64_t nbase, double lam, double amp, void* v_out, int64_t v_ld,
                             uint32_t* spk, int64_t spk_ld, void* ckpt, int64_t ck_every,
                             int64_t ck_ld, int64_t step_base, int64_t* first_bad, cudaStream_t st) {
  FwdArgs<T> a{};
  a.n = n;
  a.steps = steps;
  a.v_in = static_cast<const T*>(v_in);
  a.g_in = static_cast<const T*>(g_in);
  a.g_ld = g_ld;
  a.v_fin = static_cast<T*>(v_fin);
  a.g_fin = static_cast<T*>(g_fin);
  a.v_out = static_cast<T*>(v_out);
  a.v_ld = v_ld;
  a.spk = spk;
  a.spk_ld = spk_ld;
  a.ckpt = static_cast<T*>(ckpt);
  a.ck_every = ck_every;
  a.ck_ld = ck_ld;
  a.step_base = step_base;
  a.first_bad = reinterpret_cast<long long*>(first_bad);
  a.seed = seed;
  a.nbase = nbase;
  const PoissonTab<T> tab = poisson_table<T>(lam, amp);
  return Flavour<T>::forward(P, a, &tab, st);
}

template <typename T>
static int backward_t(const hhb_params_t* P, const hhb_surrogate_t* S, int64_t n, int64_t steps,
                      const void* i_ext, int64_t i_st, int64_t i_sn, const void* ckpt,
                      int64_t ck_every, int64_t ck_ld, void* seg, const void* seed_v,
                      int64_t sv_ld, const void* seed_s, int64_t ss_ld, void* adj_v, void* adj_g,
                      int64_t ag_ld, void* d_i, int64_t di_ld, double* d_params, double* partials,
                      int64_t step_base, int64_t* first_bad, cudaStream_t st, void* di_hi = nullptr,
                      void* di_lo = nullptr, int64_t dh_ld = 0, float* di_sum = nullptr, int64_t dh_grp = 0,
                      int64_t dh_pitch = 0, const float* sv_scale = nullptr) {
  BwdArgs<T> a{};
  a.sv_scale = sv_scale;
  a.dh_grp = dh_grp;
  a.dh_pitch = dh_pitch;
  a.di_hi = static_cast<uint16_t*>(di_hi);
  a.di_lo = static_cast<uint16_t*>(di_lo);
  a.dh_ld = dh_ld;
  a.di_sum = di_sum;
  a.n = n;
  a.steps = steps;
  a.i_ext = static_cast<const T*>(i_ext);
  a.i_st = i_st;
  a.i_sn = i_sn;
  a.ckpt = static_cast<const T*>(ckpt);
  a.ck_every = ck_every;
  a.ck_ld = ck_ld;
  a.seg = static_cast<T*>(seg);
  a.seed_v = static_cast<const T*>(seed_v);
  a.sv_ld = sv_ld;
  a.seed_s = static_cast<const T*>(seed_s);
  a.ss_ld = ss_ld;
  a.adj_v = static_cast<T*>(adj_v);
  a.adj_g = static_cast<T*>(adj_g);
  a.ag_ld = ag_ld;
  a.d_i = static_cast<T*>(d_i);
  a.di_ld = di_ld;
  a.partials = partials;
  a.step_base = step_base;
  a.first_bad = reinterpret_cast<long long*>(first_bad);
  return Flavour<T>::backward(P, S, a, d_params, st);
}

}  // namespace hhb

using namespace hhb;

// out = x * (scale[0] * c): the autograd seed of a reduction loss (learn.py:86-88
// seed 2 diff / n times the incoming gradient) in one vectorised pass, the scale
// read on the device (no host sync)
static __global__ void k_scale_f32(int64_t n4, const float4* x, const float* scale, float c, float4* out) {
  const float k = scale[0] * c;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    float4 v = x[i];
    v.x *= k;
    v.y *= k;
    v.z *= k;
    v.w *= k;
    out[i] = v;
  }
}
static __global__ void k_scale_tail(int64_t n, const float* x, const float* scale, float c, float* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[i] * (scale[0] * c);
}

// independent 8-wide chains so the probe measures pipe throughput, not latency
static __global__ void __launch_bounds__(256) k_pipe_probe(int which, int64_t iters, float* sink) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = 0.001f * float(threadIdx.x + j);
  if (which == 0) {
    for (int64_t k = 0; k < iters; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = ex2_(-x[j]);
    }
  } else if (which == 1) {
    for (int64_t k = 0; k < iters; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma_(x[j], 0.999f, 0.0001f);
    }
  } else {
    for (int64_t k = 0; k < iters; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = rcp_(x[j] + 1.0f);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678f) sink[0] = s;  // keep the chains alive
}

#define ST(s) static_cast<cudaStream_t>(s)

extern "C" {

int hhb_abi_version(void) { return HHB_ABI_VERSION; }

const char* hhb_last_error(void) { return g_last_error.c_str(); }

int hhb_check_params(const hhb_params_t* params) { return check_params(params); }

int hhb_forward(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld,
                uint32_t* spk_out, int64_t spk_ld, void* ckpt, int64_t ckpt_every,
                int64_t ckpt_ld, int64_t step_base, int64_t* first_bad, void* stream) {
  return hhb_forward_ex(params, dtype, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, i_ext, i_st, i_sn, v_out,
                        v_ld, spk_out, spk_ld, nullptr, 0, ckpt, ckpt_every, ckpt_ld, step_base, first_bad,
                        nullptr, nullptr, stream);
}

int hhb_forward_ex2(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                   const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                   const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld,
                   uint32_t* spk_out, int64_t spk_ld, void* spk_val, int64_t spk_val_ld, void* ckpt,
                   int64_t ckpt_every, int64_t ckpt_ld, int64_t step_base, int64_t* first_bad,
                   const int64_t* step_base_dev, double* sq_partials, void* spk_bf16, int64_t spk_bf16_ld,
                    void* stream) {
  if (spk_bf16 && spk_bf16_ld < n) return fail(HHB_EINVAL, "spk_bf16_ld < n");
  if (spk_val && spk_val_ld < n) return fail(HHB_EINVAL, "spk_val_ld < n");
  int rc = check_params(params);
  if (rc) return rc;
  if ((rc = check_dtype(dtype))) return rc;
  if (n < 0 || n_steps < 0) return fail(HHB_EINVAL, "n and n_steps must be >= 0");
  if (n == 0) return HHB_OK;
  if (!v_in || !v_fin || first_bad == nullptr) return fail(HHB_EINVAL, "v_in, v_fin, first_bad required");
  if (params->n_gates > 0 && (!g_in || !g_fin || g_ld < n)) return fail(HHB_EINVAL, "gate state required");
  if (n_steps > 0 && i_ext == nullptr) return fail(HHB_EINVAL, "i_ext required");
  if (v_out && v_ld < n) return fail(HHB_EINVAL, "v_ld < n");
  if (spk_out && spk_ld < (n + 31) / 32) return fail(HHB_EINVAL, "spk_ld < ceil(n/32)");
  if (ckpt && (ckpt_every < 1 || ckpt_ld < n)) return fail(HHB_EINVAL, "bad checkpoint layout");
  if (dtype == HHB_F32)
    return forward_t<float>(params, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, i_ext, i_st, i_sn,
                            v_out, v_ld, spk_out, spk_ld, ckpt, ckpt_every, ckpt_ld, step_base,
                            first_bad, ST(stream), spk_val, spk_val_ld, step_base_dev, sq_partials, spk_bf16,
                            spk_bf16_ld);
  return forward_t<double>(params, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, i_ext, i_st, i_sn,
                           v_out, v_ld, spk_out, spk_ld, ckpt, ckpt_every, ckpt_ld, step_base,
                           first_bad, ST(stream), spk_val, spk_val_ld, step_base_dev, sq_partials, spk_bf16,
                            spk_bf16_ld);
}

int hhb_forward_ex(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                   const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                   const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld,
                   uint32_t* spk_out, int64_t spk_ld, void* spk_val, int64_t spk_val_ld, void* ckpt,
                   int64_t ckpt_every, int64_t ckpt_ld, int64_t step_base, int64_t* first_bad,
                   const int64_t* step_base_dev, double* sq_partials, void* stream) {
  return hhb_forward_ex2(params, dtype, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, i_ext, i_st, i_sn, v_out, v_ld,
                         spk_out, spk_ld, spk_val, spk_val_ld, ckpt, ckpt_every, ckpt_ld, step_base, first_bad,
                         step_base_dev, sq_partials, nullptr, 0, stream);
}

int64_t hhb_forward_partials(int64_t n) { return (n < 1 ? 1 : (n + 31) / 32) + 1; }

int hhb_forward_poisson(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                        const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                        uint64_t seed, int64_t neuron_base, double lam, double amp, void* v_out,
                        int64_t v_ld, uint32_t* spk_out, int64_t spk_ld, void* ckpt, int64_t ckpt_every,
                        int64_t ckpt_ld, int64_t step_base, int64_t* first_bad, void* stream) {
  int rc = check_params(params);
  if (rc) return rc;
  if ((rc = check_dtype(dtype))) return rc;
  if (n < 0 || n_steps < 0 || !(lam >= 0)) return fail(HHB_EINVAL, "bad n, n_steps or lam");
  if (n == 0) return HHB_OK;
  if (!v_in || !v_fin || first_bad == nullptr) return fail(HHB_EINVAL, "v_in, v_fin, first_bad required");
  if (params->n_gates > 0 && (!g_in || !g_fin || g_ld < n)) return fail(HHB_EINVAL, "gate state required");
  if (v_out && v_ld < n) return fail(HHB_EINVAL, "v_ld < n");
  if (spk_out && spk_ld < (n + 31) / 32) return fail(HHB_EINVAL, "spk_ld < ceil(n/32)");
  if (ckpt && (ckpt_every < 1 || ckpt_ld < n)) return fail(HHB_EINVAL, "bad checkpoint layout");
  if (dtype == HHB_F32)
    return forward_poisson_t<float>(params, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, seed, neuron_base,
                                    lam, amp, v_out, v_ld, spk_out, spk_ld, ckpt, ckpt_every, ckpt_ld,
                                    step_base, first_bad, ST(stream));
  return forward_poisson_t<double>(params, n, n_steps, v_in, g_in, g_ld, v_fin, g_fin, seed, neuron_base,
                                   lam, amp, v_out, v_ld, spk_out, spk_ld, ckpt, ckpt_every, ckpt_ld,
                                   step_base, first_bad, ST(stream));
}

int64_t hhb_backward_partials(int64_t n, int32_t dtype) {
  (void)dtype;
  return bwd_blocks(n < 1 ? 1 : n) * kSlots;
}

int hhb_backward(const hhb_params_t* params, const hhb_surrogate_t* surrogate, int32_t dtype,
                 int64_t n, int64_t n_steps, const void* i_ext, int64_t i_st, int64_t i_sn,
                 const void* ckpt, int64_t ckpt_every, int64_t ckpt_ld, void* seg_buf,
                 const void* seed_v, int64_t seed_v_ld, const void* seed_spk, int64_t seed_spk_ld,
                 void* adj_v, void* adj_g, int64_t adj_g_ld, void* d_i, int64_t d_i_ld,
                 double* d_params, double* partials, int64_t step_base, int64_t* first_bad,
                 void* stream) {
  return hhb_backward_ex(params, surrogate, dtype, n, n_steps, i_ext, i_st, i_sn, ckpt, ckpt_every, ckpt_ld,
                         seg_buf, seed_v, seed_v_ld, seed_spk, seed_spk_ld, adj_v, adj_g, adj_g_ld, d_i, d_i_ld,
                         d_params, partials, step_base, first_bad, nullptr, nullptr, 0, 0, 0, nullptr, nullptr,
                         stream);
}

int hhb_backward_ex(const hhb_params_t* params, const hhb_surrogate_t* surrogate, int32_t dtype,
                    int64_t n, int64_t n_steps, const void* i_ext, int64_t i_st, int64_t i_sn,
                    const void* ckpt, int64_t ckpt_every, int64_t ckpt_ld, void* seg_buf,
                    const void* seed_v, int64_t seed_v_ld, const void* seed_spk, int64_t seed_spk_ld,
                    void* adj_v, void* adj_g, int64_t adj_g_ld, void* d_i, int64_t d_i_ld,
                    double* d_params, double* partials, int64_t step_base, int64_t* first_bad,
                    void* d_i_hi, void* d_i_lo, int64_t d_split_ld, int64_t d_split_group,
                    int64_t d_split_pitch, float* d_i_sum, const float* seed_v_scale, void* stream) {
  if (d_split_group < 0 || (d_split_group > 0 && d_split_pitch < d_split_group))
    return fail(HHB_EINVAL, "d_split_pitch < d_split_group");
  if ((d_i_hi || d_i_lo || d_i_sum) && dtype != HHB_F32)
    return fail(HHB_EINVAL, "split / summed dI outputs are float-only");
  const int64_t split_cols = d_split_group > 0 ? (n + d_split_group - 1) / d_split_group * d_split_pitch : n;
  if ((d_i_hi != nullptr) != (d_i_lo != nullptr) || (d_i_hi && d_split_ld < split_cols))
    return fail(HHB_EINVAL, "d_i_hi and d_i_lo go together, with d_split_ld >= n");
  int rc = check_params(params);
  if (rc) return rc;
  if ((rc = check_dtype(dtype))) return rc;
  if (!surrogate || !(surrogate->width > 0) || surrogate->kind < 0 || surrogate->kind > 1)
    return fail(HHB_EINVAL, "bad surrogate");
  if (n < 0 || n_steps < 0) return fail(HHB_EINVAL, "n and n_steps must be >= 0");
  if (n == 0 || n_steps == 0) return HHB_OK;
  if (!i_ext || !ckpt || !adj_v || !d_params || !partials || !first_bad)
    return fail(HHB_EINVAL, "missing required pointer");
  if (ckpt_every < 1 || ckpt_ld < n) return fail(HHB_EINVAL, "bad checkpoint layout");
  if (ckpt_every > 1 && !seg_buf) return fail(HHB_EINVAL, "seg_buf required when ckpt_every > 1");
  if (params->n_gates > 0 && (!adj_g || adj_g_ld < n)) return fail(HHB_EINVAL, "adj_g required");
  if (dtype == HHB_F32)
    return backward_t<float>(params, surrogate, n, n_steps, i_ext, i_st, i_sn, ckpt, ckpt_every,
                             ckpt_ld, seg_buf, seed_v, seed_v_ld, seed_spk, seed_spk_ld, adj_v,
                             adj_g, adj_g_ld, d_i, d_i_ld, d_params, partials, step_base,
                             first_bad, ST(stream), d_i_hi, d_i_lo, d_split_ld, d_i_sum, d_split_group,
                             d_split_pitch, seed_v_scale);
  return backward_t<double>(params, surrogate, n, n_steps, i_ext, i_st, i_sn, ckpt, ckpt_every,
                            ckpt_ld, seg_buf, seed_v, seed_v_ld, seed_spk, seed_spk_ld, adj_v,
                            adj_g, adj_g_ld, d_i, d_i_ld, d_params, partials, step_base, first_bad,
                            ST(stream), nullptr, nullptr, 0, nullptr, 0, 0, seed_v_scale);
}

int hhb_gate_rates(const hhb_gate_t* gate, double rate_scale, int32_t dtype, int64_t n,
                   const void* v, void* alpha, void* beta, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!gate) return fail(HHB_EINVAL, "gate is NULL");
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::gate_rates(gate, rate_scale, n, (const float*)v, (float*)alpha,
                                      (float*)beta, ST(stream));
  return Flavour<double>::gate_rates(gate, rate_scale, n, (const double*)v, (double*)alpha,
                                     (double*)beta, ST(stream));
}

int hhb_rate_eval(const hhb_rate_t* rate, int32_t with_slope, int32_t dtype, int64_t n,
                  const void* v, void* out, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!rate || rate->kind < 0 || rate->kind > 2 || rate->b == 0.0) return fail(HHB_EINVAL, "bad rate");
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::rate_eval(rate, with_slope, n, (const float*)v, (float*)out, ST(stream));
  return Flavour<double>::rate_eval(rate, with_slope, n, (const double*)v, (double*)out, ST(stream));
}

int hhb_gate_step(int32_t dtype, int64_t n, const void* p, const void* alpha, const void* beta,
                  double dt, void* out, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::gate_step(n, (const float*)p, (const float*)alpha, (const float*)beta, dt,
                                     (float*)out, ST(stream));
  return Flavour<double>::gate_step(n, (const double*)p, (const double*)alpha, (const double*)beta,
                                    dt, (double*)out, ST(stream));
}

int hhb_ionic_current(const hhb_params_t* params, int32_t dtype, int64_t n, const void* v,
                      const void* g, int64_t g_ld, void* out, void* stream) {
  int rc = check_params(params);
  if (rc) return rc;
  if ((rc = check_dtype(dtype))) return rc;
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::ionic(params, n, (const float*)v, (const float*)g, g_ld, (float*)out,
                                 ST(stream));
  return Flavour<double>::ionic(params, n, (const double*)v, (const double*)g, g_ld, (double*)out,
                                ST(stream));
}

int hhb_spike_detect(int32_t dtype, int64_t n, const void* v_prev, const void* v_new, double theta,
                     uint8_t* out, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::spike_detect(n, (const float*)v_prev, (const float*)v_new, theta, out,
                                        ST(stream));
  return Flavour<double>::spike_detect(n, (const double*)v_prev, (const double*)v_new, theta, out,
                                       ST(stream));
}

int hhb_surrogate_grad(const hhb_surrogate_t* surrogate, int32_t dtype, int64_t n, const void* u,
                       void* out, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!surrogate || !(surrogate->width > 0)) return fail(HHB_EINVAL, "bad surrogate");
  if (n <= 0) return HHB_OK;
  if (dtype == HHB_F32)
    return Flavour<float>::surrogate(surrogate, n, (const float*)u, (float*)out, ST(stream));
  return Flavour<double>::surrogate(surrogate, n, (const double*)u, (double*)out, ST(stream));
}

int hhb_unpack_spikes(const uint32_t* bits, int64_t words_ld, int64_t n_steps, int64_t n,
                      uint8_t* out, int64_t out_ld, void* stream) {
  if (n <= 0 || n_steps <= 0) return HHB_OK;
  if (!bits || !out || words_ld < (n + 31) / 32 || out_ld < n) return fail(HHB_EINVAL, "bad unpack args");
  const dim3 grid{unsigned((n + 255) / 256), unsigned(n_steps < 65535 ? n_steps : 65535), 1u};
  k_unpack<uint8_t><<<grid, 256, 0, ST(stream)>>>(bits, words_ld, n_steps, n, out, out_ld);
  return cuda_check("k_unpack launch");
}

int hhb_unpack_spikes_f32(const uint32_t* bits, int64_t words_ld, int64_t n_steps, int64_t n, float* out,
                          int64_t out_ld, void* stream) {
  if (n <= 0 || n_steps <= 0) return HHB_OK;
  if (!bits || !out || words_ld < (n + 31) / 32 || out_ld < n) return fail(HHB_EINVAL, "bad unpack args");
  const dim3 grid{unsigned((n + 255) / 256), unsigned(n_steps < 65535 ? n_steps : 65535), 1u};
  k_unpack<float><<<grid, 256, 0, ST(stream)>>>(bits, words_ld, n_steps, n, out, out_ld);
  return cuda_check("k_unpack launch");
}

int hhb_poisson_current(int32_t dtype, int64_t n, int64_t n_steps, uint64_t seed,
                        int64_t neuron_base, int64_t step_base, double lam, double amp, void* out,
                        int64_t ld, void* stream) {
  int rc = check_dtype(dtype);
  if (rc) return rc;
  if (!(lam >= 0) || ld < n || !out) return fail(HHB_EINVAL, "bad poisson args");
  if (dtype == HHB_F32)
    return Flavour<float>::poisson(n, n_steps, seed, neuron_base, step_base, lam, amp, (float*)out,
                                   ld, ST(stream));
  return Flavour<double>::poisson(n, n_steps, seed, neuron_base, step_base, lam, amp, (double*)out,
                                  ld, ST(stream));
}

int hhb_scale_f32(int64_t n, const float* x, const float* scale, double c, float* out, void* stream) {
  if (n <= 0) return HHB_OK;
  if (!x || !scale || !out) return fail(HHB_EINVAL, "hhb_scale_f32: NULL pointer");
  cudaStream_t st = ST(stream);
  int64_t done = 0;
  if (reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0) {
    const int64_t n4 = n / 4;
    if (n4 > 0)
      k_scale_f32<<<grid_1d(n4, 256), 256, 0, st>>>(n4, reinterpret_cast<const float4*>(x), scale, float(c),
                                                    reinterpret_cast<float4*>(out));
    done = n4 * 4;
  }
  if (done < n) k_scale_tail<<<grid_1d(n - done, 256), 256, 0, st>>>(n - done, x + done, scale, float(c), out + done);
  return cuda_check("k_scale launch");
}

const char* hhb_jit_status(void) { return jit_status(); }

int64_t hhb_jit_cubin(const hhb_params_t* params, int32_t kind, void* buf, int64_t cap) {
  if (check_params(params)) return -1;
  if ((kind > 2 && kind < 16) || kind > 16 + 255 || kind < -128) {
    fail(HHB_EINVAL, "jit_cubin: kind 0..2, 16 + BF flags or -1 - FF flags");
    return -1;
  }
  std::vector<char> cubin;
  std::string log;
  if (jit_cubin(params, kind, cubin, log) != HHB_OK) {
    fail(HHB_ECUDA, "nvrtc: " + log.substr(0, 4000));
    return -1;
  }
  if (buf && cap >= int64_t(cubin.size())) memcpy(buf, cubin.data(), cubin.size());
  return int64_t(cubin.size());
}

int64_t hhb_jit_source(const hhb_params_t* params, char* buf, int64_t cap) {
  if (check_params(params)) return -1;
  const std::string src = jit_source(params);
  if (buf && cap > 0) {
    const int64_t n = int64_t(src.size()) < cap - 1 ? int64_t(src.size()) : cap - 1;
    memcpy(buf, src.data(), size_t(n));
    buf[n] = '\0';
  }
  return int64_t(src.size()) + 1;
}

int hhb_pipe_probe(int32_t which, int64_t iters, float* sink, int64_t* ops, void* stream) {
  if (which < 0 || which > 2 || iters < 1 || !sink || !ops) return fail(HHB_EINVAL, "bad probe args");
  const int blocks = kNumSMs * 8, threads = 256;
  k_pipe_probe<<<blocks, threads, 0, ST(stream)>>>(which, iters, sink);
  *ops = int64_t(blocks) * threads * iters * 8;
  return cuda_check("k_pipe_probe launch");
}

}  // extern "C"
