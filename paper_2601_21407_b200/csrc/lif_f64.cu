// lif_f64.cu -- LIF kernels (lif.cuh), both flavours, and their C ABI.  Built
// with -fmad=false: the float64 flavour then rounds like NumPy.
#include "lif.cuh"

using namespace hhb;

namespace {
template <typename T>
int lif_fwd(int64_t n, int64_t steps, double tau, double dt, double theta, double v_reset, const void* v_in,
            const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, uint8_t* spk, void* v_fin,
            cudaStream_t st) {
  const T k = T(dt / tau);
  lif::k_lif_forward<T><<<grid_1d(n, 256), 256, 0, st>>>(n, steps, k, T(theta), T(v_reset), (const T*)v_in,
                                                         (const T*)i_ext, i_st, i_sn, (T*)v_out, spk, (T*)v_fin);
  return cuda_check("k_lif_forward launch");
}
template <typename T>
int lif_bwd(int64_t n, double tau, double dt, double theta, double v_reset, const hhb_surrogate_t* S, const void* v,
            const void* i_ext, int64_t i_sn, const void* g_v, const void* g_s, void* d_v, void* d_i, int64_t* bad,
            cudaStream_t st) {
  const T k = T(dt / tau);
  lif::k_lif_backward<T><<<grid_1d(n, 256), 256, 0, st>>>(n, k, T(theta), T(v_reset), pack_sur<T>(S), (const T*)v,
                                                          (const T*)i_ext, i_sn, (const T*)g_v, (const T*)g_s,
                                                          (T*)d_v, (T*)d_i, reinterpret_cast<long long*>(bad));
  return cuda_check("k_lif_backward launch");
}
// causal FIR along the leading (time) axis in scipy.signal.lfilter's direct
// form II transposed order (learn.py:52-55, a = [1]): y = b0 x + z0,
// z_i = z_{i+1} + b_{i+1} x, z_{L-2} = b_{L-1} x; one thread per column, the
// taps in shared memory, the delay line in a per-thread local array
constexpr int kMaxTaps = 256;
template <typename T>
__global__ void k_psp_filter(int64_t steps, int64_t cols, int ntaps, const double* taps, const T* x, T* y) {
  __shared__ T b[kMaxTaps];
  for (int k = threadIdx.x; k < ntaps; k += blockDim.x) b[k] = T(taps[k]);
  __syncthreads();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  T z[kMaxTaps];
  for (int k = 0; k < ntaps - 1; ++k) z[k] = T(0);
  for (int64_t t = 0; t < steps; ++t) {
    const T xv = x[t * cols + c];
    y[t * cols + c] = ntaps > 1 ? add_(mul_(b[0], xv), z[0]) : mul_(b[0], xv);
    for (int k = 0; k + 2 < ntaps; ++k) z[k] = add_(z[k + 1], mul_(b[k + 1], xv));
    if (ntaps > 1) z[ntaps - 2] = mul_(b[ntaps - 1], xv);
  }
}
}  // namespace

extern "C" {

int hhb_psp_filter(int32_t dtype, int64_t steps, int64_t cols, int32_t ntaps, const double* taps_dev,
                   const void* x, void* y, void* stream) {
  if (ntaps < 1 || ntaps > kMaxTaps) return fail(HHB_EINVAL, "psp_filter: 1..256 taps");
  if (steps < 0 || cols < 0) return fail(HHB_EINVAL, "psp_filter: negative size");
  if (steps == 0 || cols == 0) return HHB_OK;
  if (!taps_dev || !x || !y) return fail(HHB_EINVAL, "psp_filter: NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = unsigned((cols + 127) / 128);
  if (dtype == HHB_F64) k_psp_filter<double><<<grid, 128, 0, st>>>(steps, cols, ntaps, taps_dev, (const double*)x,
                                                                   (double*)y);
  else if (dtype == HHB_F32) k_psp_filter<float><<<grid, 128, 0, st>>>(steps, cols, ntaps, taps_dev, (const float*)x,
                                                                       (float*)y);
  else return fail(HHB_EINVAL, "dtype");
  return cuda_check("k_psp_filter launch");
}


int hhb_lif_forward(int32_t dtype, int64_t n, int64_t n_steps, double tau, double dt, double v_theta,
                    double v_reset, const void* v_in, const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out,
                    uint8_t* spk_out, void* v_fin, void* stream) {
  if (!(tau > 0) || !(dt > 0) || !(v_theta > v_reset)) return fail(HHB_EINVAL, "bad LIF parameters");
  if (n < 0 || n_steps < 0) return fail(HHB_EINVAL, "n and n_steps must be >= 0");
  if (n == 0) return HHB_OK;
  if (!v_in || !v_fin || (n_steps > 0 && !i_ext)) return fail(HHB_EINVAL, "v_in, v_fin, i_ext required");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HHB_F32)
    return lif_fwd<float>(n, n_steps, tau, dt, v_theta, v_reset, v_in, i_ext, i_st, i_sn, v_out, spk_out, v_fin, st);
  if (dtype == HHB_F64)
    return lif_fwd<double>(n, n_steps, tau, dt, v_theta, v_reset, v_in, i_ext, i_st, i_sn, v_out, spk_out, v_fin,
                           st);
  return fail(HHB_EINVAL, "dtype");
}

int hhb_lif_backward(int32_t dtype, int64_t n, double tau, double dt, double v_theta, double v_reset,
                     const hhb_surrogate_t* surrogate, const void* v, const void* i_ext, int64_t i_sn,
                     const void* g_v_out, const void* g_spike, void* d_v_in, void* d_i, int64_t* bad,
                     void* stream) {
  if (!(tau > 0) || !(dt > 0)) return fail(HHB_EINVAL, "bad LIF parameters");
  if (!surrogate || !(surrogate->width > 0)) return fail(HHB_EINVAL, "bad surrogate");
  if (n <= 0) return HHB_OK;
  if (!v || !i_ext || !g_v_out || !d_v_in || !d_i || !bad) return fail(HHB_EINVAL, "missing pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HHB_F32)
    return lif_bwd<float>(n, tau, dt, v_theta, v_reset, surrogate, v, i_ext, i_sn, g_v_out, g_spike, d_v_in, d_i,
                          bad, st);
  if (dtype == HHB_F64)
    return lif_bwd<double>(n, tau, dt, v_theta, v_reset, surrogate, v, i_ext, i_sn, g_v_out, g_spike, d_v_in, d_i,
                           bad, st);
  return fail(HHB_EINVAL, "dtype");
}

}  // extern "C"
