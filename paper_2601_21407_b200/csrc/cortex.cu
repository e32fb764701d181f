// cortex.cu -- per-step input and spike delivery of the recurrent HH network
// (BASELINE config 5; reference cortex.py:225-310).
//
//   k_cortex_input   ring drain + exponential PSP + compound-Poisson background
//                    (host-supplied sample, or Philox on the device)
//   k_spike_deliver  one block per 32-source bitmap word: every set bit walks
//                    that source's synapse row (targets local to this rank) and
//                    adds its fixed-point weight into ring[(t + d) % D][target]
//
// The ring holds int64 fixed-point currents (weight quantum 2^-24 uA): integer
// atomics commute, so delivery is deterministic for any arrival order and any
// sharding of the population (SURVEY §8 e3 bit-exactness requirement).
#include "hh_host.cuh"

namespace hhb {
namespace cortex {

template <typename T>
__global__ void k_cortex_input(int64_t n, int64_t t, int64_t depth, long long* ring, T* psp, T decay, int mode,
                               const T* bg, const double* lam, T mu, T sigma, uint64_t seed, int64_t nbase,
                               const T* extra, T* cur, T w_scale) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long* slot = ring + (t % depth) * n + i;
  const long long arr = *slot;
  *slot = 0;
  // reference order: psp *= decay; psp += arrived; psp += background (cortex.py:287-297)
  T x = psp[i] * decay;
  x = x + T(double(arr)) * w_scale;
  if (mode == 1) {
    x = x + bg[i];
  } else if (mode == 2) {
    // compound Poisson N*mu + sigma*sqrt(N)*z, N ~ Poisson(lam), z ~ N(0,1) (cortex.py:225-232);
    // Philox-4x32-10 keyed by (seed, global neuron, step): identical on every rank layout
    const uint4 r = Philox::run(make_uint4(uint32_t(i + nbase), uint32_t(uint64_t(i + nbase) >> 32), uint32_t(t),
                                           uint32_t(uint64_t(t) >> 32)),
                                make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
    const double L = lam[i];
    const double u = (double(r.x) + 0.5) * 2.3283064365386963e-10;
    double p = exp(-L), c = p;
    int k = 0;
    while (u > c && k < 64) {
      ++k;
      p *= L / k;
      c += p;
    }
    double add = double(k) * double(mu);
    if (sigma > T(0) && k > 0) {
      const double u1 = (double(r.y) + 0.5) * 2.3283064365386963e-10;
      const double u2 = (double(r.z) + 0.5) * 2.3283064365386963e-10;
      const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
      add += double(sigma) * sqrt(double(k)) * z;
    }
    x = x + T(add);
  }
  psp[i] = x;
  cur[i] = extra ? x + extra[i] : x;
}

__global__ void __launch_bounds__(128) k_spike_deliver(int64_t words, const uint32_t* bits, const int64_t* off,
                                                       const int32_t* tgt, const int32_t* w, const int32_t* delay,
                                                       int64_t t, int64_t depth, int64_t n, long long* ring) {
  const int64_t b = blockIdx.x;
  if (b >= words) return;
  uint32_t word = bits[b];
  while (word) {
    const int bit = __ffs(int(word)) - 1;
    word &= word - 1;
    const int64_t s = b * 32 + bit;
    const int64_t lo = off[s], hi = off[s + 1];
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
      const int64_t slot = (t + delay[j]) % depth;
      atomicAdd(reinterpret_cast<unsigned long long*>(ring + slot * n + tgt[j]),
                static_cast<unsigned long long>(static_cast<long long>(w[j])));
    }
  }
}

}  // namespace cortex
}  // namespace hhb

using namespace hhb;

extern "C" {

int hhb_cortex_input(int32_t dtype, int64_t n, int64_t t, int64_t depth, int64_t* ring, void* psp, double decay,
                     int32_t bg_mode, const void* bg, const double* lam, double mu, double sigma, uint64_t seed,
                     int64_t neuron_base, const void* extra, void* cur, double w_scale, void* stream) {
  if (n <= 0) return HHB_OK;
  if (!ring || !psp || !cur || depth < 1 || (bg_mode == 1 && !bg) || (bg_mode == 2 && !lam))
    return fail(HHB_EINVAL, "bad cortex_input args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long* rg = reinterpret_cast<long long*>(ring);
  const unsigned grid = unsigned((n + 255) / 256);
  if (dtype == HHB_F32) {
    cortex::k_cortex_input<float><<<grid, 256, 0, st>>>(n, t, depth, rg, (float*)psp, float(decay), bg_mode,
                                                        (const float*)bg, lam, float(mu), float(sigma), seed,
                                                        neuron_base, (const float*)extra, (float*)cur,
                                                        float(w_scale));
  } else if (dtype == HHB_F64) {
    cortex::k_cortex_input<double><<<grid, 256, 0, st>>>(n, t, depth, rg, (double*)psp, decay, bg_mode,
                                                         (const double*)bg, lam, mu, sigma, seed, neuron_base,
                                                         (const double*)extra, (double*)cur, w_scale);
  } else {
    return fail(HHB_EINVAL, "dtype");
  }
  return cuda_check("k_cortex_input launch");
}

int hhb_spike_deliver(int64_t words, const uint32_t* bits, const int64_t* offsets, const int32_t* targets,
                      const int32_t* weights_fx, const int32_t* delays, int64_t t, int64_t depth, int64_t n_local,
                      int64_t* ring, void* stream) {
  if (words <= 0 || n_local <= 0) return HHB_OK;
  if (!bits || !offsets || !ring || depth < 1) return fail(HHB_EINVAL, "bad spike_deliver args");
  cortex::k_spike_deliver<<<unsigned(words), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      words, bits, offsets, targets, weights_fx, delays, t, depth, n_local, reinterpret_cast<long long*>(ring));
  return cuda_check("k_spike_deliver launch");
}

}  // extern "C"
