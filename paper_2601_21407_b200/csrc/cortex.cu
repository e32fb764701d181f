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

// compound Poisson N mu + sigma sqrt(N) z (cortex.py:225-232) in single
// precision, explicit roundings (repeated verbatim by jit.cu hh_net's bg_draw)
__device__ __forceinline__ float bg_draw_f32(float L, float mu, float sigma, uint4 r) {
  const float u = __fmul_rn(__fadd_rn(__uint2float_rn(r.x), 0.5f), 2.3283064365386963e-10f);
  float p = __expf(-L), c = p;
  int k = 0;
  while (u > c && k < 64) {
    ++k;
    p = __fmul_rn(p, __fdividef(L, float(k)));
    c = __fadd_rn(c, p);
  }
  float add = __fmul_rn(float(k), mu);
  if (sigma > 0.0f && k > 0) {
    const float u1 = __fmul_rn(__fadd_rn(__uint2float_rn(r.y), 0.5f), 2.3283064365386963e-10f);
    const float u2 = __fmul_rn(__fadd_rn(__uint2float_rn(r.z), 0.5f), 2.3283064365386963e-10f);
    const float z = __fmul_rn(__fsqrt_rn(__fmul_rn(-2.0f, __logf(u1))), __cosf(__fmul_rn(6.283185307179586f, u2)));
    add = __fadd_rn(add, __fmul_rn(__fmul_rn(sigma, __fsqrt_rn(float(k))), z));
  }
  return add;
}

// thalamic current of neuron i at step t (cortex.py:423-428: rng.random(n_syn)
// < lam, np.add.at of the firing synapses' weights): its CSR row in order,
// synapse k firing iff word (id mod 4) of Philox block (id / 4, t) < thr,
// id = base + k.  Sequential adds in row order -- repeated verbatim (float) by
// jit.cu hh_net, so the per-step kernels and the persistent kernel agree bit
// for bit.
template <typename T>
__device__ __forceinline__ T thal_sum(const int64_t* off, const T* w, int64_t base, uint32_t thr, uint64_t seed,
                                      int64_t i, int64_t t) {
  const int64_t k0 = off[i], k1 = off[i + 1];
  T s = T(0);
  for (int64_t g = (base + k0) >> 2; 4 * g - base < k1; ++g) {
    const uint4 r = Philox::run(make_uint4(uint32_t(g), uint32_t(uint64_t(g) >> 32), uint32_t(t),
                                           uint32_t(uint64_t(t) >> 32)),
                                make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
    const uint32_t wd[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t k = 4 * g + q - base;
      if (k >= k0 && k < k1 && wd[q] < thr) {
        if constexpr (sizeof(T) == 4) s = __fadd_rn(s, w[k]);
        else s = s + w[k];
      }
    }
  }
  return s;
}

template <typename T>
__global__ void k_thalamic(int64_t n, int64_t t, const long long* t_dev, const int64_t* off, const T* w,
                           int64_t base, int64_t t_on, int64_t t_off, uint32_t thr, uint64_t seed, T* extra) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (t_dev) t = *t_dev;
  extra[i] = (t >= t_on && t < t_off) ? thal_sum<T>(off, w, base, thr, seed, i, t) : T(0);
}

// t_dev != NULL: the step index is read from device memory (CUDA-graph replay
// of the network step; hhb_cortex_tick advances it), else t is used
template <typename T>
__global__ void k_cortex_input(int64_t n, int64_t t, const long long* t_dev, int64_t depth, long long* ring, T* psp,
                               T decay, int mode, const T* bg, const double* lam, T mu, T sigma, uint64_t seed,
                               int64_t nbase, const T* extra, T* cur, T w_scale, int64_t rep_ring = 0) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (t_dev) t = *t_dev;
  // replica blockIdx.y: its own ring / psp / current rows and key seed + r
  const int64_t r = blockIdx.y;
  ring += r * rep_ring;
  psp += r * n;
  cur += r * n;
  seed += uint64_t(r);
  long long* slot = ring + (t % depth) * n + i;
  const long long arr = *slot;
  *slot = 0;
  // reference order: psp *= decay; psp += arrived; psp += background (cortex.py:287-297);
  // single precision with explicit roundings: the persistent network kernel
  // (jit.cu hh_net) repeats this arithmetic bit for bit
  T x;
  if constexpr (sizeof(T) == 4) {
    x = __fadd_rn(__fmul_rn(psp[i], decay), __fmul_rn(float(double(arr)), w_scale));
  } else {
    x = psp[i] * decay;
    x = x + T(double(arr)) * w_scale;
  }
  if (mode == 1) {
    x = x + bg[i];
  } else if (mode == 2 && sizeof(T) == 4) {
    const uint4 r = Philox::run(make_uint4(uint32_t(i + nbase), uint32_t(uint64_t(i + nbase) >> 32), uint32_t(t),
                                           uint32_t(uint64_t(t) >> 32)),
                                make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
    x = __fadd_rn(float(x), bg_draw_f32(float(lam[i]), float(mu), float(sigma), r));
  } else if (mode == 2) {
    // compound Poisson N*mu + sigma*sqrt(N)*z, N ~ Poisson(lam), z ~ N(0,1) (cortex.py:225-232);
    // Philox-4x32-10 keyed by (seed, global neuron, step): identical on every rank layout
    const uint4 r = Philox::run(make_uint4(uint32_t(i + nbase), uint32_t(uint64_t(i + nbase) >> 32), uint32_t(t),
                                           uint32_t(uint64_t(t) >> 32)),
                                make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
    // single precision with fast intrinsics: the draw sits on every step's
    // critical path (one thread per neuron, few warps per SM), and the sampler
    // only has to be distributionally exact (Philox stream, not the reference RNG)
    const float L = float(lam[i]);
    const float u = (float(r.x) + 0.5f) * 2.3283064365386963e-10f;
    float p = __expf(-L), c = p;
    int k = 0;
    while (u > c && k < 64) {
      ++k;
      p *= __fdividef(L, float(k));
      c += p;
    }
    float add = float(k) * float(mu);
    if (sigma > T(0) && k > 0) {
      const float u1 = (float(r.y) + 0.5f) * 2.3283064365386963e-10f;
      const float u2 = (float(r.z) + 0.5f) * 2.3283064365386963e-10f;
      const float z = sqrtf(-2.0f * __logf(u1)) * __cosf(6.283185307179586f * u2);
      add += float(sigma) * sqrtf(float(k)) * z;
    }
    x = x + T(add);
  }
  psp[i] = x;
  cur[i] = extra ? x + extra[i] : x;
}

__global__ void __launch_bounds__(128) k_spike_deliver(int64_t words, const uint32_t* bits, const int64_t* off,
                                                       const int32_t* tgt, const int32_t* w, const int32_t* delay,
                                                       int64_t t, const long long* t_dev, int64_t depth, int64_t n,
                                                       long long* ring) {
  const int64_t b = blockIdx.x;
  if (b >= words) return;
  if (t_dev) t = *t_dev;
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

__global__ void k_tick(long long* t) { *t += 1; }

// Spike bitmap [T][words] (bit i of word w = neuron 32w + i, neurons >= n
// ignored) -> event list sorted by (step, neuron), the order of NumPy's
// nonzero over the unpacked raster (SpikeRecord, cortex.py:422-438).  Pass 1
// counts each row's events; the caller scans the counts; pass 2 writes each
// row's events at its offset (one block per row, block-wide scan of the
// per-thread word counts).
constexpr int kEvThreads = 256;
__device__ __forceinline__ uint32_t ev_word(const uint32_t* row, int64_t w, int64_t n) {
  uint32_t x = row[w];
  const int64_t left = n - w * 32;
  if (left < 32) x &= left <= 0 ? 0u : ((1u << left) - 1u);
  return x;
}
__global__ void __launch_bounds__(kEvThreads) k_event_counts(int64_t words, const uint32_t* bits, int64_t n,
                                                             int64_t* counts) {
  const uint32_t* row = bits + int64_t(blockIdx.x) * words;
  int c = 0;
  for (int64_t w = threadIdx.x; w < words; w += kEvThreads) c += __popc(ev_word(row, w, n));
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int part[kEvThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int k = 0; k < kEvThreads / 32; ++k) s += part[k];
    counts[blockIdx.x] = s;
  }
}
__global__ void __launch_bounds__(kEvThreads) k_event_write(int64_t words, const uint32_t* bits, int64_t n,
                                                            const int64_t* offsets, int32_t* out_t,
                                                            int32_t* out_id) {
  const int64_t t = blockIdx.x;
  const uint32_t* row = bits + t * words;
  // contiguous word range per thread keeps the output ascending
  const int64_t per = (words + kEvThreads - 1) / kEvThreads;
  const int64_t w0 = threadIdx.x * per, w1 = min(words, w0 + per);
  int c = 0;
  for (int64_t w = w0; w < w1; ++w) c += __popc(ev_word(row, w, n));
  __shared__ int scan[kEvThreads];
  scan[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < kEvThreads; o <<= 1) {
    const int v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t k = offsets[t] + scan[threadIdx.x] - c;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t x = ev_word(row, w, n);
    while (x) {
      const int b = __ffs(int(x)) - 1;
      x &= x - 1;
      out_t[k] = int32_t(t);
      out_id[k] = int32_t(w * 32 + b);
      ++k;
    }
  }
}

// Flattened delivery for the latency-bound per-step case (a few dozen spikes
// out of ~10^5 sources, ~10^3 synapses each): k_spike_compact (one block)
// lists the spiking sources of the bitmap in ascending order with the
// exclusive prefix of their synapse-row lengths; k_spike_scatter then gives
// every (spike, synapse) pair its own thread (grid-stride), instead of one
// block walking each word's rows serially.  The int64 fixed-point atomics
// commute, so the ring is bit-identical to k_spike_deliver's.
constexpr int kCompactThreads = 1024;
__global__ void __launch_bounds__(kCompactThreads) k_spike_compact(int64_t words, const uint32_t* bits,
                                                                    const int64_t* off, int32_t* src,
                                                                    int64_t* pre, int64_t* totals,
                                                                    int64_t rep_scratch = 0) {
  __shared__ int64_t scan[kCompactThreads];
  {  // replica blockIdx.x: its bitmap and its slice of the scratch
    const int64_t r = blockIdx.x;
    bits += r * words;
    totals = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(totals) + r * rep_scratch);
    pre = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(pre) + r * rep_scratch);
    src = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(src) + r * rep_scratch);
  }
  const int tid = threadIdx.x;
  const int64_t per = (words + kCompactThreads - 1) / kCompactThreads;
  const int64_t w0 = tid * per, w1 = min(words, w0 + per);
  int cnt = 0;
  int64_t len = 0;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t x = bits[w];
    cnt += __popc(x);
    while (x) {
      const int b = __ffs(int(x)) - 1;
      x &= x - 1;
      const int64_t s = w * 32 + b;
      len += off[s + 1] - off[s];
    }
  }
  // block-wide exclusive scans of (count, length), packed: count << 40 | length
  scan[tid] = (int64_t(cnt) << 40) | len;
  __syncthreads();
  for (int o = 1; o < kCompactThreads; o <<= 1) {
    const int64_t v = tid >= o ? scan[tid - o] : 0;
    __syncthreads();
    scan[tid] += v;
    __syncthreads();
  }
  const int64_t incl = scan[tid];
  const int64_t excl = incl - ((int64_t(cnt) << 40) | len);
  int64_t k = excl >> 40, acc = excl & ((int64_t(1) << 40) - 1);
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t x = bits[w];
    while (x) {
      const int b = __ffs(int(x)) - 1;
      x &= x - 1;
      const int64_t s = w * 32 + b;
      src[k] = int32_t(s);
      pre[k] = acc;
      acc += off[s + 1] - off[s];
      ++k;
    }
  }
  if (tid == kCompactThreads - 1) {
    totals[0] = incl >> 40;                               // spikes
    totals[1] = incl & ((int64_t(1) << 40) - 1);          // synapses
    pre[incl >> 40] = totals[1];
  }
}

__global__ void __launch_bounds__(256) k_spike_scatter(const int32_t* src, const int64_t* pre, const int64_t* totals,
                                                       const int64_t* off, const int32_t* tgt, const int32_t* w,
                                                       const int32_t* delay, int64_t t, const long long* t_dev,
                                                       int64_t depth, int64_t n, long long* ring,
                                                       int64_t rep_scratch = 0, int64_t rep_ring = 0) {
  {  // replica blockIdx.y
    const int64_t r = blockIdx.y;
    totals = reinterpret_cast<const int64_t*>(reinterpret_cast<const char*>(totals) + r * rep_scratch);
    pre = reinterpret_cast<const int64_t*>(reinterpret_cast<const char*>(pre) + r * rep_scratch);
    src = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(src) + r * rep_scratch);
    ring += r * rep_ring;
  }
  const int64_t ns = totals[0], total = totals[1];
  if (t_dev) t = *t_dev;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
    // last k with pre[k] <= g
    int64_t lo = 0, hi = ns;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(pre + mid) <= g) lo = mid;
      else hi = mid;
    }
    const int64_t j = off[src[lo]] + (g - pre[lo]);
    const int64_t slot = (t + delay[j]) % depth;
    atomicAdd(reinterpret_cast<unsigned long long*>(ring + slot * n + tgt[j]),
              static_cast<unsigned long long>(static_cast<long long>(w[j])));
  }
}

}  // namespace cortex
}  // namespace hhb

using namespace hhb;

extern "C" {

int hhb_cortex_input(int32_t dtype, int64_t n, int64_t t, int64_t depth, int64_t* ring, void* psp, double decay,
                     int32_t bg_mode, const void* bg, const double* lam, double mu, double sigma, uint64_t seed,
                     int64_t neuron_base, const void* extra, void* cur, double w_scale, void* stream) {
  return hhb_cortex_input_dev(dtype, n, t, nullptr, depth, ring, psp, decay, bg_mode, bg, lam, mu, sigma, seed,
                              neuron_base, extra, cur, w_scale, stream);
}

int hhb_cortex_input_dev(int32_t dtype, int64_t n, int64_t t, const int64_t* t_dev, int64_t depth, int64_t* ring,
                         void* psp, double decay, int32_t bg_mode, const void* bg, const double* lam, double mu,
                         double sigma, uint64_t seed, int64_t neuron_base, const void* extra, void* cur,
                         double w_scale, void* stream) {
  const long long* td = reinterpret_cast<const long long*>(t_dev);
  if (n <= 0) return HHB_OK;
  if (!ring || !psp || !cur || depth < 1 || (bg_mode == 1 && !bg) || (bg_mode == 2 && !lam))
    return fail(HHB_EINVAL, "bad cortex_input args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long* rg = reinterpret_cast<long long*>(ring);
  const unsigned grid = unsigned((n + 255) / 256);
  if (dtype == HHB_F32) {
    cortex::k_cortex_input<float><<<grid, 256, 0, st>>>(n, t, td, depth, rg, (float*)psp, float(decay), bg_mode,
                                                        (const float*)bg, lam, float(mu), float(sigma), seed,
                                                        neuron_base, (const float*)extra, (float*)cur,
                                                        float(w_scale));
  } else if (dtype == HHB_F64) {
    cortex::k_cortex_input<double><<<grid, 256, 0, st>>>(n, t, td, depth, rg, (double*)psp, decay, bg_mode,
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
  return hhb_spike_deliver_dev(words, bits, offsets, targets, weights_fx, delays, t, nullptr, depth, n_local, ring,
                               stream);
}

int hhb_spike_deliver_dev(int64_t words, const uint32_t* bits, const int64_t* offsets, const int32_t* targets,
                          const int32_t* weights_fx, const int32_t* delays, int64_t t, const int64_t* t_dev,
                          int64_t depth, int64_t n_local, int64_t* ring, void* stream) {
  if (words <= 0 || n_local <= 0) return HHB_OK;
  if (!bits || !offsets || !ring || depth < 1) return fail(HHB_EINVAL, "bad spike_deliver args");
  cortex::k_spike_deliver<<<unsigned(words), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      words, bits, offsets, targets, weights_fx, delays, t, reinterpret_cast<const long long*>(t_dev), depth,
      n_local, reinterpret_cast<long long*>(ring));
  return cuda_check("k_spike_deliver launch");
}

int64_t hhb_spike_scratch(int64_t n_sources) { return 2 * n_sources + 3; }


int hhb_spike_deliver_flat(int64_t words, const uint32_t* bits, const int64_t* offsets, const int32_t* targets,
                           const int32_t* weights_fx, const int32_t* delays, int64_t t, const int64_t* t_dev,
                           int64_t depth, int64_t n_local, int64_t* ring, int64_t* scratch, void* stream) {
  if (words <= 0 || n_local <= 0) return HHB_OK;
  if (!bits || !offsets || !ring || depth < 1 || !scratch) return fail(HHB_EINVAL, "bad spike_deliver_flat args");
  if (words * 32 >= (int64_t(1) << 23))    // the compaction packs spike counts in 23 bits
    return hhb_spike_deliver_dev(words, bits, offsets, targets, weights_fx, delays, t, t_dev, depth, n_local, ring,
                                 stream);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // scratch (int64): totals[2] | pre[words*32 + 1] | src (int32, words*32)
  int64_t* totals = scratch;
  int64_t* pre = scratch + 2;
  int32_t* src = reinterpret_cast<int32_t*>(pre + words * 32 + 1);
  cortex::k_spike_compact<<<1, cortex::kCompactThreads, 0, st>>>(words, bits, offsets, src, pre, totals);
  cortex::k_spike_scatter<<<2 * kNumSMs, 256, 0, st>>>(src, pre, totals, offsets, targets, weights_fx, delays, t,
                                                        reinterpret_cast<const long long*>(t_dev), depth, n_local,
                                                        reinterpret_cast<long long*>(ring));
  return cuda_check("k_spike_compact / k_spike_scatter launch");
}

int hhb_cortex_step_batch(int32_t dtype, int64_t replicas, int64_t n_pad, int64_t words, const int64_t* t_dev,
                          int64_t depth, int64_t* ring, void* psp, double decay, const double* lam, double mu,
                          double sigma, uint64_t seed, void* cur, double w_scale, const uint32_t* bits,
                          const int64_t* offsets, const int32_t* targets, const int32_t* weights_fx,
                          const int32_t* delays, int64_t* scratch, int32_t phase, void* stream) {
  // phase 0: the input of every replica; phase 1: compaction + delivery of every
  // replica's bitmap (the HH step of all replicas' neurons runs in between as
  // one population of replicas * n_pad neurons)
  if (replicas < 1 || n_pad <= 0 || n_pad % 32 || words != n_pad / 32 || !t_dev || !ring)
    return fail(HHB_EINVAL, "bad cortex batch args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  long long* rg = reinterpret_cast<long long*>(ring);
  const int64_t rep_ring = depth * n_pad;
  if (phase == 0) {
    if (!psp || !cur || !lam) return fail(HHB_EINVAL, "bad cortex batch input args");
    const dim3 grid{unsigned((n_pad + 255) / 256), unsigned(replicas), 1u};
    const long long* td = reinterpret_cast<const long long*>(t_dev);
    if (dtype == HHB_F32)
      cortex::k_cortex_input<float><<<grid, 256, 0, st>>>(n_pad, 0, td, depth, rg, (float*)psp, float(decay), 2,
                                                          nullptr, lam, float(mu), float(sigma), seed, 0, nullptr,
                                                          (float*)cur, float(w_scale), rep_ring);
    else if (dtype == HHB_F64)
      cortex::k_cortex_input<double><<<grid, 256, 0, st>>>(n_pad, 0, td, depth, rg, (double*)psp, decay, 2, nullptr,
                                                           lam, mu, sigma, seed, 0, nullptr, (double*)cur, w_scale,
                                                           rep_ring);
    else
      return fail(HHB_EINVAL, "dtype");
    return cuda_check("k_cortex_input (batch) launch");
  }
  if (!bits || !offsets || !scratch) return fail(HHB_EINVAL, "bad cortex batch delivery args");
  if (words * 32 >= (int64_t(1) << 23)) return fail(HHB_EINVAL, "cortex batch: too many neurons per replica");
  const int64_t per = hhb_spike_scratch(words * 32);         // int64 per replica
  int64_t* totals = scratch;
  int64_t* pre = scratch + 2;
  int32_t* src = reinterpret_cast<int32_t*>(pre + words * 32 + 1);
  cortex::k_spike_compact<<<unsigned(replicas), cortex::kCompactThreads, 0, st>>>(words, bits, offsets, src, pre,
                                                                                  totals, per * 8);
  const dim3 g2{unsigned(kNumSMs), unsigned(replicas), 1u};
  cortex::k_spike_scatter<<<g2, 256, 0, st>>>(src, pre, totals, offsets, targets, weights_fx, delays, 0,
                                              reinterpret_cast<const long long*>(t_dev), depth, n_pad, rg, per * 8,
                                              rep_ring);
  return cuda_check("k_spike_compact / k_spike_scatter (batch) launch");
}

static int cortex_run_impl(const hhb_params_t* params, int64_t replicas, int64_t ld, int64_t n, int64_t steps,
                           int64_t t0, int64_t depth, int64_t* ring, float* psp, double decay, int32_t bg_mode,
                           const double* lam, double mu, double sigma, uint64_t seed, int64_t neuron_base,
                           double w_scale, float* v, float* g, int64_t g_ld, uint32_t* bits, int32_t record,
                           int64_t words, const int64_t* segments, int64_t tiles, const int32_t* targets,
                           const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad, uint32_t* barrier,
                           uint64_t* timing, const hhb_thalamic_t* thal, void* stream) {
  int rc = check_params(params);
  if (rc) return rc;
  if (n <= 0 || steps <= 0) return HHB_OK;
  if (replicas < 1 || ld < n) return fail(HHB_EINVAL, "cortex_run: replicas >= 1 and ld >= n");
  if (tiles != (n + 255) / 256) return fail(HHB_EINVAL, "cortex_run: tiles != ceil(n / 256)");
  if (!ring || !psp || !v || (params->n_gates > 0 && (!g || g_ld < n)) || !bits || !segments || !first_bad ||
      !barrier || depth < 1 || words != (n + 31) / 32 || (bg_mode != 0 && bg_mode != 2) || (bg_mode == 2 && !lam) ||
      (params->n_gates > 0 && g_ld < replicas * ld))
    return fail(HHB_EINVAL, "bad cortex_run args");
  CortexRunArgs a{};
  a.n = n;
  a.steps = steps;
  a.t0 = t0;
  a.depth = depth;
  a.ring = reinterpret_cast<long long*>(ring);
  a.psp = psp;
  a.lam = lam;
  a.decay = float(decay);
  a.mu = float(mu);
  a.sigma = float(sigma);
  a.w_scale = float(w_scale);
  a.mode = bg_mode;
  a.rec = record ? 1 : 0;
  a.seed = seed;
  a.nbase = neuron_base;
  a.v = v;
  a.g = g;
  a.g_ld = g_ld;
  a.bits = bits;
  a.words = words;
  a.seg = segments;
  a.tiles = tiles;
  a.tgt = targets;
  a.w = weights_fx;
  a.delay = delays;
  a.first_bad = first_bad;
  a.bar = barrier;
  a.timing = reinterpret_cast<unsigned long long*>(timing);
  a.reps = replicas;
  a.ld = ld;
  if (thal) {
    if (replicas != 1) return fail(HHB_EINVAL, "cortex_run: the thalamic drive needs one replica");
    if (!thal->offsets || !thal->weights) return fail(HHB_EINVAL, "cortex_run: bad thalamic table");
    a.th_off = thal->offsets;
    a.th_w = static_cast<const float*>(thal->weights);
    a.th_base = thal->id_base;
    a.th_on = thal->t_on;
    a.th_end = thal->t_off;
    a.th_thr = thal->threshold;
    a.th_seed = thal->seed;
  }
  if (!jit_cortex_run(params, a, static_cast<cudaStream_t>(stream), rc))
    return fail(HHB_ENOTSUP, std::string("persistent network kernel unavailable: ") + jit_status());
  return rc;
}

int hhb_spike_event_counts(int64_t steps, int64_t words, const uint32_t* bits, int64_t n, int64_t* counts,
                           void* stream) {
  if (steps < 0 || words < 0 || n < 0 || n > words * 32) return fail(HHB_EINVAL, "spike_event_counts: bad sizes");
  if (steps == 0) return HHB_OK;
  if (!bits || !counts) return fail(HHB_EINVAL, "spike_event_counts: NULL pointer");
  cortex::k_event_counts<<<unsigned(steps), cortex::kEvThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      words, bits, n, counts);
  return cuda_check("k_event_counts launch");
}

int hhb_spike_events(int64_t steps, int64_t words, const uint32_t* bits, int64_t n, const int64_t* offsets,
                     int32_t* out_step, int32_t* out_neuron, void* stream) {
  if (steps < 0 || words < 0 || n < 0 || n > words * 32) return fail(HHB_EINVAL, "spike_events: bad sizes");
  if (steps == 0) return HHB_OK;
  if (!bits || !offsets || !out_step || !out_neuron) return fail(HHB_EINVAL, "spike_events: NULL pointer");
  cortex::k_event_write<<<unsigned(steps), cortex::kEvThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      words, bits, n, offsets, out_step, out_neuron);
  return cuda_check("k_event_write launch");
}

int hhb_cortex_run_replicas(const hhb_params_t* params, int64_t replicas, int64_t ld, int64_t n, int64_t steps,
                            int64_t t0, int64_t depth, int64_t* ring, float* psp, double decay, int32_t bg_mode,
                            const double* lam, double mu, double sigma, uint64_t seed, int64_t neuron_base,
                            double w_scale, float* v, float* g, int64_t g_ld, uint32_t* bits, int32_t record,
                            int64_t words, const int64_t* segments, int64_t tiles, const int32_t* targets,
                            const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad, uint32_t* barrier,
                            uint64_t* timing, void* stream) {
  return cortex_run_impl(params, replicas, ld, n, steps, t0, depth, ring, psp, decay, bg_mode, lam, mu, sigma, seed,
                         neuron_base, w_scale, v, g, g_ld, bits, record, words, segments, tiles, targets, weights_fx,
                         delays, first_bad, barrier, timing, nullptr, stream);
}

int hhb_cortex_run_ex(const hhb_params_t* params, int64_t n, int64_t steps, int64_t t0, int64_t depth, int64_t* ring,
                      float* psp, double decay, int32_t bg_mode, const double* lam, double mu, double sigma,
                      uint64_t seed, int64_t neuron_base, double w_scale, float* v, float* g, int64_t g_ld,
                      uint32_t* bits, int32_t record, int64_t words, const int64_t* segments, int64_t tiles,
                      const int32_t* targets, const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad,
                      uint32_t* barrier, uint64_t* timing, const hhb_thalamic_t* thal, void* stream) {
  return cortex_run_impl(params, 1, n, n, steps, t0, depth, ring, psp, decay, bg_mode, lam, mu, sigma, seed,
                         neuron_base, w_scale, v, g, g_ld, bits, record, words, segments, tiles, targets, weights_fx,
                         delays, first_bad, barrier, timing, thal, stream);
}

int hhb_cortex_run(const hhb_params_t* params, int64_t n, int64_t steps, int64_t t0, int64_t depth, int64_t* ring,
                   float* psp, double decay, int32_t bg_mode, const double* lam, double mu, double sigma,
                   uint64_t seed, int64_t neuron_base, double w_scale, float* v, float* g, int64_t g_ld,
                   uint32_t* bits, int32_t record, int64_t words, const int64_t* segments, int64_t tiles,
                   const int32_t* targets, const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad,
                   uint32_t* barrier, uint64_t* timing, void* stream) {
  return hhb_cortex_run_replicas(params, 1, n, n, steps, t0, depth, ring, psp, decay, bg_mode, lam, mu, sigma, seed,
                                 neuron_base, w_scale, v, g, g_ld, bits, record, words, segments, tiles, targets,
                                 weights_fx, delays, first_bad, barrier, timing, stream);
}

int hhb_thalamic_drive(int32_t dtype, int64_t n, int64_t t, const int64_t* t_dev, const hhb_thalamic_t* thal,
                       void* extra, void* stream) {
  if (n <= 0) return HHB_OK;
  if (!thal || !thal->offsets || !thal->weights || !extra) return fail(HHB_EINVAL, "bad thalamic_drive args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long* td = reinterpret_cast<const long long*>(t_dev);
  const unsigned grid = unsigned((n + 255) / 256);
  if (dtype == HHB_F32) {
    cortex::k_thalamic<float><<<grid, 256, 0, st>>>(n, t, td, thal->offsets, (const float*)thal->weights,
                                                    thal->id_base, thal->t_on, thal->t_off, thal->threshold,
                                                    thal->seed, (float*)extra);
  } else if (dtype == HHB_F64) {
    cortex::k_thalamic<double><<<grid, 256, 0, st>>>(n, t, td, thal->offsets, (const double*)thal->weights,
                                                     thal->id_base, thal->t_on, thal->t_off, thal->threshold,
                                                     thal->seed, (double*)extra);
  } else {
    return fail(HHB_EINVAL, "dtype");
  }
  return cuda_check("k_thalamic launch");
}

int hhb_cortex_tick(int64_t* t_dev, void* stream) {
  if (!t_dev) return fail(HHB_EINVAL, "t_dev is NULL");
  cortex::k_tick<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<long long*>(t_dev));
  return cuda_check("k_tick launch");
}

}  // extern "C"
