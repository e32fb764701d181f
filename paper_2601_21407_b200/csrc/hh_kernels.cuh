// hh_kernels.cuh -- sm_100a kernels of the HH hot path, templated on the
// scalar type (float = throughput build, double = parity build) and on the
// gate count NG, so the gate state lives in registers.
//
//   k_forward   time-fused forward (simulate/hh_step, dynamics.py:443-586)
//   k_backward  reverse sweep with checkpoint-segment recompute
//               (backward_through_time/hh_step_backward, adjoint.py:102-365)
//   k_reduce    deterministic second pass of the parameter-gradient sums
//   k_* small   elementwise ops of dynamics.py:324-381 / adjoint.py:60-66
//   k_poisson   Philox-keyed Poisson stimulus (BASELINE config 2 input)
#pragma once

#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "hh_device.cuh"
#include "pdl.cuh"

namespace hhb {

constexpr int kFwdThreads = 256;
constexpr int kBwdThreads = 128;

template <typename T>
struct FwdArgs {
  int64_t n, steps;
  const T* v_in;
  const T* g_in;
  int64_t g_ld;
  T* v_fin;
  T* g_fin;
  const T* i_ext;
  int64_t i_st, i_sn;
  T* v_out;
  int64_t v_ld;
  uint32_t* spk;
  int64_t spk_ld;
  T* ckpt;
  int64_t ck_every, ck_ld;
  int64_t step_base;
  long long* first_bad;
  uint64_t seed;    // fused Poisson stimulus (hhb_forward_poisson): Philox key
  int64_t nbase;    //   global id of neuron 0 of this launch
  T* spk_val;       // optional spike flags as 0/1 values [steps][spkv_ld] (SNN layer output)
  int64_t spkv_ld;
  const long long* step_dev;   // optional: device value added to step_base
  double* sq_part;             // optional: per-block partial sums of V'^2 (fused MSE(V, 0) forward)
  uint16_t* spk_bf;            // optional: spike flags as bf16 0/1 [steps][spkb_ld] (the next layer's GEMM operand)
  int64_t spkb_ld;
};

template <typename T>
struct BwdArgs {
  int64_t n, steps;
  const T* i_ext;
  int64_t i_st, i_sn;
  const T* ckpt;
  int64_t ck_every, ck_ld;
  T* seg;
  const T* seed_v;
  int64_t sv_ld;
  const T* seed_s;
  int64_t ss_ld;
  T* adj_v;
  T* adj_g;
  int64_t ag_ld;
  T* d_i;
  int64_t di_ld;
  double* partials;
  int64_t step_base;
  long long* first_bad;
  // layer outputs (float only; NULL = off): dI as bf16 hi + lo planes
  // ([steps][dh_ld] each, hi = bf16(dI), lo = bf16(dI - hi)) for the bf16x2
  // gradient GEMMs, and per-neuron sums of dI over the steps (+=) for d_bias
  uint16_t* di_hi;
  uint16_t* di_lo;
  int64_t dh_ld;
  float* di_sum;
  int64_t dh_grp, dh_pitch;   // > 0: neuron i at column (i / grp) * pitch + i % grp
  const float* sv_scale;      // optional: seed_v is read times *sv_scale (fused MSE(V, 0) backward)
};

__host__ __device__ inline int64_t split_col(int64_t i, int64_t grp, int64_t pitch) {
  return grp > 0 ? (i / grp) * pitch + i % grp : i;
}

__device__ __forceinline__ void split_bf16(float x, uint16_t& hi, uint16_t& lo) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t h = (b + 0x7FFFu + ((b >> 16) & 1u)) & 0xFFFF0000u;
  const uint32_t c = __float_as_uint(__fsub_rn(x, __uint_as_float(h)));
  hi = uint16_t(h >> 16);
  lo = uint16_t((c + 0x7FFFu + ((c >> 16) & 1u)) >> 16);
}

// ------------------------------------------------------------ vector I/O
template <typename T, int VEC>
struct Vec;
template <>
struct Vec<float, 1> {
  __device__ static void ld(const float* p, float (&x)[1]) { x[0] = __ldg(p); }
  __device__ static void st(float* p, const float (&x)[1]) { *p = x[0]; }
};
template <>
struct Vec<float, 4> {
  __device__ static void ld(const float* p, float (&x)[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
  }
  __device__ static void st(float* p, const float (&x)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
  }
};
template <>
struct Vec<double, 1> {
  __device__ static void ld(const double* p, double (&x)[1]) { x[0] = __ldg(p); }
  __device__ static void st(double* p, const double (&x)[1]) { *p = x[0]; }
};
template <>
struct Vec<double, 2> {
  __device__ static void ld(const double* p, double (&x)[2]) {
    const double2 q = __ldg(reinterpret_cast<const double2*>(p));
    x[0] = q.x; x[1] = q.y;
  }
  __device__ static void st(double* p, const double (&x)[2]) {
    *reinterpret_cast<double2*>(p) = make_double2(x[0], x[1]);
  }
};

// ------------------------------------------------------------ stimulus RNG
// Philox-4x32-10 (Salmon et al. 2011): counter = (global neuron / 4, global
// step), key = seed; word i of a block drives global neuron 4*group + i.
struct Philox {
  __device__ static uint4 run(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
  __device__ static uint4 block(uint64_t seed, int64_t group, int64_t gt) {
    return run(make_uint4(uint32_t(group), uint32_t(uint64_t(group) >> 32), uint32_t(gt),
                          uint32_t(uint64_t(gt) >> 32)),
               make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
  }
  // the word of global neuron gj at global step gt
  __device__ static uint32_t word(uint64_t seed, int64_t gj, int64_t gt) {
    const uint4 r = block(seed, gj >> 2, gt);
    const int i = int(gj & 3);
    return i == 0 ? r.x : i == 1 ? r.y : i == 2 ? r.z : r.w;
  }
};

// inverse-CDF table of Poisson(lam), built on the host in fp64
template <typename T>
struct PoissonTab {
  int size;      // entries used; cdf[size-1] >= 1 - 2^-33
  T amp;
  T cdf[48];
};

// amp * Poisson(lam) from one uniform 32-bit word (inverse CDF)
template <typename T>
__device__ __forceinline__ T poisson_draw(const PoissonTab<T>& tab, uint32_t word) {
  const T u = (T(word) + T(0.5)) * T(2.3283064365386963e-10);
  int k = 0;
  while (k < tab.size - 1 && u > tab.cdf[k]) ++k;
  return tab.amp * T(k);
}

// The same draw through a guide table (Chen & Asau 1974) in shared memory:
// guide[b] = min{k : cdf[k] >= b/256} <= the answer for every word whose top
// byte is b (float(word) >= b * 2^24 exactly), so the search starts there and
// usually stops at once.  Bit-identical to poisson_draw; avoids the warp
// paying the longest of 32 (x VEC) linear searches.
//
// Each bucket stores {amp*k0, C(k0), C(k0+1), C(k0+2)} (C(j) = cdf[j], raised to 2 > any
// u from j = size-1 on, where the capped search stops), so a draw is one 16-byte
// shared load, two compares and, for the rare u > C(k0+2), a tail walk.  The
// uniform is (word >> 9) * 2^-23, built from the mantissa bits (no int->float).
template <typename T>
struct PoissonSmem {
  __align__(16) T g4[256][4];
  int k0[256];
  T cdf[48];
  T amp;
  __device__ void fill(const PoissonTab<T>& tab) {
    for (int k = threadIdx.x; k < 48; k += blockDim.x) cdf[k] = k < tab.size - 1 ? tab.cdf[k] : T(2);
    if (threadIdx.x == 0) amp = tab.amp;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
      const T lo = T(b) * T(0.00390625);
      int k = 0;
      while (k < tab.size - 1 && tab.cdf[k] < lo) ++k;
      k0[b] = k;
      const auto C = [&](int j) { return j < tab.size - 1 ? tab.cdf[j] : T(2); };
      g4[b][0] = tab.amp * T(k);
      g4[b][1] = C(k);
      g4[b][2] = C(k + 1);
      g4[b][3] = C(k + 2);
    }
  }
  __device__ __forceinline__ static T uniform(uint32_t w) {
    if constexpr (sizeof(T) == 4) {
      return __uint_as_float(0x3F800000u | (w >> 9)) - 1.0f;
    } else {
      return T(w >> 9) * T(1.1920928955078125e-07);
    }
  }
  // the draw, and whether it needs the tail walk (u beyond C(k0+2))
  __device__ __forceinline__ T draw(uint32_t w, bool& tail) const {
    const T u = uniform(w);
    const T* e = g4[w >> 24];
    T val = e[0];
    val = (u > e[1]) ? val + amp : val;
    val = (u > e[2]) ? val + amp : val;
    tail = u > e[3];
    return val;
  }
  __device__ T tail_draw(uint32_t w) const {
    const T u = uniform(w);
    int k = k0[w >> 24] + 3;
    while (u > cdf[k]) ++k;
    return amp * T(k);
  }
};

// current of VEC consecutive neurons at step t; vector load when dense
template <typename T, int VEC>
__device__ __forceinline__ void load_cur(const FwdArgs<T>& a, int64_t t, int64_t n0, bool full,
                                         T (&c)[VEC]) {
  if (VEC > 1 && full && a.i_sn == 1) {
    Vec<T, VEC>::ld(a.i_ext + t * a.i_st + n0, c);
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j)
      c[j] = (n0 + j < a.n) ? __ldg(a.i_ext + t * a.i_st + (n0 + j) * a.i_sn) : T(0);
  }
}

// pack VEC spike flags per lane into the bitmap word of 32 neurons
template <int VEC>
__device__ __forceinline__ uint32_t spike_word(const bool (&s)[VEC], int lane) {
  if constexpr (VEC == 1) {
    return __ballot_sync(0xffffffffu, s[0]);
  } else {
    static_assert(32 % VEC == 0, "VEC must divide 32");
    uint32_t nib = 0;
#pragma unroll
    for (int j = 0; j < VEC; ++j) nib |= uint32_t(s[j]) << j;
    constexpr int kLanes = 32 / VEC;  // lanes sharing one word
    uint32_t w = nib << (VEC * (lane % kLanes));
#pragma unroll
    for (int o = 1; o < kLanes; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
    return w;
  }
}

// Per-thread source of the injected current: the i_ext array (load, with the
// next step prefetched by the caller) or, for POIS, the Poisson stimulus drawn
// in registers from the Philox block of (global neuron / 4, global step) --
// the exact stream k_poisson writes, without its HBM round trip.  VEC == 4
// needs (nbase + n0) % 4 == 0 (the host checks nbase % 4) and then uses one
// block per thread and step.
template <typename T, int VEC, bool POIS>
struct Stimulus {
  __device__ __forceinline__ void at(const FwdArgs<T>& a, const PoissonSmem<T>& tab, int64_t t, int64_t n0,
                                     bool full, T (&c)[VEC]) {
    if constexpr (POIS) {
      const int64_t gt = a.step_base + t;
      uint32_t w[VEC];
      if constexpr (VEC == 4) {
        const uint4 r = Philox::block(a.seed, (a.nbase + n0) >> 2, gt);
        w[0] = r.x;
        w[1] = r.y;
        w[2] = r.z;
        w[3] = r.w;
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) w[j] = Philox::word(a.seed, a.nbase + n0 + j, gt);
      }
      bool tail[VEC], any_tail = false;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        c[j] = tab.draw(w[j], tail[j]);
        any_tail = any_tail || tail[j];
      }
      if (__any_sync(0xffffffffu, any_tail)) {  // one vote for all VEC draws
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (tail[j]) c[j] = tab.tail_draw(w[j]);
      }
    } else {
      load_cur<T, VEC>(a, t, n0, full, c);
    }
  }
};

// ------------------------------------------------------------ forward
template <typename T, int NG, int VEC, bool POIS>
__global__ void __launch_bounds__(kFwdThreads) k_forward(const DevTable<T> tb, const FwdArgs<T> a_in,
                                                         const PoissonTab<T> ptab) {
  FwdArgs<T> a = a_in;
  if (a.step_dev != nullptr) a.step_base += *a.step_dev;
  constexpr int NGX = NG > 0 ? NG : 1;
  const int lane = threadIdx.x & 31;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n0 = tid * VEC;
  const bool full = n0 + VEC <= a.n;
  Stimulus<T, VEC, POIS> stim;
  __shared__ PoissonSmem<T> ps;
  if constexpr (POIS) {
    ps.fill(ptab);
    __syncthreads();
  }

  T v[VEC];
  T p[VEC][NGX];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const bool on = n0 + j < a.n;
    v[j] = on ? a.v_in[n0 + j] : T(-65);
#pragma unroll
    for (int g = 0; g < NG; ++g) p[j][g] = on ? a.g_in[g * a.g_ld + n0 + j] : T(0.5);
  }
  long long bad = LLONG_MAX;
  int64_t ck_slot = 0;
  int64_t ck_count = 0;
  double sq = 0.0;

  // one neuron per thread (small, latency-bound populations): the loaded
  // current is prefetched PF steps ahead through registers that rotate by
  // name (loop unrolled PF times); the loads are unconditional (padding lanes
  // read element 0, rows past the end re-read the last one) and the value is
  // copied out with an explicit add, so no register move waits on a load
  // (float only: the float64 step is long enough to cover the load, and unrolling it
  // measured slower -- instruction-cache pressure of four copies of the float64 step)
  constexpr int PF = (VEC == 1 && !POIS && sizeof(T) == 4) ? 4 : 1;
  T cur[VEC];
  T pre[PF];
  const T* ib1 = (n0 < a.n) ? a.i_ext + n0 * a.i_sn : a.i_ext;
  if (a.steps > 0) {
    if constexpr (PF > 1) {
#pragma unroll
      for (int k = 0; k < PF; ++k) pre[k] = __ldg(ib1 + (k < a.steps ? k : a.steps - 1) * a.i_st);
    } else {
      stim.at(a, ps, 0, n0, full, cur);
    }
  }
  for (int64_t t_blk = 0; t_blk < a.steps; t_blk += PF)
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int64_t t = t_blk + k;
    if (PF > 1 && t >= a.steps) break;
    T nxt[VEC];
    if constexpr (PF > 1) {
      cur[0] = pre[k] + T(0);
      const int64_t r = t + PF < a.steps ? t + PF : a.steps - 1;
      pre[k] = __ldg(ib1 + r * a.i_st);
    } else {
      if (t + 1 < a.steps) stim.at(a, ps, t + 1, n0, full, nxt);
    }
    if (a.ckpt != nullptr && ck_count == 0) {  // state BEFORE step t
      T* base = a.ckpt + ck_slot * (1 + NG) * a.ck_ld;
      if (full) {
        Vec<T, VEC>::st(base + n0, v);
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          T q[VEC];
#pragma unroll
          for (int j = 0; j < VEC; ++j) q[j] = p[j][g];
          Vec<T, VEC>::st(base + (1 + g) * a.ck_ld + n0, q);
        }
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          if (n0 + j < a.n) {
            base[n0 + j] = v[j];
#pragma unroll
            for (int g = 0; g < NG; ++g) base[(1 + g) * a.ck_ld + n0 + j] = p[j][g];
          }
        }
      }
      ++ck_slot;
      ck_count = a.ck_every;
    }
    --ck_count;

    bool spk[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const T vn = step_forward<T, NG>(tb, v[j], p[j], cur[j]);
      spk[j] = (v[j] < tb.theta) && (vn >= tb.theta);  // spike_detect, dynamics.py:379-381
      if (!finite_(vn) && bad == LLONG_MAX && n0 + j < a.n) bad = a.step_base + t;
      if (a.sq_part != nullptr && n0 + j < a.n) sq += double(vn) * double(vn);
      v[j] = vn;
    }
    if (a.v_out != nullptr) {
      T* row = a.v_out + t * a.v_ld;
      if (full) {
        Vec<T, VEC>::st(row + n0, v);
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (n0 + j < a.n) row[n0 + j] = v[j];
      }
    }
    if (a.spk_val != nullptr) {
      T* row = a.spk_val + t * a.spkv_ld;
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (n0 + j < a.n) row[n0 + j] = spk[j] ? T(1) : T(0);
    }
    if (a.spk_bf != nullptr) {
      uint16_t* row = a.spk_bf + t * a.spkb_ld;
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (n0 + j < a.n) row[n0 + j] = spk[j] ? uint16_t(0x3F80) : uint16_t(0);
    }
    if (a.spk != nullptr) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) spk[j] = spk[j] && (n0 + j < a.n);
      const uint32_t w = spike_word<VEC>(spk, lane);
      if (lane % (32 / VEC) == 0 && n0 < a.n) a.spk[t * a.spk_ld + n0 / 32] = w;
    }
    if constexpr (PF == 1) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) cur[j] = nxt[j];
    }
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    if (n0 + j < a.n) {
      a.v_fin[n0 + j] = v[j];
#pragma unroll
      for (int g = 0; g < NG; ++g) a.g_fin[g * a.g_ld + n0 + j] = p[j][g];
    }
  }
  if (bad != LLONG_MAX) atomicMin(a.first_bad, bad);
  if (a.sq_part != nullptr) {   // block partial of sum V'^2: warp shuffle, warps in fixed order
    __shared__ double red[kFwdThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double x = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) x += red[w];
      a.sq_part[blockIdx.x] = x;
    }
  }
}

// ------------------------------------------------------------ backward
template <typename T, int NG>
__device__ __forceinline__ void load_state(const T* base, int64_t ld, int64_t i, T& v,
                                           T (&p)[NG > 0 ? NG : 1]) {
  v = base[i];
#pragma unroll
  for (int g = 0; g < NG; ++g) p[g] = base[(1 + g) * ld + i];
}
template <typename T, int NG>
__device__ __forceinline__ void store_state(T* base, int64_t ld, int64_t i, T v,
                                            const T (&p)[NG > 0 ? NG : 1]) {
  base[i] = v;
#pragma unroll
  for (int g = 0; g < NG; ++g) base[(1 + g) * ld + i] = p[g];
}

template <typename T, int NG>
__global__ void __launch_bounds__(kBwdThreads) k_backward(const DevTable<T> tb, const DevSur<T> sur,
                                                          const BwdArgs<T> a) {
  constexpr int NGX = NG > 0 ? NG : 1;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool on = i < a.n;
  const int64_t ii = on ? i : 0;  // inactive lanes shadow neuron 0, never store

  double acc[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) acc[s] = 0.0;
  long long bad = -1;
  double csum = 0.0;

  T d_v = on ? a.adj_v[ii] : T(0);
  T d_p[NGX];
#pragma unroll
  for (int g = 0; g < NG; ++g) d_p[g] = on ? a.adj_g[g * a.ag_ld + ii] : T(0);

  const int64_t K = a.ck_every;
  const int64_t nseg = (a.steps + K - 1) / K;
  const int64_t state_stride = (1 + NG) * a.ck_ld;
  for (int64_t seg = nseg - 1; seg >= 0; --seg) {
    const int64_t lo = seg * K;
    const int64_t hi = (lo + K < a.steps) ? lo + K : a.steps;
    const T* ck = a.ckpt + seg * state_stride;
    T v;
    T p[NGX];
    load_state<T, NG>(ck, a.ck_ld, ii, v, p);
    if (K > 1) {
      // recompute the segment's states (adjoint.py:340-348) into seg_buf
      for (int64_t t = lo; t < hi - 1; ++t) {
        const T cur = __ldg(a.i_ext + t * a.i_st + ii * a.i_sn);
        v = step_forward<T, NG>(tb, v, p, cur);
        if (on) store_state<T, NG>(a.seg + (t + 1 - lo) * state_stride, a.ck_ld, ii, v, p);
      }
    }
    for (int64_t t = hi - 1; t >= lo; --t) {
      if (t != hi - 1 || K == 1) {
        const T* src = (K == 1) ? a.ckpt + t * state_stride
                                : (t == lo ? ck : a.seg + (t - lo) * state_stride);
        load_state<T, NG>(src, a.ck_ld, ii, v, p);
      }
      const T cur = __ldg(a.i_ext + t * a.i_st + ii * a.i_sn);
      if (a.seed_v != nullptr)
        d_v = add_(d_v, a.sv_scale != nullptr ? T(__ldg(a.seed_v + t * a.sv_ld + ii) * T(*a.sv_scale))
                                              : __ldg(a.seed_v + t * a.sv_ld + ii));
      const bool has_s = a.seed_s != nullptr;
      const T ds = has_s ? __ldg(a.seed_s + t * a.ss_ld + ii) : T(0);
      const T di = step_backward<T, NG>(tb, sur, v, p, cur, d_v, d_p, ds, has_s, acc);
      if (on && a.d_i != nullptr) a.d_i[t * a.di_ld + ii] = di;
      if constexpr (sizeof(T) == 4) {
        if (on && a.di_hi != nullptr) {
          uint16_t h, l;
          split_bf16(float(di), h, l);
          const int64_t col = split_col(ii, a.dh_grp, a.dh_pitch);
          a.di_hi[t * a.dh_ld + col] = h;
          a.di_lo[t * a.dh_ld + col] = l;
        }
        csum += double(di);
      }
      bool ok = finite_(d_v);
#pragma unroll
      for (int g = 0; g < NG; ++g) ok = ok && finite_(d_p[g]);
      if (!ok && bad < 0 && on) bad = a.step_base + t;
    }
  }
  if (on) {
    a.adj_v[ii] = d_v;
#pragma unroll
    for (int g = 0; g < NG; ++g) a.adj_g[g * a.ag_ld + ii] = d_p[g];
    if (a.di_sum != nullptr) a.di_sum[ii] += float(csum);
  }
  if (bad >= 0) atomicMax(a.first_bad, bad);

  // block partials: warp shuffle, then warps in fixed order
  __shared__ double red[kBwdThreads / 32][kSlots];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    double x = on ? acc[s] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][s] = x;
  }
  __syncthreads();
  if (threadIdx.x < kSlots) {
    double x = 0.0;
    for (int w = 0; w < kBwdThreads / 32; ++w) x += red[w][threadIdx.x];
    a.partials[int64_t(blockIdx.x) * kSlots + threadIdx.x] = x;
  }
}

// second pass: one block per slot, fixed assignment + fixed tree => deterministic
template <typename T>
__global__ void __launch_bounds__(256) k_reduce(const DevTable<T> tb, const double* partials,
                                                int64_t nblocks, double* d_params) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x;
  double x = 0.0;
  for (int64_t b = threadIdx.x; b < nblocks; b += blockDim.x) x += partials[b * kSlots + s];
  __shared__ double red[256];
  red[threadIdx.x] = x;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const double tot = red[0];
  if (s == 0) {
    d_params[0] += tot * double(tb.cm_coef);
  } else if (s < 1 + kMaxGates) {
    const int g = s - 1;
    if (g < tb.ng && tb.gate[g].last) d_params[1 + tb.gate[g].channel] += tot * double(tb.ndt_cm);
  } else {
    const int j = s - 1 - kMaxGates;
    if (j < tb.nleak) d_params[1 + tb.leak_ch[j]] += tot * double(tb.ndt_cm);
  }
}

// ------------------------------------------------------------ elementwise
template <typename T>
__global__ void k_rates(const DevTable<T> tb, int64_t n, const T* v, T* al, T* be) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    al[i] = scaled(tb, rate_val(tb.gate[0].al, v[i]));
    be[i] = scaled(tb, rate_val(tb.gate[0].be, v[i]));
  }
}

template <typename T>
__global__ void k_rate_eval(const DevRate<T> r, int slope, int64_t n, const T* v, T* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (slope) {
      T val, d;
      rate_val_slope(r, v[i], val, d);
      out[i] = d;
    } else {
      out[i] = rate_val(r, v[i]);
    }
  }
}

// gate_step (dynamics.py:335-346): p_inf = where(s > 0, a/s, p); p_inf + (p - p_inf) e
template <typename T>
__global__ void k_gate_step(int64_t n, const T* p, const T* al, const T* be, T dt, T* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T s = add_(al[i], be[i]);
    T pinf, e;
    if constexpr (sizeof(T) == 4) {
      pinf = (s > 0.0f) ? mul_(al[i], rcp_(s)) : p[i];
      e = ex2_(mul_(mul_(-dt, s), 1.4426950408889634f));
    } else {
      pinf = (s > 0.0) ? al[i] / s : p[i];
      e = exp(mul_(-dt, s));
    }
    out[i] = add_(pinf, mul_(sub_(p[i], pinf), e));
  }
}

// ionic_current (dynamics.py:360-376), channel order
template <typename T, int NG>
__global__ void k_ionic(const DevTable<T> tb, int64_t n, const T* v, const T* g, int64_t g_ld,
                        T* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T vi = v[i];
    T ion = leak_current(tb, vi);
    T eta = T(1);
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      const DevGate<T>& G = tb.gate[q];
      const T pk = ipow_(g[q * g_ld + i], G.k);
      eta = G.first ? pk : mul_(eta, pk);
      if (G.last) ion = leak_after(tb, G, vi, add_(ion, channel_term(G.g, G.e, eta, vi)));
    }
    out[i] = ion;
  }
}

template <typename T>
__global__ void k_spike_detect(int64_t n, const T* vp, const T* vn, T theta, uint8_t* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = (vp[i] < theta) && (vn[i] >= theta);
}

template <typename T>
__global__ void k_surrogate(const DevSur<T> s, int64_t n, const T* u, T* out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = surrogate(s, u[i]);
}

// ------------------------------------------------------------ stimulus
template <typename T>
__global__ void __launch_bounds__(256) k_poisson(int64_t n, int64_t steps, uint64_t seed,
                                                 int64_t nbase, int64_t tbase,
                                                 const PoissonTab<T> tab, T* out, int64_t ld) {
  // one thread = 4 consecutive neurons (one Philox block per step when the
  // global ids are 4-aligned), steps strided over gridDim.y; no early exit:
  // draw() votes across the warp
  __shared__ PoissonSmem<T> ps;
  ps.fill(tab);
  __syncthreads();
  const int64_t j0 = 4 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
  const bool aligned = (nbase & 3) == 0;
  const bool vec = aligned && j0 + 4 <= n && (ld & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) % (4 * sizeof(T))) == 0;
  for (int64_t t = blockIdx.y; t < steps; t += gridDim.y) {
    uint32_t w[4];
    if (aligned) {
      const uint4 r = Philox::block(seed, (nbase + j0) >> 2, tbase + t);
      w[0] = r.x;
      w[1] = r.y;
      w[2] = r.z;
      w[3] = r.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = Philox::word(seed, nbase + j0 + q, tbase + t);
    }
    T c[4];
    bool tail[4], any_tail = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      c[q] = ps.draw(w[q], tail[q]);
      any_tail = any_tail || tail[q];
    }
    if (__any_sync(0xffffffffu, any_tail)) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (tail[q]) c[q] = ps.tail_draw(w[q]);
    }
    T* row = out + t * ld + j0;
    if (vec) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(row) = make_float4(c[0], c[1], c[2], c[3]);
      } else {
        reinterpret_cast<double2*>(row)[0] = make_double2(c[0], c[1]);
        reinterpret_cast<double2*>(row)[1] = make_double2(c[2], c[3]);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (j0 + q < n) row[q] = c[q];
    }
  }
}

// bitmap row t -> one value per neuron (uint8 0/1 for Trace.spike_series, or
// float 0/1 for the SNN layer); grid.y strides the steps, grid.x the neurons
template <typename O>
__global__ void k_unpack(const uint32_t* bits, int64_t wld, int64_t steps, int64_t n, O* out, int64_t old) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t t = blockIdx.y; t < steps; t += gridDim.y)
    out[t * old + i] = O((bits[t * wld + (i >> 5)] >> (i & 31)) & 1u);
}

}  // namespace hhb
