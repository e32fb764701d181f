// Readout model plumbing either side of the HH point neuron:
// the single-output dendrite layer of learn.ReadoutModel (learn.py:238-247)
// and its weight gradient (learn.py:269-273).
//
//   hhb_readout_drive : drive[t][b] = bias + sum_c x(b,t,c) * w[c]
//                       written time-major, i.e. directly the i_series the
//                       HH forward / BPTT kernels read.
//   hhb_readout_grad  : d_w[c] = sum_{t,b} d_drive[t][b] * x(b,t,c),
//                       d_b    = sum_{t,b} d_drive[t][b]
//                       deterministic two-stage reduction (no atomics).
//
// x(b,t,c) lives at x[b*x_sb + t*x_st + c]: the reference's (B,T,C) layout
// (x_sb = T*C, x_st = C) and the time-major (T,B,C) one (x_sb = C,
// x_st = B*C) are both accepted without a copy.  HBM-bound GEMVs: one warp per
// (t,b) row for the drive (C contiguous -> coalesced), a C-wide x row-phase
// tile per block for the gradient.
#include <cstdint>

#include "hh_host.cuh"

using namespace hhb;

namespace {

constexpr int kGradBlocks = 296;   // 2 per SM; partial rows [kGradBlocks][C+1]
constexpr int kGradThreads = 256;
constexpr int64_t kMinRowsPerBlock = 128;

template <typename T>
__global__ void k_readout_drive(int64_t B, int64_t Tn, int64_t C, const T* __restrict__ x, int64_t sb, int64_t st,
                                const T* __restrict__ w, const T* __restrict__ bias, T* __restrict__ drive) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = B * Tn;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const int64_t t = r / B, b = r - t * B;   // r enumerates the time-major output
    const T* xr = x + b * sb + t * st;
    T acc = T(0);
    for (int64_t c = lane; c < C; c += 32) acc = fma(xr[c], w[c], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) drive[r] = acc + bias[0];
  }
}

// Stage 1: block g reduces rows [g*per, (g+1)*per) (time-major order) into
// part[g][0..C) and part[g][C] (the bias gradient).  Threads tile as
// (ty rows) x (tx columns); the ty partials are combined in a fixed order.
template <typename T>
__global__ void k_readout_grad_part(int64_t B, int64_t Tn, int64_t C, const T* __restrict__ x, int64_t sb,
                                    int64_t st, const T* __restrict__ dd, int64_t per, T* __restrict__ part) {
  extern __shared__ unsigned char smem_raw[];
  T* sh = reinterpret_cast<T*>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
  const int64_t rows = B * Tn;
  const int64_t r0 = int64_t(blockIdx.x) * per, r1 = r0 + per < rows ? r0 + per : rows;
  for (int64_t c0 = 0; c0 < C + 1; c0 += bx) {
    const int64_t c = c0 + tx;
    T acc = T(0);
    if (c <= C) {
      for (int64_t r = r0 + ty; r < r1; r += by) {
        const int64_t t = r / B, b = r - t * B;
        const T g = dd[r];
        acc = (c < C) ? fma(g, x[b * sb + t * st + c], acc) : acc + g;
      }
    }
    sh[ty * bx + tx] = acc;
    __syncthreads();
    if (ty == 0 && c <= C) {
      T s = sh[tx];
      for (int y = 1; y < by; ++y) s += sh[y * bx + tx];
      part[int64_t(blockIdx.x) * (C + 1) + c] = s;
    }
    __syncthreads();
  }
}

// Stage 2: one warp per column, lanes stride the block partials, fixed-order
// butterfly: deterministic for a given (rows, C).
template <typename T>
__global__ void k_readout_grad_sum(int64_t C, int nblk, const T* __restrict__ part, T* __restrict__ d_w,
                                   T* __restrict__ d_b) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t c = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); c <= C; c += warps) {
    T s = T(0);
    for (int g = lane; g < nblk; g += 32) s += part[int64_t(g) * (C + 1) + c];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (c < C) d_w[c] = s;
      else d_b[0] = s;
    }
  }
}

template <typename T>
int readout_grad(int64_t B, int64_t Tn, int64_t C, const void* x, int64_t sb, int64_t st, const void* dd, void* d_w,
                 void* d_b, void* ws, cudaStream_t s) {
  const int64_t rows = B * Tn;
  int64_t per = (rows + kGradBlocks - 1) / kGradBlocks;
  if (per < kMinRowsPerBlock) per = kMinRowsPerBlock;
  const int nblk = int((rows + per - 1) / per);
  int bx = 32;
  while (bx < C + 1 && bx < kGradThreads) bx <<= 1;
  const dim3 blk(bx, kGradThreads / bx);
  k_readout_grad_part<T><<<nblk, blk, sizeof(T) * kGradThreads, s>>>(B, Tn, C, (const T*)x, sb, st, (const T*)dd,
                                                                        per, (T*)ws);
  k_readout_grad_sum<T><<<unsigned((C + 1 + 7) / 8), 256, 0, s>>>(C, nblk, (const T*)ws, (T*)d_w, (T*)d_b);
  return cuda_check("k_readout_grad launch");
}

}  // namespace

extern "C" {

int64_t hhb_readout_workspace(int32_t dtype, int64_t n_in) {
  const int64_t es = dtype == HHB_F32 ? 4 : 8;
  return int64_t(kGradBlocks) * (n_in + 1) * es;
}

int hhb_readout_drive(int32_t dtype, int64_t batch, int64_t steps, int64_t n_in, const void* x, int64_t x_sb,
                      int64_t x_st, const void* w, const void* bias, void* drive, void* stream) {
  if (batch < 0 || steps < 0 || n_in < 0) return fail(HHB_EINVAL, "readout_drive: negative size");
  if (batch == 0 || steps == 0) return HHB_OK;
  if (!w || !bias || !drive || (n_in > 0 && !x)) return fail(HHB_EINVAL, "readout_drive: NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t rows = batch * steps;
  const unsigned grid = unsigned(rows / 8 + 1 < 148 * 16 ? rows / 8 + 1 : 148 * 16);
  if (dtype == HHB_F64)
    k_readout_drive<double><<<grid, 256, 0, st>>>(batch, steps, n_in, (const double*)x, x_sb, x_st, (const double*)w,
                                                  (const double*)bias, (double*)drive);
  else if (dtype == HHB_F32)
    k_readout_drive<float><<<grid, 256, 0, st>>>(batch, steps, n_in, (const float*)x, x_sb, x_st, (const float*)w,
                                                 (const float*)bias, (float*)drive);
  else
    return fail(HHB_EINVAL, "dtype");
  return cuda_check("k_readout_drive launch");
}

int hhb_readout_grad(int32_t dtype, int64_t batch, int64_t steps, int64_t n_in, const void* x, int64_t x_sb,
                     int64_t x_st, const void* d_drive, void* d_w, void* d_b, void* workspace, int64_t ws_bytes,
                     void* stream) {
  if (batch < 0 || steps < 0 || n_in < 0) return fail(HHB_EINVAL, "readout_grad: negative size");
  if (!d_w || !d_b) return fail(HHB_EINVAL, "readout_grad: NULL output");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t es = dtype == HHB_F32 ? 4 : 8;
  if (batch == 0 || steps == 0) {
    if (n_in > 0 && cudaMemsetAsync(d_w, 0, size_t(n_in * es), st) != cudaSuccess) return cuda_check("memset");
    if (cudaMemsetAsync(d_b, 0, size_t(es), st) != cudaSuccess) return cuda_check("memset");
    return HHB_OK;
  }
  if (!d_drive || (n_in > 0 && !x) || !workspace) return fail(HHB_EINVAL, "readout_grad: NULL pointer");
  if (ws_bytes < hhb_readout_workspace(dtype, n_in)) return fail(HHB_EINVAL, "readout_grad: workspace too small");
  if (dtype == HHB_F64) return readout_grad<double>(batch, steps, n_in, x, x_sb, x_st, d_drive, d_w, d_b, workspace, st);
  if (dtype == HHB_F32) return readout_grad<float>(batch, steps, n_in, x, x_sb, x_st, d_drive, d_w, d_b, workspace, st);
  return fail(HHB_EINVAL, "dtype");
}

}  // extern "C"
