// Throughput probe: scalar FFMA / FMUL vs packed FFMA2 / FMUL2 (sm_100a f32x2), and a
// mixed MUFU + FFMA2 stream.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/ffma2 tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 4096, CH = 8;
__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITER; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fmaf_rn(x[c], a, b);
  float s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[CH / 2];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int c = 0; c < CH / 2; ++c) x[c] = make_float2(threadIdx.x + 2 * c, threadIdx.x + 2 * c + 1);
  for (int i = 0; i < ITER; ++i)
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) x[c] = __ffma2_rn(x[c], A, B);
  float s = 0; for (int c = 0; c < CH / 2; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fmul(float* out, float a) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITER; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __fmul_rn(x[c], a);
  float s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fmul2(float* out, float a) {
  float2 x[CH / 2];
  const float2 A = make_float2(a, a);
  for (int c = 0; c < CH / 2; ++c) x[c] = make_float2(threadIdx.x + 2 * c, threadIdx.x + 2 * c + 1);
  for (int i = 0; i < ITER; ++i)
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) x[c] = __fmul2_rn(x[c], A);
  float s = 0; for (int c = 0; c < CH / 2; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// 1 MUFU.EX2 per 4 scalar FFMA (per chain), or per 2 FFMA2 (same flops)
__global__ void k_mix1(float* out, float a, float b) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITER / 4; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
      x[c] = __fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(y, a, b), a, b), a, b), a, b);
    }
  float s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix2(float* out, float a, float b) {
  float2 x[CH / 2];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int c = 0; c < CH / 2; ++c) x[c] = make_float2(threadIdx.x + 2 * c, threadIdx.x + 2 * c + 1);
  for (int i = 0; i < ITER / 4; ++i)
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) {
      float y0, y1;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(x[c].x));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(x[c].y));
      float2 y = make_float2(y0, y1);
      x[c] = __ffma2_rn(__ffma2_rn(__ffma2_rn(__ffma2_rn(y, A, B), A, B), A, B), A, B);
    }
  float s = 0; for (int c = 0; c < CH / 2; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// dependent-chain latency: one chain per thread, one warp per SM
__global__ void k_lat1(float* out, float a, float b, long long* clk) {
  float x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) x = __fmaf_rn(x, a, b);
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void k_lat2(float* out, float a, float b, long long* clk) {
  float2 x = make_float2(threadIdx.x, threadIdx.x + 1);
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  const long long t0 = clock64();
  for (int i = 0; i < ITER; ++i) x = __ffma2_rn(x, A, B);
  const long long t1 = clock64();
  out[threadIdx.x] = x.x + x.y;
  if (threadIdx.x == 0) clk[0] = t1 - t0;
}
template <class F>
void run(const char* name, F launch, double ops_per_thread, int blocks, int threads) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch();
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double tot = ops_per_thread * blocks * threads * 10;
  printf("%-8s %8.3f ms  %.3e fp32-op/s (%s)\n", name, ms / 10, tot / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  for (int thr : {256, 512}) {
    const int bl = 148 * (2048 / thr);
    printf("threads/SM 2048 (%d x %d)\n", bl, thr);
    run("ffma", [&] { k_ffma<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
    run("ffma2", [&] { k_ffma2<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
    run("fmul", [&] { k_fmul<<<bl, thr>>>(out, 0.999f); }, double(ITER) * CH, bl, thr);
    run("fmul2", [&] { k_fmul2<<<bl, thr>>>(out, 0.999f); }, double(ITER) * CH, bl, thr);
    run("mix1", [&] { k_mix1<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
    run("mix2", [&] { k_mix2<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
  }
  // low occupancy (4 warps per SMSP), like the HH kernels
  const int bl = 148 * 2, thr = 256;
  printf("threads/SM 512\n");
  run("ffma", [&] { k_ffma<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
  run("ffma2", [&] { k_ffma2<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
  run("mix1", [&] { k_mix1<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
  run("mix2", [&] { k_mix2<<<bl, thr>>>(out, 0.999f, 0.001f); }, double(ITER) * CH, bl, thr);
  long long* clk; cudaMallocManaged(&clk, 8);
  k_lat1<<<1, 32>>>(out, 0.999f, 0.001f, clk); cudaDeviceSynchronize();
  k_lat1<<<1, 32>>>(out, 0.999f, 0.001f, clk); cudaDeviceSynchronize();
  printf("FFMA dependent latency  %.2f clk\n", double(clk[0]) / ITER);
  k_lat2<<<1, 32>>>(out, 0.999f, 0.001f, clk); cudaDeviceSynchronize();
  k_lat2<<<1, 32>>>(out, 0.999f, 0.001f, clk); cudaDeviceSynchronize();
  printf("FFMA2 dependent latency %.2f clk\n", double(clk[0]) / ITER);
  return 0;
}
