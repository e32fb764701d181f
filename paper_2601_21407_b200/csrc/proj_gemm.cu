// proj_gemm.cu -- dense synaptic projection of the HH SNN layer on the 5th-gen
// tensor cores (DenseLayer learn.py:203-216, its gradient
// learn.py:264-274).
//
//   D[M][N] (fp32) = A[M][K] . B[N][K]^T (+ bias[N])      both operands K-major
//
// Forward  I = X W^T + b          : A = X  [T*B][K_in],   B = W   [N_out][K_in]
// dX       = dI W                 : A = dI [T*B][N_out],  B = W^T [K_in][N_out]
// dW       = dI^T X               : A = dI^T [N_out][T*B], B = X^T [K_in][T*B]
// (the transposes are produced by hhb_transpose; fp32 operands use kind::tf32).
//
// One CTA computes a 128 x BN tile: warp 0 (one lane) streams A/B k-blocks
// with TMA into a 4-stage ring of 128B-swizzled smem tiles, warp 1 (one lane)
// issues tcgen05.mma (M=128, N=BN, K=16 bf16 / 8 tf32) into a TMEM
// accumulator and releases smem stages with tcgen05.commit, warps 2-5 drain
// TMEM with tcgen05.ld (32 lanes x 32 columns each) and store fp32 rows.
// Split-K writes fp32 partial slices that hhb_gemm_reduce sums in a fixed
// order (deterministic).
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "hh_host.cuh"

namespace hhb {
namespace gemm {

constexpr int BM = 128;
constexpr int kThreads = 192;
// CTA-pair kernel: producer warp, MMA warp, EPI2_WARPS epilogue warps
#ifndef EPI2_WARPS
#define EPI2_WARPS 8
#endif
#ifndef EPI2_BUFS
#define EPI2_BUFS 1
#endif
constexpr int kThreads2 = 64 + 32 * EPI2_WARPS;

struct Args {
  int64_t M, N, K;
  float* D;
  int64_t ldd;
  const float* bias;
  int64_t split_stride;  // floats between split slices of D (0 when splits == 1)
  int kb_per_split;
  int kb_total;
  uint32_t idesc;
  int kb_switch;        // > 0 (K-major A, not DUAL): k-blocks >= kb_switch read A2 at k - kb_switch * 64
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int32_t x,
                                            int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand tile with 128B swizzle (TMA SWIZZLE_128B layout): rows of
// 128 B, 8-row atoms of 1024 B -> SBO = 1024 B, LBO unused (1), version 1.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t d = 0;
  d |= uint64_t((a & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

template <bool TF32>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                     uint32_t accumulate) {
  if constexpr (TF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// MN-major operand tile (bf16, SWIZZLE_128B): TMA boxes of 64 MN-elements x 64
// K-rows (8 KB), placed 8 KB apart along MN.  Canonical UMMA MN-major layout
// ((8,n),(8,k)) : ((1,LBO),(8,SBO)) in 16-byte units: LBO = 8192 B between
// 64-element MN chunks, SBO = 1024 B between 8-row K groups.
__device__ __forceinline__ uint64_t smem_desc_mn(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t d = 0;
  d |= uint64_t((a & 0x3FFFF) >> 4);
  d |= uint64_t(8192 >> 4) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

template <int BN, bool TF32, bool DUAL>
struct Cfg {
  static constexpr uint32_t kStageA = BM * 128;
  static constexpr uint32_t kStageB = BN * 128;
  static constexpr uint32_t kStage = kStageA * (DUAL ? 2 : 1) + kStageB;
  static constexpr int kStages = (200 * 1024) / kStage > 6 ? 6 : (200 * 1024) / kStage;
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + 256;
};

// D = sum_s A_s . B^T over the K range of this split; A_s = A (and A2 when DUAL:
// the bf16 hi and lo halves of an fp32 operand, accumulated into one TMEM
// tile).  A_MN / B_MN: operand stored MN-major ([K][M] / [K][N], MN
// contiguous) -- the natural layout of dI^T, X and W^T in the layer gradients,
// so no transposed copy is ever made.
template <int BN, bool TF32, bool A_MN, bool B_MN, bool DUAL>
__global__ void __launch_bounds__(kThreads, 1)
    k_umma_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                const __grid_constant__ CUtensorMap tb, const Args args) {
  using C = Cfg<BN, TF32, DUAL>;
  constexpr int STAGES_ = C::kStages;
  constexpr uint32_t kStageA = C::kStageA;
  constexpr uint32_t kStageB = C::kStageB;
  constexpr int kUmmaK = TF32 ? 8 : 16;                // elements per MMA
  constexpr int kBK = TF32 ? 32 : 64;                  // elements per 128 B row
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // [stage][A (, A2)]
  uint8_t* sB = smem + STAGES_ * kStageA * (DUAL ? 2 : 1);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES_ * kStageB);
  uint64_t* empty = full + STAGES_;
  uint64_t* tmem_full = empty + STAGES_;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
  constexpr uint32_t kAStride = kStageA * (DUAL ? 2 : 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
  const int kb0 = blockIdx.z * args.kb_per_split;
  const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
  const int nkb = max(0, kb1 - kb0);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    if (DUAL) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    for (int s = 0; s < STAGES_; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(uint32_t(BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  pdl_wait();       // the prologue above overlaps the predecessor's tail (pdl.cuh)
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES_;
        const uint32_t ph = (i / STAGES_) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], kStageA * (DUAL ? 2 : 1) + kStageB);
        const int32_t kx = (kb0 + i) * kBK;
        uint8_t* a_dst = sA + s * kAStride;
        if (A_MN) {
#pragma unroll
          for (int c = 0; c < BM / 64; ++c) {
            tma_load_2d(&ta, &full[s], a_dst + c * 8192, int32_t(m0) + 64 * c, kx);
            if (DUAL) tma_load_2d(&ta2, &full[s], a_dst + kStageA + c * 8192, int32_t(m0) + 64 * c, kx);
          }
        } else if (!DUAL && args.kb_switch > 0 && kb0 + i >= args.kb_switch) {
          tma_load_2d(&ta2, &full[s], a_dst, kx - args.kb_switch * kBK, int32_t(m0));
        } else {
          tma_load_2d(&ta, &full[s], a_dst, kx, int32_t(m0));
          if (DUAL) tma_load_2d(&ta2, &full[s], a_dst + kStageA, kx, int32_t(m0));
        }
        if (B_MN) {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(&tb, &full[s], sB + s * kStageB + c * 8192, int32_t(n0) + 64 * c, kx);
        } else {
          tma_load_2d(&tb, &full[s], sB + s * kStageB, kx, int32_t(n0));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = args.idesc;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES_;
        const uint32_t ph = (i / STAGES_) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* a_src = sA + s * kAStride;
        const uint8_t* b_src = sB + s * kStageB;
#pragma unroll
        for (int k = 0; k < kBK / kUmmaK; ++k) {
          const uint64_t bd = B_MN ? smem_desc_mn(b_src + k * 2048) : smem_desc(b_src + k * 32);
          const uint64_t ad = A_MN ? smem_desc_mn(a_src + k * 2048) : smem_desc(a_src + k * 32);
          umma<TF32>(tmem, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
          if (DUAL) {
            const uint64_t ad2 = A_MN ? smem_desc_mn(a_src + kStageA + k * 2048) : smem_desc(a_src + kStageA + k * 32);
            umma<TF32>(tmem, ad2, bd, idesc, 1u);
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {  // epilogue warps 2..5: TMEM lane quarter = warp % 4
    const int q = warp & 3;
    const int64_t row = m0 + q * 32 + lane;
    float* drow = args.D + int64_t(blockIdx.z) * args.split_stride + row * args.ldd;
    const bool add_bias = args.bias != nullptr && args.split_stride == 0;
    if (nkb > 0) {
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      if (nkb > 0) {
        tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c0), r);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      if (row < args.M) {
        const int64_t cb = n0 + c0;
        const bool vec = (cb + 32 <= args.N) && ((args.ldd & 3) == 0) &&
                         ((reinterpret_cast<uintptr_t>(drow) & 15) == 0);
        if (vec) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o;
            o.x = __uint_as_float(r[j + 0]) + (add_bias ? __ldg(args.bias + cb + j + 0) : 0.f);
            o.y = __uint_as_float(r[j + 1]) + (add_bias ? __ldg(args.bias + cb + j + 1) : 0.f);
            o.z = __uint_as_float(r[j + 2]) + (add_bias ? __ldg(args.bias + cb + j + 2) : 0.f);
            o.w = __uint_as_float(r[j + 3]) + (add_bias ? __ldg(args.bias + cb + j + 3) : 0.f);
            *reinterpret_cast<float4*>(drow + cb + j) = o;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb + j < args.N)
              drow[cb + j] = __uint_as_float(r[j]) + (add_bias ? __ldg(args.bias + cb + j) : 0.f);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(BN)));
  }
}

// ---------------------------------------------------------------- persistent
// Persistent variant: one CTA per SM walks the tile list (tile = blockIdx.x,
// + gridDim.x, ...).  The accumulator is double-buffered in tensor memory
// (2 x BN columns), so the MMA warp starts tile i+1 while the epilogue warps
// drain tile i; the epilogue stages 32x32 fp32 blocks in 128B-swizzled shared
// memory and writes them with TMA bulk-tensor stores (full 128-byte lines,
// asynchronous), instead of per-thread row stores.
template <int BN, bool DUAL>
struct PCfg {
  static constexpr uint32_t kStageA = BM * 128;
  static constexpr uint32_t kStageB = BN * 128;
  static constexpr uint32_t kStage = kStageA * (DUAL ? 2 : 1) + kStageB;
  static constexpr uint32_t kStaging = 4 * 2 * 32 * 32 * 4;   // 4 warps x 2 buffers x 32x32 fp32
  static constexpr int kStages = int((225 * 1024 - kStaging) / kStage) > 6 ? 6 : int((225 * 1024 - kStaging) / kStage);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + kStaging + 256;
};

struct PArgs {
  int64_t M, N;
  int m_tiles, n_tiles, splits, tiles;
  int kb_per_split, kb_total;
  uint32_t idesc;
  const float* bias;   // only when splits == 1
  int kb_switch;       // > 0 (K-major A, not DUAL): k-blocks >= kb_switch read A2 at k - kb_switch * 64
  // fp32-A GEMM only: the on-chip bf16 conversion of A also written out (hi at
  // xs[m][k], lo at xs[m][xs_slot + k]; null = not written)
  uint16_t* xs;
  int64_t xs_ld, xs_slot, K;
  int n_fast;          // tile order: 1 = column tiles fastest (pairs on one row block run together), 0 = rows fastest
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int32_t x, int32_t y,
                                             int32_t z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}

template <int BN, bool A_MN, bool B_MN, bool DUAL>
__global__ void __launch_bounds__(kThreads, 1)
    k_umma_gemm_p(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                  const __grid_constant__ CUtensorMap tb, const __grid_constant__ CUtensorMap td, const PArgs args) {
  using C = PCfg<BN, DUAL>;
  constexpr int ST = C::kStages;
  constexpr uint32_t kStageA = C::kStageA, kStageB = C::kStageB;
  constexpr uint32_t kAStride = kStageA * (DUAL ? 2 : 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * kAStride;
  float* stg = reinterpret_cast<float*>(sB + ST * kStageB);          // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + C::kStaging);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;      // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    if (DUAL) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&td)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  pdl_wait();       // the prologue above overlaps the predecessor's tail (pdl.cuh)
  pdl_trigger();
  const int per_split = args.m_tiles * args.n_tiles;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int it = 0;
      for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
        const int z = tile / per_split, r = tile % per_split;
        const int64_t m0 = int64_t(args.n_fast ? r / args.n_tiles : r % args.m_tiles) * BM;
        const int64_t n0 = int64_t(args.n_fast ? r % args.n_tiles : r / args.m_tiles) * BN;
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          mbar_expect_tx(&full[s], kAStride + kStageB);
          const int32_t kx = kb * 64;
          uint8_t* a_dst = sA + s * kAStride;
          if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) {
              tma_load_2d(&ta, &full[s], a_dst + c * 8192, int32_t(m0) + 64 * c, kx);
              if (DUAL) tma_load_2d(&ta2, &full[s], a_dst + kStageA + c * 8192, int32_t(m0) + 64 * c, kx);
            }
          } else if (!DUAL && args.kb_switch > 0 && kb >= args.kb_switch) {
            tma_load_2d(&ta2, &full[s], a_dst, kx - args.kb_switch * 64, int32_t(m0));
          } else {
            tma_load_2d(&ta, &full[s], a_dst, kx, int32_t(m0));
            if (DUAL) tma_load_2d(&ta2, &full[s], a_dst + kStageA, kx, int32_t(m0));
          }
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(&tb, &full[s], sB + s * kStageB + c * 8192, int32_t(n0) + 64 * c, kx);
          } else {
            tma_load_2d(&tb, &full[s], sB + s * kStageB, kx, int32_t(n0));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x, ++local) {
        const int z = tile / per_split;
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int b = local & 1;
        mbar_wait(&tempty[b], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + uint32_t(b * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* a_src = sA + s * kAStride;
          const uint8_t* b_src = sB + s * kStageB;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = B_MN ? smem_desc_mn(b_src + k * 2048) : smem_desc(b_src + k * 32);
            const uint64_t ad = A_MN ? smem_desc_mn(a_src + k * 2048) : smem_desc(a_src + k * 32);
            umma<false>(acc, ad, bd, args.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            if (DUAL) {
              const uint64_t ad2 =
                  A_MN ? smem_desc_mn(a_src + kStageA + k * 2048) : smem_desc(a_src + kStageA + k * 32);
              umma<false>(acc, ad2, bd, args.idesc, 1u);
            }
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[b]);
      }
    }
  } else {  // epilogue warps 2..5: TMEM lane quarter q = warp % 4
    const int q = warp & 3;
    float* my_stg = stg + (warp - 2) * 2 * 1024;
    int local = 0, nstore = 0;
    for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x, ++local) {
      const int z = tile / per_split, r = tile % per_split;
      const int64_t m0 = int64_t(args.n_fast ? r / args.n_tiles : r % args.m_tiles) * BM;
      const int64_t n0 = int64_t(args.n_fast ? r % args.n_tiles : r / args.m_tiles) * BN;
      const int kb0 = z * args.kb_per_split;
      const bool any_k = min(args.kb_total, kb0 + args.kb_per_split) > kb0;
      const int b = local & 1;
      mbar_wait(&tfull[b], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int32_t row0 = int32_t(m0 + q * 32);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        if (n0 + c0 >= args.N) break;
        uint32_t rr[32];
        if (any_k) {
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * BN + c0), rr);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = 0u;
        }
        float* buf = my_stg + (nstore & 1) * 1024;
        // the store that last used this buffer must have finished reading it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        // row `lane` of the 32x32 block, 16-byte chunks XOR-swizzled by row % 8
        // bias of the chunk's 32 columns (the same for every row / lane):
        // float4 loads when the chunk is full and aligned, else per element
        const bool bvec = args.bias != nullptr && n0 + c0 + 32 <= args.N &&
                          (reinterpret_cast<uintptr_t>(args.bias + n0 + c0) & 15) == 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o;
          const int64_t cb = n0 + c0 + 4 * j;
          o.x = __uint_as_float(rr[4 * j + 0]);
          o.y = __uint_as_float(rr[4 * j + 1]);
          o.z = __uint_as_float(rr[4 * j + 2]);
          o.w = __uint_as_float(rr[4 * j + 3]);
          if (bvec) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(args.bias + cb));
            o.x += bb.x;
            o.y += bb.y;
            o.z += bb.z;
            o.w += bb.w;
          } else if (args.bias != nullptr) {
            o.x += cb + 0 < args.N ? __ldg(args.bias + cb + 0) : 0.f;
            o.y += cb + 1 < args.N ? __ldg(args.bias + cb + 1) : 0.f;
            o.z += cb + 2 < args.N ? __ldg(args.bias + cb + 2) : 0.f;
            o.w += cb + 3 < args.N ? __ldg(args.bias + cb + 3) : 0.f;
          }
          *reinterpret_cast<float4*>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&td, buf, int32_t(n0 + c0), row0, z);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++nstore;
      }
      // all TMEM reads of this accumulator are complete (tcgen05.ld waited)
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(2 * BN)));
  }
}

// ---------------------------------------------------------------- CTA pair
// 2-SM variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x BN tile.  Each CTA loads its own 128 rows of A and half (BN/2) of the
// columns of B; the leader (rank 0) issues tcgen05.mma.cta_group::2 (M = 256),
// which reads B from both CTAs' shared memory, and each CTA's tensor memory
// holds the accumulator of its 128 rows.  Per SM that halves the shared-memory
// traffic of the operands (a 1-SM 128x256 tile needs ~192 B/clk of smem at
// tensor peak against 128 B/clk available; the pair needs ~128).
// Synchronisation: both CTAs' TMA loads complete on the LEADER's full barrier
// (expect_tx = both halves, two arrivals); the leader's commits multicast to
// both CTAs' empty / tmem-full barriers; the peer's epilogue warps arrive on
// the leader's tmem-empty barrier (8 arrivals).
template <int BN, bool DUAL>
struct P2Cfg {
  static constexpr uint32_t kStageA = BM * 128;             // this CTA's 128 rows x 64 k
  static constexpr uint32_t kStageB = (BN / 2) * 128;       // half of B
  static constexpr uint32_t kStage = kStageA * (DUAL ? 2 : 1) + kStageB;
  static constexpr int kEpiWarps = EPI2_WARPS;                // 2 per TMEM lane quadrant, each half of the columns
  static constexpr int kStgBufs = EPI2_BUFS;                  // TMA-store staging buffers per epilogue warp
  static constexpr uint32_t kStaging = kEpiWarps * kStgBufs * 32 * 32 * 4;
#ifndef GEMM2_MAX_STAGES
#define GEMM2_MAX_STAGES 8
#endif
  static constexpr int kStages = int((225 * 1024 - kStaging) / kStage) > GEMM2_MAX_STAGES
                                     ? GEMM2_MAX_STAGES
                                     : int((225 * 1024 - kStaging) / kStage);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + kStaging + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion goes to the pair leader's mbarrier (bit 24 of a
// shared::cluster address selects the odd CTA of the pair)
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* map, uint64_t* bar, void* dst, int32_t x,
                                                int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                      uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

template <int BN, bool A_MN, bool B_MN, bool DUAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    k_umma_gemm_2sm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                    const __grid_constant__ CUtensorMap tb, const __grid_constant__ CUtensorMap td, const PArgs args) {
  using C = P2Cfg<BN, DUAL>;
  constexpr int ST = C::kStages;
  constexpr uint32_t kStageA = C::kStageA, kStageB = C::kStageB;
  constexpr uint32_t kAStride = kStageA * (DUAL ? 2 : 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * kAStride;
  float* stg = reinterpret_cast<float*>(sB + ST * kStageB);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + C::kStaging);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;      // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    if (DUAL) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&td)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * C::kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  pdl_wait();       // the prologue above overlaps the predecessor's tail (pdl.cuh)
  pdl_trigger();
  const int per_split = args.m_tiles * args.n_tiles;      // m_tiles counts 256-row pair tiles
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own A rows, own half of B
      int it = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs) {
        const int z = tile / per_split, r = tile % per_split;
        const int64_t m0 = int64_t(args.n_fast ? r / args.n_tiles : r % args.m_tiles) * (2 * BM) + int64_t(rank) * BM;
        const int64_t n0 = int64_t(args.n_fast ? r % args.n_tiles : r / args.m_tiles) * BN + int64_t(rank) * (BN / 2);
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          if (leader) mbar_expect_tx_only(&full[s], 2 * (kAStride + kStageB));
          else mbar_arrive_leader(&full[s]);
          const int32_t kx = kb * 64;
          uint8_t* a_dst = sA + s * kAStride;
          if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) {
              tma_load_2d_2sm(&ta, &full[s], a_dst + c * 8192, int32_t(m0) + 64 * c, kx);
              if (DUAL) tma_load_2d_2sm(&ta2, &full[s], a_dst + kStageA + c * 8192, int32_t(m0) + 64 * c, kx);
            }
          } else if (!DUAL && args.kb_switch > 0 && kb >= args.kb_switch) {
            tma_load_2d_2sm(&ta2, &full[s], a_dst, kx - args.kb_switch * 64, int32_t(m0));
          } else {
            tma_load_2d_2sm(&ta, &full[s], a_dst, kx, int32_t(m0));
            if (DUAL) tma_load_2d_2sm(&ta2, &full[s], a_dst + kStageA, kx, int32_t(m0));
          }
          if (B_MN) {
#pragma unroll
            for (int c = 0; c < (BN / 2) / 64; ++c)
              tma_load_2d_2sm(&tb, &full[s], sB + s * kStageB + c * 8192, int32_t(n0) + 64 * c, kx);
          } else {
            tma_load_2d_2sm(&tb, &full[s], sB + s * kStageB, kx, int32_t(n0));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer: the pair leader only
      int it = 0, local = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
        const int z = tile / per_split;
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int b = local & 1;
        mbar_wait(&tempty[b], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + uint32_t(b * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* a_src = sA + s * kAStride;
          const uint8_t* b_src = sB + s * kStageB;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = B_MN ? smem_desc_mn(b_src + k * 2048) : smem_desc(b_src + k * 32);
            const uint64_t ad = A_MN ? smem_desc_mn(a_src + k * 2048) : smem_desc(a_src + k * 32);
            umma2(acc, ad, bd, args.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            if (DUAL) {
              const uint64_t ad2 =
                  A_MN ? smem_desc_mn(a_src + kStageA + k * 2048) : smem_desc(a_src + kStageA + k * 32);
              umma2(acc, ad2, bd, args.idesc, 1u);
            }
          }
          umma2_commit(&empty[s]);
        }
        umma2_commit(&tfull[b]);
      }
    }
  } else {  // epilogue warps of both CTAs: this CTA's 128 rows; warp w reads TMEM lane quadrant w % 4
    const int q = warp & 3;
    const int half = C::kEpiWarps == 8 ? (warp - 2) >> 2 : 0;    // which half of the tile's columns
    constexpr int kCols = C::kEpiWarps == 8 ? BN / 2 : BN;
    float* my_stg = stg + (warp - 2) * C::kStgBufs * 1024;
    int local = 0, nstore = 0;
    for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
      const int z = tile / per_split, r = tile % per_split;
      const int64_t m0 = int64_t(args.n_fast ? r / args.n_tiles : r % args.m_tiles) * (2 * BM) + int64_t(rank) * BM;
      const int64_t n0 = int64_t(args.n_fast ? r % args.n_tiles : r / args.m_tiles) * BN;
      const int kb0 = z * args.kb_per_split;
      const bool any_k = min(args.kb_total, kb0 + args.kb_per_split) > kb0;
      const int b = local & 1;
      mbar_wait(&tfull[b], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int32_t row0 = int32_t(m0 + q * 32);
#pragma unroll 1
      for (int c0 = half * kCols; c0 < (half + 1) * kCols; c0 += 32) {
        if (n0 + c0 >= args.N) break;
        uint32_t rr[32];
        if (any_k) {
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * BN + c0), rr);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = 0u;
        }
        float* buf = my_stg + (nstore % C::kStgBufs) * 1024;
        // the store that last used this buffer (kStgBufs stores ago) must have read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(C::kStgBufs - 1) : "memory");
        __syncwarp();
        // bias of the chunk's 32 columns (the same for every row / lane):
        // float4 loads when the chunk is full and aligned, else per element
        const bool bvec = args.bias != nullptr && n0 + c0 + 32 <= args.N &&
                          (reinterpret_cast<uintptr_t>(args.bias + n0 + c0) & 15) == 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o;
          const int64_t cb = n0 + c0 + 4 * j;
          o.x = __uint_as_float(rr[4 * j + 0]);
          o.y = __uint_as_float(rr[4 * j + 1]);
          o.z = __uint_as_float(rr[4 * j + 2]);
          o.w = __uint_as_float(rr[4 * j + 3]);
          if (bvec) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(args.bias + cb));
            o.x += bb.x;
            o.y += bb.y;
            o.z += bb.z;
            o.w += bb.w;
          } else if (args.bias != nullptr) {
            o.x += cb + 0 < args.N ? __ldg(args.bias + cb + 0) : 0.f;
            o.y += cb + 1 < args.N ? __ldg(args.bias + cb + 1) : 0.f;
            o.z += cb + 2 < args.N ? __ldg(args.bias + cb + 2) : 0.f;
            o.w += cb + 3 < args.N ? __ldg(args.bias + cb + 3) : 0.f;
          }
          *reinterpret_cast<float4*>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&td, buf, int32_t(n0 + c0), row0, z);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++nstore;
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[b]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(2 * BN)));
  }
}

// ---------------------------------------------------------------- fp32 A, converted on chip
// CTA-pair GEMM whose A operand is fp32 in global memory (the layer input x):
// TMA brings each CTA's 128 x 64 fp32 tile (two 128B-swizzled boxes of 32
// columns) into shared memory, four converter warps round it to bf16 in place
// (SPLIT: bf16 hi into the first half and lo = x - hi into the second), in the
// K-major 128B-swizzled layout the MMA reads, and signal the pair leader; the
// leader's MMAs are then those of the bf16 kernel (SPLIT: hi.B + lo.B + hi.B2,
// B = W_hi, B2 = W_lo -- the fp32-class product of proj="bf16x3").  Replaces the
// separate cast / split pass over x (read 4 B + write 2-6 B per element) by the
// GEMM's own 4-byte read; the products and their order are those of the
// unfused path, so D is bit-identical to it.
template <int BN, bool SPLIT>
struct PCvtCfg {
  static constexpr uint32_t kStageF = BM * 64 * 4;           // 128 rows x 64 fp32 (-> bf16 hi [+ lo] in place)
  static constexpr uint32_t kStageB = (BN / 2) * 128;        // half of B (and of B2)
  static constexpr uint32_t kStage = kStageF + kStageB * (SPLIT ? 2 : 1);
  static constexpr int kEpiWarps = EPI2_WARPS;
#ifndef CVT_WARPS
#define CVT_WARPS 8   // single-product form: 8 converter warps (66.7 vs 77.6 us at config 3; tools/cvt_check.py)
#endif
#ifndef CVT_SPLIT_WARPS
#define CVT_SPLIT_WARPS 4   // three-product form: 8 measured the same (107.2 vs 106.9 us)
#endif
  static constexpr int kCvtWarps = SPLIT ? CVT_SPLIT_WARPS : CVT_WARPS;
  static constexpr int kJobs = 1024 / (32 * kCvtWarps);    // 16-byte output chunks per converter thread
  static constexpr int kThreads = 64 + 32 * (kEpiWarps + kCvtWarps);
  static constexpr uint32_t kStaging = kEpiWarps * 32 * 32 * 4;
  static constexpr int kStages = int((225 * 1024 - kStaging) / kStage) > 6 ? 6 : int((225 * 1024 - kStaging) / kStage);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + kStaging + 512;
};

template <int W>
__device__ __forceinline__ void cvt_bar_sync() {   // the converter warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;" ::"n"(32 * W) : "memory");
}

template <int BN, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PCvtCfg<BN, SPLIT>::kThreads, 1)
    k_umma_gemm_2sm_cvt(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                        const __grid_constant__ CUtensorMap tb2, const __grid_constant__ CUtensorMap td,
                        const __grid_constant__ CUtensorMap txh, const __grid_constant__ CUtensorMap txl,
                        const PArgs args) {
  using C = PCvtCfg<BN, SPLIT>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sF = smem;                                   // [ST][kStageF]
  uint8_t* sB = smem + ST * C::kStageF;                 // [ST][kStageB (x2 with SPLIT)]
  constexpr uint32_t kBStride = C::kStageB * (SPLIT ? 2 : 1);
  float* stg = reinterpret_cast<float*>(sB + ST * kBStride);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + C::kStaging);
  uint64_t* afull = full + ST;
  uint64_t* cfull = afull + ST;
  uint64_t* empty = cfull + ST;
  uint64_t* tfull = empty + ST;      // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    if (SPLIT) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&td)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 2);      // B: the leader's expect_tx + the peer's arrival
      mbar_init(&afull[s], 1);     // this CTA's fp32 A tile
      mbar_init(&cfull[s], 2);     // both CTAs' converted A tiles
      mbar_init(&empty[s], 2);     // the MMA's commit + this CTA's converter (its x store has read the stage)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * C::kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  // tile order: column tiles fastest -- the pairs on one 256-row block of x run
  // together, so its fp32 tile comes from HBM once and from L2 for the others
  const int per_split = args.m_tiles * args.n_tiles;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr int kCvt0 = 2 + C::kEpiWarps;               // first converter warp

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own fp32 A rows, own half of B (and B2)
      int it = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs) {
        const int z = tile / per_split, r = tile % per_split;
        const int64_t m0 = int64_t(r / args.n_tiles) * (2 * BM) + int64_t(rank) * BM;
        const int64_t n0 = int64_t(r % args.n_tiles) * BN + int64_t(rank) * (BN / 2);
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          const int32_t kx = kb * 64;
          uint8_t* f_dst = sF + s * C::kStageF;
          mbar_expect_tx(&afull[s], C::kStageF);
          tma_load_2d(&ta, &afull[s], f_dst, kx, int32_t(m0));
          tma_load_2d(&ta, &afull[s], f_dst + C::kStageF / 2, kx + 32, int32_t(m0));
          if (leader) mbar_expect_tx_only(&full[s], 2 * kBStride);
          else mbar_arrive_leader(&full[s]);
          uint8_t* b_dst = sB + s * kBStride;
          tma_load_2d_2sm(&tb, &full[s], b_dst, kx, int32_t(n0));
          if (SPLIT) tma_load_2d_2sm(&tb2, &full[s], b_dst + C::kStageB, kx, int32_t(n0));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer: the pair leader only
      int it = 0, local = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
        const int z = tile / per_split;
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int b = local & 1;
        mbar_wait(&tempty[b], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + uint32_t(b * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          mbar_wait(&cfull[s], (it / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* a_src = sF + s * C::kStageF;
          const uint8_t* b_src = sB + s * kBStride;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc(a_src + k * 32);
            const uint64_t bd = smem_desc(b_src + k * 32);
            umma2(acc, ad, bd, args.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            if (SPLIT) {
              umma2(acc, smem_desc(a_src + C::kStageF / 2 + k * 32), bd, args.idesc, 1u);     // lo . W_hi
              umma2(acc, ad, smem_desc(b_src + C::kStageB + k * 32), args.idesc, 1u);         // hi . W_lo
            }
          }
          umma2_commit(&empty[s]);
        }
        umma2_commit(&tfull[b]);
      }
    }
  } else if (warp >= kCvt0) {  // converter warps: fp32 tile -> bf16 (hi [, lo]) in place
    const int ct = threadIdx.x - kCvt0 * 32;            // 0..127
    int it = 0, pend = -1;                              // pend: stage whose x store may still be reading
    for (int tile = pair; tile < args.tiles; tile += npairs) {
      const int z = tile / per_split, rt = tile % per_split;
      const bool xs_out = args.xs != nullptr && rt % args.n_tiles == 0;
      const int64_t xm0 = int64_t(rt / args.n_tiles) * (2 * BM) + int64_t(rank) * BM;
      const int kb0 = z * args.kb_per_split;
      const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % ST;
        uint8_t* f = sF + s * C::kStageF;
        mbar_wait(&afull[s], (it / ST) & 1);
        // job q: row r = j / 8, 8-column chunk c = j % 8 (8 lanes per row: each
        // quarter-warp reads one 128 B row of a swizzled box, conflict-free)
        float x[C::kJobs][8];
#pragma unroll
        for (int q = 0; q < C::kJobs; ++q) {
          const int j = ct + 32 * C::kCvtWarps * q, r = j >> 3, c = j & 7;
          const uint8_t* box = f + (c >> 2) * (C::kStageF / 2) + r * 128;
          const int j0 = (2 * (c & 3)) ^ (r & 7), j1 = (2 * (c & 3) + 1) ^ (r & 7);
          const float4 u = *reinterpret_cast<const float4*>(box + j0 * 16);
          const float4 w = *reinterpret_cast<const float4*>(box + j1 * 16);
          x[q][0] = u.x; x[q][1] = u.y; x[q][2] = u.z; x[q][3] = u.w;
          x[q][4] = w.x; x[q][5] = w.y; x[q][6] = w.z; x[q][7] = w.w;
        }
        cvt_bar_sync<C::kCvtWarps>();                    // every fp32 value read before the tile is overwritten
#pragma unroll
        for (int q = 0; q < C::kJobs; ++q) {
          const int j = ct + 32 * C::kCvtWarps * q, r = j >> 3, c = j & 7;
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 hb = __floats2bfloat162_rn(x[q][2 * e], x[q][2 * e + 1]);
            h[e] = *reinterpret_cast<const uint32_t*>(&hb);
            if (SPLIT) {
              const float2 hf = __bfloat1622float2(hb);
              const __nv_bfloat162 lb =
                  __floats2bfloat162_rn(__fsub_rn(x[q][2 * e], hf.x), __fsub_rn(x[q][2 * e + 1], hf.y));
              l[e] = *reinterpret_cast<const uint32_t*>(&lb);
            }
          }
          const int off = r * 128 + ((c ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(f + off) = make_uint4(h[0], h[1], h[2], h[3]);
          if (SPLIT) *reinterpret_cast<uint4*>(f + C::kStageF / 2 + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> the MMA's async reads
        cvt_bar_sync<C::kCvtWarps>();
        if (ct == 0) {
          mbar_arrive_leader(&cfull[s]);
          // the previous stage's x store (if any) has had a whole conversion to read
          // its tile: release that stage now, then start this stage's store
          if (pend >= 0) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            mbar_arrive_local(&empty[pend]);
            pend = -1;
          }
          if (xs_out) {   // the converted operand for the weight gradient (first column tile only), by TMA
            tma_store_2d(&txh, f, kb * 64, int32_t(xm0));
            if (SPLIT) tma_store_2d(&txl, f + C::kStageF / 2, kb * 64, int32_t(xm0));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            pend = s;
          } else {
            mbar_arrive_local(&empty[s]);   // the stage may be reloaded once the MMA has also committed
          }
        }
      }
    }
    if (ct == 0 && pend >= 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      mbar_arrive_local(&empty[pend]);
    }
  } else {  // epilogue warps of both CTAs (as k_umma_gemm_2sm)
    const int q = warp & 3;
    const int half = C::kEpiWarps == 8 ? (warp - 2) >> 2 : 0;
    constexpr int kCols = C::kEpiWarps == 8 ? BN / 2 : BN;
    float* my_stg = stg + (warp - 2) * 1024;
    int local = 0;
    for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
      const int z = tile / per_split, r = tile % per_split;
      const int64_t m0 = int64_t(r / args.n_tiles) * (2 * BM) + int64_t(rank) * BM;
      const int64_t n0 = int64_t(r % args.n_tiles) * BN;
      const int kb0 = z * args.kb_per_split;
      const bool any_k = min(args.kb_total, kb0 + args.kb_per_split) > kb0;
      const int b = local & 1;
      mbar_wait(&tfull[b], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int32_t row0 = int32_t(m0 + q * 32);
#pragma unroll 1
      for (int c0 = half * kCols; c0 < (half + 1) * kCols; c0 += 32) {
        if (n0 + c0 >= args.N) break;
        uint32_t rr[32];
        if (any_k) {
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * BN + c0), rr);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = 0u;
        }
        float* buf = my_stg;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        const bool bvec = args.bias != nullptr && n0 + c0 + 32 <= args.N &&
                          (reinterpret_cast<uintptr_t>(args.bias + n0 + c0) & 15) == 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o;
          const int64_t cb = n0 + c0 + 4 * j;
          o.x = __uint_as_float(rr[4 * j + 0]);
          o.y = __uint_as_float(rr[4 * j + 1]);
          o.z = __uint_as_float(rr[4 * j + 2]);
          o.w = __uint_as_float(rr[4 * j + 3]);
          if (bvec) {
            const float4 bb = __ldg(reinterpret_cast<const float4*>(args.bias + cb));
            o.x += bb.x;
            o.y += bb.y;
            o.z += bb.z;
            o.w += bb.w;
          } else if (args.bias != nullptr) {
            o.x += cb + 0 < args.N ? __ldg(args.bias + cb + 0) : 0.f;
            o.y += cb + 1 < args.N ? __ldg(args.bias + cb + 1) : 0.f;
            o.z += cb + 2 < args.N ? __ldg(args.bias + cb + 2) : 0.f;
            o.w += cb + 3 < args.N ? __ldg(args.bias + cb + 3) : 0.f;
          }
          *reinterpret_cast<float4*>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&td, buf, int32_t(n0 + c0), row0, z);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[b]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(2 * BN)));
  }
}

// Weight-gradient form of the on-chip split: D[m][n] = sum_k (A + A2)[k][m] . B_hi[k][n]
// + A[k][m] . B_lo[k][n] with A / A2 the bf16 hi / lo halves of dI (MN-major)
// and B the fp32 layer input x, MN-major (x[k][n], k = the (t, b) row), rounded
// and split into bf16 hi / lo on chip by the converter warps in the MN-major
// 128B-swizzled layout (64-column chunks of 64 k-rows x 128 B).  The
// three-product fp32-class dW of proj="bf16x3" in one GEMM, reading x in fp32
// -- so the forward projection need not write x_hi / x_lo.
// SPLIT = false: x rounded to bf16 only, D = sum_k (A + A2)[k][m] . bf16(B)[k][n]
// (the dW of proj="bf16", two products per k-step).
template <bool SPLIT>
struct PCvtbCfg {
  static constexpr int kEpiWarps = EPI2_WARPS;
  static constexpr int kCvtWarps = SPLIT ? CVT_SPLIT_WARPS : CVT_WARPS;
  static constexpr int kThreads = 64 + 32 * (kEpiWarps + kCvtWarps);
  static constexpr int kJobs = 1024 / (32 * kCvtWarps);
  static constexpr uint32_t kStage = 64 * 1024;           // fp32 x (32 KB) + A hi / lo (2 x 16 KB)
  static constexpr uint32_t kStaging = kEpiWarps * 32 * 32 * 4;
  static constexpr int kStages = int((225 * 1024 - kStaging) / kStage);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStage + kStaging + 512;
};

template <int BN, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PCvtbCfg<SPLIT>::kThreads, 1)
    k_umma_gemm_2sm_cvtb(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap ta2,
                         const __grid_constant__ CUtensorMap tbf, const __grid_constant__ CUtensorMap td,
                         const PArgs args) {
  using C = PCvtbCfg<SPLIT>;
  constexpr int ST = C::kStages;
  constexpr uint32_t kStageF = 64 * (BN / 2) * 4;        // this CTA's 64 k-rows x BN/2 columns of fp32 x
  constexpr uint32_t kStageA = BM * 128;                 // 128 rows of A (hi; lo after it)
  static_assert(BN == 256 && kStageF + 2 * kStageA == C::kStage, "cvtb stage layout");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sF = smem;                                   // [ST][kStageF]: x fp32 -> B_hi | B_lo in place
  uint8_t* sA = smem + ST * kStageF;                    // [ST][2 * kStageA]: A hi | A lo
  float* stg = reinterpret_cast<float*>(sA + ST * 2 * kStageA);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + C::kStaging);
  uint64_t* afull = full + ST;
  uint64_t* cfull = afull + ST;
  uint64_t* empty = cfull + ST;
  uint64_t* tfull = empty + ST;      // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tbf)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&td)) : "memory");
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 2);      // A: the leader's expect_tx + the peer's arrival
      mbar_init(&afull[s], 1);     // this CTA's fp32 x tile
      mbar_init(&cfull[s], 2);     // both CTAs' converted B tiles
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * C::kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(uint32_t(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_holder;
  pdl_wait();
  pdl_trigger();
  const int per_split = args.m_tiles * args.n_tiles;    // column tiles fastest
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr int kCvt0 = 2 + C::kEpiWarps;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs): own A rows (hi, lo), own half of the x columns (fp32)
      int it = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs) {
        const int z = tile / per_split, r = tile % per_split;
        const int64_t m0 = int64_t(r / args.n_tiles) * (2 * BM) + int64_t(rank) * BM;
        const int64_t n0 = int64_t(r % args.n_tiles) * BN + int64_t(rank) * (BN / 2);
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          const int32_t kx = kb * 64;
          uint8_t* f_dst = sF + s * kStageF;
          mbar_expect_tx(&afull[s], kStageF);
#pragma unroll
          for (int c = 0; c < (BN / 2) / 32; ++c) tma_load_2d(&tbf, &afull[s], f_dst + c * 8192, int32_t(n0) + 32 * c, kx);
          if (leader) mbar_expect_tx_only(&full[s], 2 * 2 * kStageA);
          else mbar_arrive_leader(&full[s]);
          uint8_t* a_dst = sA + s * 2 * kStageA;
#pragma unroll
          for (int c = 0; c < BM / 64; ++c) {
            tma_load_2d_2sm(&ta, &full[s], a_dst + c * 8192, int32_t(m0) + 64 * c, kx);
            tma_load_2d_2sm(&ta2, &full[s], a_dst + kStageA + c * 8192, int32_t(m0) + 64 * c, kx);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // MMA issuer
      int it = 0, local = 0;
      for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
        const int z = tile / per_split;
        const int kb0 = z * args.kb_per_split;
        const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
        const int b = local & 1;
        mbar_wait(&tempty[b], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + uint32_t(b * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          mbar_wait(&cfull[s], (it / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* a_src = sA + s * 2 * kStageA;
          const uint8_t* f_src = sF + s * kStageF;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ah = smem_desc_mn(a_src + k * 2048), al = smem_desc_mn(a_src + kStageA + k * 2048);
            const uint64_t bh = smem_desc_mn(f_src + k * 2048), bl = smem_desc_mn(f_src + kStageF / 2 + k * 2048);
            umma2(acc, ah, bh, args.idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            umma2(acc, al, bh, args.idesc, 1u);
            if (SPLIT) umma2(acc, ah, bl, args.idesc, 1u);
          }
          umma2_commit(&empty[s]);
        }
        umma2_commit(&tfull[b]);
      }
    }
  } else if (warp >= kCvt0) {  // converter warps: fp32 x (MN-major) -> bf16 hi | lo in place
    const int ct = threadIdx.x - kCvt0 * 32;
    int it = 0;
    for (int tile = pair; tile < args.tiles; tile += npairs) {
      const int z = tile / per_split;
      const int kb0 = z * args.kb_per_split;
      const int kb1 = min(args.kb_total, kb0 + args.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % ST;
        uint8_t* f = sF + s * kStageF;
        mbar_wait(&afull[s], (it / ST) & 1);
        // job: k-row r = j / 16, 8-column chunk c = j % 16 of this CTA's 128 columns
        float x[C::kJobs][8];
#pragma unroll
        for (int q = 0; q < C::kJobs; ++q) {
          const int j = ct + 32 * C::kCvtWarps * q, r = j >> 4, c = j & 15;
          const uint8_t* box = f + (c >> 2) * 8192 + r * 128;
          const int j0 = (2 * (c & 3)) ^ (r & 7), j1 = (2 * (c & 3) + 1) ^ (r & 7);
          const float4 u = *reinterpret_cast<const float4*>(box + j0 * 16);
          const float4 w = *reinterpret_cast<const float4*>(box + j1 * 16);
          x[q][0] = u.x; x[q][1] = u.y; x[q][2] = u.z; x[q][3] = u.w;
          x[q][4] = w.x; x[q][5] = w.y; x[q][6] = w.z; x[q][7] = w.w;
        }
        cvt_bar_sync<C::kCvtWarps>();
#pragma unroll
        for (int q = 0; q < C::kJobs; ++q) {
          const int j = ct + 32 * C::kCvtWarps * q, r = j >> 4, c = j & 15;
          uint32_t h[4], l[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 hb = __floats2bfloat162_rn(x[q][2 * e], x[q][2 * e + 1]);
            h[e] = *reinterpret_cast<const uint32_t*>(&hb);
            if (SPLIT) {
              const float2 hf = __bfloat1622float2(hb);
              const __nv_bfloat162 lb =
                  __floats2bfloat162_rn(__fsub_rn(x[q][2 * e], hf.x), __fsub_rn(x[q][2 * e + 1], hf.y));
              l[e] = *reinterpret_cast<const uint32_t*>(&lb);
            }
          }
          // MN-major bf16: 64-column chunk c / 8 (8 KB), k-row r, 16-byte chunk (c % 8) ^ (r % 8)
          const int off = (c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4);
          *reinterpret_cast<uint4*>(f + off) = make_uint4(h[0], h[1], h[2], h[3]);
          if (SPLIT) *reinterpret_cast<uint4*>(f + kStageF / 2 + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        cvt_bar_sync<C::kCvtWarps>();
        if (ct == 0) mbar_arrive_leader(&cfull[s]);
      }
    }
  } else {  // epilogue warps (as k_umma_gemm_2sm)
    const int q = warp & 3;
    const int half = C::kEpiWarps == 8 ? (warp - 2) >> 2 : 0;
    constexpr int kCols = C::kEpiWarps == 8 ? BN / 2 : BN;
    float* my_stg = stg + (warp - 2) * 1024;
    int local = 0;
    for (int tile = pair; tile < args.tiles; tile += npairs, ++local) {
      const int z = tile / per_split, r = tile % per_split;
      const int64_t m0 = int64_t(r / args.n_tiles) * (2 * BM) + int64_t(rank) * BM;
      const int64_t n0 = int64_t(r % args.n_tiles) * BN;
      const int kb0 = z * args.kb_per_split;
      const bool any_k = min(args.kb_total, kb0 + args.kb_per_split) > kb0;
      const int b = local & 1;
      mbar_wait(&tfull[b], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int32_t row0 = int32_t(m0 + q * 32);
#pragma unroll 1
      for (int c0 = half * kCols; c0 < (half + 1) * kCols; c0 += 32) {
        if (n0 + c0 >= args.N) break;
        uint32_t rr[32];
        if (any_k) {
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(b * BN + c0), rr);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = 0u;
        }
        float* buf = my_stg;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o;
          o.x = __uint_as_float(rr[4 * j + 0]);
          o.y = __uint_as_float(rr[4 * j + 1]);
          o.z = __uint_as_float(rr[4 * j + 2]);
          o.w = __uint_as_float(rr[4 * j + 3]);
          *reinterpret_cast<float4*>(buf + lane * 32 + ((j ^ (lane & 7)) << 2)) = o;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&td, buf, int32_t(n0 + c0), row0, z);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[b]);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(2 * BN)));
  }
}

// fixed-order split-K reduction (+ bias)
__global__ void k_gemm_reduce(int64_t M, int64_t N, const float* ws, int splits, int64_t split_stride,
                              const float* bias, float* D, int64_t ldd) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = M * N;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / N, n = i % N;
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += ws[z * split_stride + m * N + n];
    D[m * ldd + n] = acc + (bias ? bias[n] : 0.f);
  }
}

// tiled transpose dst[c][r] = src[r][c] (fp32 or bf16 in, fp32 or bf16 out).
// SPLIT: fp32 -> bf16 hi at dst[c][r] and bf16 lo = x - hi at dst[c][rows + r]
// (the bf16x2 operand that carries ~16 mantissa bits through bf16 tensor
// cores); DUP: the value is written to both halves.
enum { TR_PLAIN = 0, TR_SPLIT = 1, TR_DUP = 2 };
template <typename S, typename Dt, int MODE>
__global__ void k_transpose(int64_t rows, int64_t cols, const S* src, int64_t lds, Dt* dst, int64_t ldd) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][33];
  const int64_t r0 = int64_t(blockIdx.y) * 32, c0 = int64_t(blockIdx.x) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? float(src[r * lds + c]) : 0.f;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) {
      const float x = tile[threadIdx.x][k];
      if constexpr (MODE == TR_PLAIN) {
        dst[c * ldd + r] = Dt(x);
      } else if constexpr (MODE == TR_SPLIT) {
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        dst[c * ldd + r] = hi;
        dst[c * ldd + rows + r] = __float2bfloat16_rn(x - __bfloat162float(hi));
      } else {
        dst[c * ldd + r] = Dt(x);
        dst[c * ldd + rows + r] = Dt(x);
      }
    }
  }
}

// row-wise bf16x2 split without transposing: dst[r][c] = hi, dst[r][cols + c] = lo
__global__ void k_split_rows(int64_t rows, int64_t cols, const float* src, int64_t lds, __nv_bfloat16* dst,
                             int64_t ldd) {
  pdl_wait();
  pdl_trigger();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const float x = src[r * lds + c];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    dst[r * ldd + c] = hi;
    dst[r * ldd + cols + c] = __float2bfloat16_rn(x - __bfloat162float(hi));
  }
}

// row-wise three-slot bf16 split for the fp32-class projection (bf16x3):
// slots of width `slot` elements; order 0 writes [hi | lo | hi], order 1
// [hi | hi | lo], so A3 . B3^T = xh.Wh + xl.Wh + xh.Wl (the x_lo.W_lo term,
// ~2^-16 relative, is dropped).  Pad columns are left to the caller (zeros).
__global__ void k_split3_rows(int64_t rows, int64_t cols, const float* src, int64_t lds, __nv_bfloat16* dst,
                              int64_t ldd, int64_t slot, int order) {
  pdl_wait();
  pdl_trigger();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const float x = __ldg(src + r * lds + c);
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
    // orders 0 / 1: three column slots of one row; 2: three row blocks of `slot` rows
    const int64_t step = order == 2 ? slot * ldd : slot;
    __nv_bfloat16* d = dst + r * ldd + c;
    d[0] = hi;
    d[step] = order == 0 ? lo : hi;
    d[2 * step] = order == 0 ? hi : lo;
  }
}

// vectorised form (cols % 8 == 0, 16-byte aligned rows and slots): 8 columns
// per thread, two 16-byte loads and three 16-byte stores
__global__ void k_split3_rows_v8(int64_t rows, int64_t cols8, const float* src, int64_t lds, __nv_bfloat16* dst,
                                 int64_t ldd, int64_t slot, int order) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = rows * cols8;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / cols8, c = (q % cols8) * 8;
    const float4 a = __ldg(reinterpret_cast<const float4*>(src + r * lds + c));
    const float4 b = __ldg(reinterpret_cast<const float4*>(src + r * lds + c + 4));
    const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hi[j] = __float2bfloat16_rn(x[j]);
      lo[j] = __float2bfloat16_rn(x[j] - __bfloat162float(hi[j]));
    }
    const uint4 h = *reinterpret_cast<const uint4*>(hi), l = *reinterpret_cast<const uint4*>(lo);
    const int64_t step = order == 2 ? slot * ldd : slot;
    __nv_bfloat16* d = dst + r * ldd + c;
    *reinterpret_cast<uint4*>(d) = h;
    *reinterpret_cast<uint4*>(d + step) = order == 0 ? l : h;
    *reinterpret_cast<uint4*>(d + 2 * step) = order == 0 ? h : l;
  }
}

// 8 elements per thread: two 16-byte loads, one 16-byte store (16-byte aligned
// src/dst, checked by the caller); the scalar kernel takes the rest
__global__ void k_cast_bf16_v8(int64_t n8, const float4* src, uint4* dst) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(src + 2 * i), b = __ldg(src + 2 * i + 1);
    __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    dst[i] = *reinterpret_cast<uint4*>(h);
  }
}
__global__ void k_cast_bf16(int64_t n, const float* src, __nv_bfloat16* dst) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// deterministic column sums of a [rows][cols] fp32 matrix (bias gradient,
// learn.py:273).  Pass 1: block (bx, by) covers 32 columns x one row chunk;
// its 8 row-lanes stride the chunk in order (coalesced 128 B rows), then the
// lanes are summed in order into part[by][c].  Pass 2 sums the chunks in order.
constexpr int kColChunks = 64;
__global__ void __launch_bounds__(256) k_col_sum_part(int64_t rows, int64_t cols, const float* src, int64_t ld,
                                                      double* part) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8][33];
  const int64_t c = int64_t(blockIdx.x) * 32 + threadIdx.x;
  const int64_t per = (rows + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = int64_t(blockIdx.y) * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  if (c < cols)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) acc += double(src[r * ld + c]);
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    part[int64_t(blockIdx.y) * cols + c] = s;
  }
}
// one-pass form (rows <= kColOnePass: one row chunk) and the assigning final
// pass of hhb_col_sum_ex: out64 / out32 receive the sums (either may be null)
constexpr int64_t kColOnePass = 512;
__global__ void __launch_bounds__(256) k_col_sum_one(int64_t rows, int64_t cols, const float* src, int64_t ld,
                                                     double* out64, float* out32) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[8][33];
  const int64_t c = int64_t(blockIdx.x) * 32 + threadIdx.x;
  double acc = 0.0;
  if (c < cols)
    for (int64_t r = threadIdx.y; r < rows; r += 8) acc += double(src[r * ld + c]);
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    if (out64) out64[c] = s;
    if (out32) out32[c] = float(s);
  }
}
__global__ void k_col_sum_final_set(int64_t cols, int chunks, const double* part, double* out64, float* out32) {
  pdl_wait();
  pdl_trigger();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int k = 0; k < chunks; ++k) s += part[int64_t(k) * cols + c];
  if (out64) out64[c] = s;
  if (out32) out32[c] = float(s);
}
// fixed-order sum of n doubles (one block: strided per-thread sums in order,
// then a fixed shared-memory tree), times scale -> out64[0] / out32[0]
__global__ void __launch_bounds__(1024) k_sum_f64(int64_t n, const double* x, double scale, double* out64,
                                                  float* out32) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[1024];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double s = red[0] * scale;
    if (out64) out64[0] = s;
    if (out32) out32[0] = float(s);
  }
}
__global__ void k_col_sum_final(int64_t cols, int chunks, const double* part, double* out) {
  pdl_wait();
  pdl_trigger();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int k = 0; k < chunks; ++k) s += part[int64_t(k) * cols + c];
  out[c] += s;
}

// ------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

static int make_map(CUtensorMap* map, bool tf32, const void* base, int64_t rows, int64_t k, int64_t ld,
                    int box_rows) {
  EncodeFn enc = encoder();
  if (!enc) return fail(HHB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const int eb = tf32 ? 4 : 2;
  const cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * eb};
  const cuuint32_t box[2] = {cuuint32_t(128 / eb), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                         const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HHB_EINVAL, "cuTensorMapEncodeTiled rejected the operand layout");
  return HHB_OK;
}

// MN-major fp32 operand (converted on chip): global [K][ld] floats, boxes of 32 x 64
static int make_map_mn_f32(CUtensorMap* map, const float* base, int64_t mn, int64_t k, int64_t ld) {
  EncodeFn enc = encoder();
  if (!enc) return fail(HHB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cuuint64_t(mn), cuuint64_t(k)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  const cuuint32_t box[2] = {32u, 64u};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HHB_EINVAL, "cuTensorMapEncodeTiled rejected the fp32 MN-major operand");
  return HHB_OK;
}

// MN-major bf16 operand: global [K][ld] (MN contiguous), boxes of 64 x 64
static int make_map_mn(CUtensorMap* map, const void* base, int64_t mn, int64_t k, int64_t ld) {
  EncodeFn enc = encoder();
  if (!enc) return fail(HHB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cuuint64_t(mn), cuuint64_t(k)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
  const cuuint32_t box[2] = {64u, 64u};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HHB_EINVAL, "cuTensorMapEncodeTiled rejected the MN-major operand layout");
  return HHB_OK;
}

template <int BN, bool TF32, bool A_MN, bool B_MN, bool DUAL>
static int launch(const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tb, const Args& a, int splits,
                  cudaStream_t st) {
  const size_t smem = Cfg<BN, TF32, DUAL>::kSmem;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(k_umma_gemm<BN, TF32, A_MN, B_MN, DUAL>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  });
  if (attr_err != cudaSuccess) return fail(HHB_ECUDA, "cudaFuncSetAttribute(smem) failed");
  const dim3 grid{unsigned((a.N + BN - 1) / BN), unsigned((a.M + BM - 1) / BM), unsigned(splits)};
  launch_pdl(k_umma_gemm<BN, TF32, A_MN, B_MN, DUAL>, dim3(grid), dim3(kThreads), smem, st, ta, ta2, tb, a);
  return cuda_check("k_umma_gemm launch");
}

template <bool TF32, bool A_MN, bool B_MN, bool DUAL>
static int launch_bn(int bn, const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tb, const Args& a,
                     int splits, cudaStream_t st) {
  if (bn == 64) return launch<64, TF32, A_MN, B_MN, DUAL>(ta, ta2, tb, a, splits, st);
  if (bn == 128) return launch<128, TF32, A_MN, B_MN, DUAL>(ta, ta2, tb, a, splits, st);
  return launch<256, TF32, A_MN, B_MN, DUAL>(ta, ta2, tb, a, splits, st);
}

// D (fp32) as a 3-D tensor {N, M, splits}: 32x32 store boxes, 128B swizzle,
// clipped at the edges of each split slice
static int make_map_d(CUtensorMap* map, float* base, int64_t M, int64_t N, int64_t ldd, int splits) {
  EncodeFn enc = encoder();
  if (!enc) return fail(HHB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {cuuint64_t(N), cuuint64_t(M), cuuint64_t(splits)};
  const cuuint64_t strides[2] = {cuuint64_t(ldd) * 4, cuuint64_t(ldd) * 4 * cuuint64_t(M)};
  const cuuint32_t box[3] = {32u, 32u, 1u};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HHB_EINVAL, "cuTensorMapEncodeTiled rejected the output layout");
  return HHB_OK;
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN, bool DUAL>
static int launch_p(const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tb, const CUtensorMap& td,
                    const PArgs& a, cudaStream_t st) {
  const size_t smem = PCfg<BN, DUAL>::kSmem;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(k_umma_gemm_p<BN, A_MN, B_MN, DUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem));
  });
  if (attr_err != cudaSuccess) return fail(HHB_ECUDA, "cudaFuncSetAttribute(smem) failed");
  const int grid = a.tiles < num_sms() ? a.tiles : num_sms();
  launch_pdl(k_umma_gemm_p<BN, A_MN, B_MN, DUAL>, dim3(grid), dim3(kThreads), smem, st, ta, ta2, tb, td, a);
  return cuda_check("k_umma_gemm_p launch");
}

template <bool A_MN, bool B_MN, bool DUAL>
static int launch_p_bn(int bn, const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tb,
                       const CUtensorMap& td, const PArgs& a, cudaStream_t st) {
  if (bn == 64) return launch_p<64, A_MN, B_MN, DUAL>(ta, ta2, tb, td, a, st);
  if (bn == 128) return launch_p<128, A_MN, B_MN, DUAL>(ta, ta2, tb, td, a, st);
  return launch_p<256, A_MN, B_MN, DUAL>(ta, ta2, tb, td, a, st);
}

template <int BN, bool A_MN, bool B_MN, bool DUAL>
static int launch_2sm(const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tb, const CUtensorMap& td,
                      const PArgs& a, cudaStream_t st) {
  const size_t smem = P2Cfg<BN, DUAL>::kSmem;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(k_umma_gemm_2sm<BN, A_MN, B_MN, DUAL>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  });
  if (attr_err != cudaSuccess) return fail(HHB_ECUDA, "cudaFuncSetAttribute(smem) failed");
  // persistent: as many pairs as can be co-resident (not every SM has a
  // usable TPC partner), queried once
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
    cfg.blockDim = dim3(kThreads2, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_umma_gemm_2sm<BN, A_MN, B_MN, DUAL>, &cfg) != cudaSuccess || n <= 0)
      n = num_sms() / 2;
    (void)cudaGetLastError();
    max_pairs = n;
  }
  int pairs = max_pairs;
  if (a.tiles < pairs) pairs = a.tiles;
  if (getenv("HHB_GEMM_PAIRS_DEBUG")) fprintf(stderr, "k_umma_gemm_2sm: %d co-resident pairs\n", max_pairs);
  launch_pdl(k_umma_gemm_2sm<BN, A_MN, B_MN, DUAL>, dim3(2 * pairs), dim3(kThreads2), smem, st, ta, ta2, tb, td, a);
  return cuda_check("k_umma_gemm_2sm launch");
}

template <int BN, bool SPLIT>
static int launch_2sm_cvt(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2,
                          const CUtensorMap& td, const CUtensorMap& txh, const CUtensorMap& txl, const PArgs& a,
                          cudaStream_t st) {
  using C = PCvtCfg<BN, SPLIT>;
  const size_t smem = C::kSmem;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(k_umma_gemm_2sm_cvt<BN, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem));
  });
  if (attr_err != cudaSuccess) return fail(HHB_ECUDA, "cudaFuncSetAttribute(smem) failed (cvt)");
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
    cfg.blockDim = dim3(C::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_umma_gemm_2sm_cvt<BN, SPLIT>, &cfg) != cudaSuccess || n <= 0)
      n = num_sms() / 2;
    (void)cudaGetLastError();
    max_pairs = n;
  }
  int pairs = max_pairs;
  if (a.tiles < pairs) pairs = a.tiles;
  launch_pdl(k_umma_gemm_2sm_cvt<BN, SPLIT>, dim3(2 * pairs), dim3(C::kThreads), smem, st, ta, tb, tb2, td, txh, txl,
             a);
  return cuda_check("k_umma_gemm_2sm_cvt launch");
}

template <bool SPLIT>
static int launch_2sm_cvtb(const CUtensorMap& ta, const CUtensorMap& ta2, const CUtensorMap& tbf,
                           const CUtensorMap& td, const PArgs& a, cudaStream_t st) {
  using C = PCvtbCfg<SPLIT>;
  const size_t smem = C::kSmem;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(k_umma_gemm_2sm_cvtb<256, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  });
  if (attr_err != cudaSuccess) return fail(HHB_ECUDA, "cudaFuncSetAttribute(smem) failed (cvtb)");
  static int max_pairs = 0;
  if (max_pairs == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
    cfg.blockDim = dim3(C::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_umma_gemm_2sm_cvtb<256, SPLIT>, &cfg) != cudaSuccess || n <= 0)
      n = num_sms() / 2;
    (void)cudaGetLastError();
    max_pairs = n;
  }
  int pairs = max_pairs;
  if (a.tiles < pairs) pairs = a.tiles;
  launch_pdl(k_umma_gemm_2sm_cvtb<256, SPLIT>, dim3(2 * pairs), dim3(C::kThreads), smem, st, ta, ta2, tbf, td, a);
  return cuda_check("k_umma_gemm_2sm_cvtb launch");
}

// tile order of the persistent GEMMs: column tiles fastest unless HHB_GEMM_RASTER=m
static int gemm_n_fast() {
  static const int v = [] {
    const char* e = getenv("HHB_GEMM_RASTER");
    return (e && e[0] == 'm') ? 0 : 1;
  }();
  return v;
}

static uint32_t instr_desc(bool tf32, int bn, bool a_mn = false, bool b_mn = false, int m = BM) {
  const uint32_t fmt = tf32 ? 2u : 1u;  // TF32 : BF16
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(bn >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

}  // namespace gemm
}  // namespace hhb

using namespace hhb;

extern "C" {

int64_t hhb_gemm_workspace(int64_t M, int64_t N, int32_t splits) { return splits > 1 ? int64_t(splits) * M * N : 0; }

int hhb_gemm(int32_t in_kind, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
             int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits, float* workspace,
             void* stream) {
  using namespace hhb::gemm;
  const bool tf32 = in_kind == HHB_GEMM_TF32;
  if (in_kind != HHB_GEMM_BF16 && in_kind != HHB_GEMM_TF32) return fail(HHB_EINVAL, "in_kind");
  if (!tf32) return hhb_gemm_ex(0, M, N, K, A, nullptr, lda, B, ldb, bias, D, ldd, splits, workspace, stream);
  if (M < 0 || N < 0 || K < 0 || (M && N && (!A || !B || !D)) || ldd < N) return fail(HHB_EINVAL, "gemm shape");
  if (M == 0 || N == 0) return HHB_OK;
  const int eb = tf32 ? 4 : 2;
  if ((lda * eb) % 16 || (ldb * eb) % 16 || reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(B) % 16)
    return fail(HHB_EINVAL, "gemm operands need 16-byte aligned base and row pitch");
  if (lda < K || ldb < K) return fail(HHB_EINVAL, "lda/ldb < K");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int bk = 128 / eb;
  const int kb_total = int((K + bk - 1) / bk);
  if (splits < 1) splits = 1;
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  if (splits > 1 && !workspace) return fail(HHB_EINVAL, "split-K needs workspace");
  int bn = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  if (const char* e = getenv("HHB_GEMM_BN")) {   // experiments: force the tile width
    const int f = atoi(e);
    if ((f == 64 || f == 128 || f == 256) && f <= bn) bn = f;
  }
  CUtensorMap ta, tb;
  int rc = make_map(&ta, tf32, A, M, K, lda, BM);
  if (rc) return rc;
  if ((rc = make_map(&tb, tf32, B, N, K, ldb, bn))) return rc;
  Args a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.kb_total = kb_total;
  a.kb_per_split = (kb_total + splits - 1) / splits;
  a.idesc = instr_desc(tf32, bn);
  if (splits > 1) {
    a.D = workspace;
    a.ldd = N;
    a.split_stride = M * N;
    a.bias = nullptr;
  } else {
    a.D = D;
    a.ldd = ldd;
    a.split_stride = 0;
    a.bias = bias;
  }
  rc = tf32 ? launch_bn<true, false, false, false>(bn, ta, ta, tb, a, splits, st)
            : launch_bn<false, false, false, false>(bn, ta, ta, tb, a, splits, st);
  if (rc || splits == 1) return rc;
  launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits, int64_t(M * N), bias, D, ldd);
  return cuda_check("k_gemm_reduce launch");
}

static int gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const void* B, const void* Blo,
                     int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits, float* workspace,
                     void* stream, void* xs = nullptr, int64_t xs_ld = 0, int64_t xs_slot = 0);
static int gemm_ex_impl(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2,
                        int64_t lda, const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd,
                        int32_t splits, float* workspace, int64_t k_switch, void* stream);

int hhb_gemm_ex(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2, int64_t lda,
                const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits,
                float* workspace, void* stream) {
  return gemm_ex_impl(flags, M, N, K, A, A2, lda, B, ldb, bias, D, ldd, splits, workspace, 0, stream);
}

int hhb_gemm_ex2(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2, int64_t lda,
                 const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits,
                 float* workspace, int64_t k_switch, void* stream) {
  return gemm_ex_impl(flags, M, N, K, A, A2, lda, B, ldb, bias, D, ldd, splits, workspace, k_switch, stream);
}

int hhb_gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const void* B, const void* B_lo,
                  int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits, float* workspace,
                  void* xs, int64_t xs_ld, int64_t xs_slot, void* stream) {
  return gemm_f32a(M, N, K, A, lda, B, B_lo, ldb, bias, D, ldd, splits, workspace, stream, xs, xs_ld, xs_slot);
}

int hhb_gemm_f32b(int64_t M, int64_t N, int64_t K, const void* A, const void* A_lo, int64_t lda, const float* B,
                  int64_t ldb, int32_t split_b, float* D, int64_t ldd, int32_t splits, float* workspace,
                  void* stream) {
  using namespace hhb::gemm;
  if (M < 0 || N < 0 || K < 0 || (M && N && (!A || !A_lo || !B || !D)) || ldd < N) return fail(HHB_EINVAL, "gemm shape");
  if (M == 0 || N == 0) return HHB_OK;
  if ((lda * 2) % 16 || (ldb * 4) % 16 || reinterpret_cast<uintptr_t>(A) % 16 ||
      reinterpret_cast<uintptr_t>(A_lo) % 16 || reinterpret_cast<uintptr_t>(B) % 16)
    return fail(HHB_EINVAL, "gemm operands need 16-byte aligned base and row pitch");
  if (lda < M || ldb < N) return fail(HHB_EINVAL, "lda/ldb too small");
  if (M < 512 || N <= 128) return fail(HHB_EINVAL, "fp32-B GEMM: M >= 512 rows and N > 128 columns (256-wide pair tiles)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int bn = 256;
  const int kb_total = int((K + 63) / 64);
  if (splits < 1) {
    const int64_t tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn);
    const int64_t P = num_sms() / 2;
    const double t_kb = 0.28 * (split_b ? 3.0 : 2.0);
    const double t_mn = double(M) * double(N) * 4.0 / 5e12 * 1e6;
    double best = 1e300;
    splits = 1;
    for (int sp = 1; sp <= (kb_total >= 8 ? kb_total / 4 : 1) && sp <= 32; ++sp) {
      const int64_t units = tiles * sp;
      const double cost = double((units + P - 1) / P) * double((kb_total + sp - 1) / sp) * t_kb +
                          (sp > 1 ? double(2 * sp + 1) * t_mn : 0.0);
      if (cost < best - 1e-9) {
        best = cost;
        splits = sp;
      }
    }
  }
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  if (splits > 1 && !workspace) return fail(HHB_EINVAL, "split-K needs workspace");
  float* dst = splits > 1 ? workspace : D;
  const int64_t dld = splits > 1 ? N : ldd;
  if (dld % 4 != 0 || reinterpret_cast<uintptr_t>(dst) % 16 != 0)
    return fail(HHB_EINVAL, "fp32-B GEMM needs a 16-byte aligned output pitch");
  CUtensorMap ta, ta2, tbf, td;
  int rc = make_map_mn(&ta, A, M, K, lda);
  if (rc) return rc;
  if ((rc = make_map_mn(&ta2, A_lo, M, K, lda))) return rc;
  if ((rc = make_map_mn_f32(&tbf, B, N, K, ldb))) return rc;
  if ((rc = make_map_d(&td, dst, M, N, dld, splits))) return rc;
  PArgs pa{};
  pa.M = M;
  pa.N = N;
  pa.m_tiles = int((M + 2 * BM - 1) / (2 * BM));
  pa.n_tiles = int((N + bn - 1) / bn);
  pa.kb_total = kb_total;
  pa.kb_per_split = (kb_total + splits - 1) / splits;
  pa.splits = splits;
  pa.tiles = pa.m_tiles * pa.n_tiles * splits;
  pa.idesc = instr_desc(false, bn, true, true, 2 * BM);
  pa.bias = nullptr;
  pa.K = K;
  if ((rc = split_b ? launch_2sm_cvtb<true>(ta, ta2, tbf, td, pa, st) : launch_2sm_cvtb<false>(ta, ta2, tbf, td, pa, st)) ||
      splits == 1)
    return rc;
  launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits,
             int64_t(M * N), (const float*)nullptr, D, ldd);
  return cuda_check("k_gemm_reduce launch");
}

// fp32-A CTA-pair GEMM (k_umma_gemm_2sm_cvt): D = bf16(A) . B^T, or with B_lo
// the three-product hi.B + lo.B + hi.B_lo of proj="bf16x3"; 2-SM tiles only
static int gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const void* B, const void* Blo,
                     int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits, float* workspace,
                     void* stream, void* xs, int64_t xs_ld, int64_t xs_slot) {
  using namespace hhb::gemm;
  if (M < 0 || N < 0 || K < 0 || (M && N && (!A || !B || !D)) || ldd < N) return fail(HHB_EINVAL, "gemm shape");
  if (M == 0 || N == 0) return HHB_OK;
  if ((lda * 4) % 16 || (ldb * 2) % 16 || reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(B) % 16 ||
      reinterpret_cast<uintptr_t>(Blo) % 16)
    return fail(HHB_EINVAL, "gemm operands need 16-byte aligned base and row pitch");
  if (lda < K || ldb < K) return fail(HHB_EINVAL, "lda/ldb too small");
  const int bn = N <= 128 ? 128 : 256;
  if (M < 512) return fail(HHB_EINVAL, "fp32-A GEMM needs M >= 512 (CTA-pair tiles)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int kb_total = int((K + 63) / 64);
  if (splits < 1) {   // the bf16 path's time model (CTA pairs), the three-product form counted 3x
    const int64_t tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn);
    const int64_t P = num_sms() / 2;
    const double t_kb = 0.28 * (Blo ? 3.0 : 1.0) * (double(bn) / 256.0);
    const double t_mn = double(M) * double(N) * 4.0 / 5e12 * 1e6;
    double best = 1e300;
    splits = 1;
    for (int sp = 1; sp <= (kb_total >= 8 ? kb_total / 4 : 1) && sp <= 32; ++sp) {
      const int64_t units = tiles * sp;
      const double cost = double((units + P - 1) / P) * double((kb_total + sp - 1) / sp) * t_kb +
                          (sp > 1 ? double(2 * sp + 1) * t_mn : 0.0);
      if (cost < best - 1e-9) {
        best = cost;
        splits = sp;
      }
    }
  }
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  if (splits > 1 && !workspace) return fail(HHB_EINVAL, "split-K needs workspace");
  float* dst = splits > 1 ? workspace : D;
  const int64_t dld = splits > 1 ? N : ldd;
  if (dld % 4 != 0 || reinterpret_cast<uintptr_t>(dst) % 16 != 0)
    return fail(HHB_EINVAL, "fp32-A GEMM needs a 16-byte aligned output pitch");
  CUtensorMap ta, tb, tb2, td, txh, txl;
  int rc = make_map(&ta, true, A, M, K, lda, BM);
  if (rc) return rc;
  if ((rc = make_map(&tb, false, B, N, K, ldb, bn / 2))) return rc;
  if (Blo && (rc = make_map(&tb2, false, Blo, N, K, ldb, bn / 2))) return rc;
  if (!Blo) tb2 = tb;
  if ((rc = make_map_d(&td, dst, M, N, dld, splits))) return rc;
  PArgs pa{};
  pa.M = M;
  pa.N = N;
  pa.m_tiles = int((M + 2 * BM - 1) / (2 * BM));
  pa.n_tiles = int((N + bn - 1) / bn);
  pa.kb_total = kb_total;
  pa.kb_per_split = (kb_total + splits - 1) / splits;
  pa.splits = splits;
  pa.tiles = pa.m_tiles * pa.n_tiles * splits;
  pa.idesc = instr_desc(false, bn, false, false, 2 * BM);
  pa.bias = splits > 1 ? nullptr : bias;
  pa.kb_switch = 0;
  pa.n_fast = gemm_n_fast();
  pa.K = K;
  if (xs) {
    if (K % 8 || xs_ld % 8 || xs_slot % 8 || reinterpret_cast<uintptr_t>(xs) % 16 || xs_ld < (Blo ? xs_slot + K : K) ||
        (Blo && xs_slot < K))
      return fail(HHB_EINVAL, "converted-operand output: K, pitch and slot multiples of 8, 16-byte aligned");
    pa.xs = static_cast<uint16_t*>(xs);
    pa.xs_ld = xs_ld;
    pa.xs_slot = xs_slot;
    // hi / lo slots as separate K-wide tensors (the store of a partial last
    // k-block is clipped at K, not spilled into the next slot)
    if ((rc = make_map(&txh, false, xs, M, K, xs_ld, BM))) return rc;
    if (Blo && (rc = make_map(&txl, false, static_cast<uint16_t*>(xs) + xs_slot, M, K, xs_ld, BM))) return rc;
  }
  if (!xs) txh = ta;
  if (!xs || !Blo) txl = xs ? txh : ta;
  if (Blo) rc = bn == 128 ? launch_2sm_cvt<128, true>(ta, tb, tb2, td, txh, txl, pa, st) : launch_2sm_cvt<256, true>(ta, tb, tb2, td, txh, txl, pa, st);
  else rc = bn == 128 ? launch_2sm_cvt<128, false>(ta, tb, tb2, td, txh, txl, pa, st) : launch_2sm_cvt<256, false>(ta, tb, tb2, td, txh, txl, pa, st);
  if (rc || splits == 1) return rc;
  launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits,
             int64_t(M * N), bias, D, ldd);
  return cuda_check("k_gemm_reduce launch");
}

static int gemm_ex_impl(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2,
                        int64_t lda, const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd,
                        int32_t splits, float* workspace, int64_t k_switch, void* stream) {
  using namespace hhb::gemm;
  const bool a_mn = flags & HHB_GEMM_A_MN, b_mn = flags & HHB_GEMM_B_MN;
  // fp32 A converted on chip (HHB_GEMM_A_F32; + HHB_GEMM_A_SPLIT: hi/lo with A2 = B_lo)
  const bool a_f32 = flags & HHB_GEMM_A_F32, a_split = flags & HHB_GEMM_A_SPLIT;
  if (a_f32 || a_split) {
    if (!a_f32 || a_mn || b_mn || k_switch > 0 || (a_split != (A2 != nullptr)))
      return fail(HHB_EINVAL, "fp32-A GEMM: K-major A and B, no k_switch, A2 (= B_lo) iff HHB_GEMM_A_SPLIT");
    return gemm_f32a(M, N, K, static_cast<const float*>(A), lda, B, a_split ? A2 : nullptr, ldb, bias, D, ldd,
                     splits, workspace, stream);
  }
  // k_switch > 0: A2 is not a second addend but the A source for k >= k_switch
  // (K-concatenation of two K-major operands, e.g. [dI_hi | dI_lo] then dI_hi)
  const bool dual = A2 != nullptr && k_switch <= 0;
  if (k_switch > 0 && (a_mn || !A2 || k_switch % 64 || k_switch >= K))
    return fail(HHB_EINVAL, "k_switch needs a K-major A2, a multiple of 64 below K");
  if (flags & ~(HHB_GEMM_A_MN | HHB_GEMM_B_MN)) return fail(HHB_EINVAL, "gemm flags");
  if (M < 0 || N < 0 || K < 0 || (M && N && (!A || !B || !D)) || ldd < N) return fail(HHB_EINVAL, "gemm shape");
  if (M == 0 || N == 0) return HHB_OK;
  if ((lda * 2) % 16 || (ldb * 2) % 16 || reinterpret_cast<uintptr_t>(A) % 16 ||
      reinterpret_cast<uintptr_t>(A2) % 16 || reinterpret_cast<uintptr_t>(B) % 16)
    return fail(HHB_EINVAL, "gemm operands need 16-byte aligned base and row pitch");
  // K-switched A: each source spans only its own K range
  const int64_t ka = k_switch > 0 ? (k_switch > K - k_switch ? k_switch : K - k_switch) : K;
  if (lda < (a_mn ? M : ka) || ldb < (b_mn ? N : K)) return fail(HHB_EINVAL, "lda/ldb too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int kb_total = int((K + 63) / 64);
  // tile width: 64 / 128 for narrow N, else 256 (N = 784 measured 78.8 us
  // (dW) / 86.9 us (dX) at 256 against 90.2 / 104.7 at 128: the padding of the
  // last 256-wide tile costs less than halving B reuse, profiles/r2_gemm_variants.md).
  // HHB_GEMM_BN overrides (experiments).
  int bn = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  if (const char* e = getenv("HHB_GEMM_BN")) {
    const int v = atoi(e);
    if (v == 64 || v == 128 || v == 256) bn = v;
  }
  if (splits < 1) {
    // auto (splits <= 0): minimise a time model of the persistent grid --
    // waves x k-blocks per unit x ~0.28 us per 64-deep k-block of a tile
    // (doubled for the dual-A form), plus the split-K traffic (partials
    // written and re-read, result written: (2 sp + 1) M N fp32 at ~5 TB/s);
    // CTA-pair tiles (256 x BN) when M >= 512
    const bool pairs = bn >= 128 && M >= 512;
    const int64_t tiles = ((M + (pairs ? 2 * BM : BM) - 1) / (pairs ? 2 * BM : BM)) * ((N + bn - 1) / bn);
    const int64_t P = pairs ? hhb::gemm::num_sms() / 2 : hhb::gemm::num_sms();
    const double t_kb = 0.28 * (dual ? 2.0 : 1.0) * (pairs ? 1.0 : 0.5) * (double(bn) / 256.0);
    const double t_mn = double(M) * double(N) * 4.0 / 5e12 * 1e6;
    double best = 1e300;
    splits = 1;
    for (int sp = 1; sp <= (kb_total >= 8 ? kb_total / 4 : 1) && sp <= 32; ++sp) {
      const int64_t units = tiles * sp;
      const double cost = double((units + P - 1) / P) * double((kb_total + sp - 1) / sp) * t_kb +
                          (sp > 1 ? double(2 * sp + 1) * t_mn : 0.0);
      if (cost < best - 1e-9) {
        best = cost;
        splits = sp;
      }
    }
  }
  if (splits > kb_total) splits = kb_total > 0 ? kb_total : 1;
  if (splits > 1 && !workspace) return fail(HHB_EINVAL, "split-K needs workspace");
  CUtensorMap ta, ta2, tb;
  int rc = a_mn ? make_map_mn(&ta, A, M, K, lda) : make_map(&ta, false, A, M, K, lda, BM);
  if (rc) return rc;
  if (dual && (rc = a_mn ? make_map_mn(&ta2, A2, M, K, lda) : make_map(&ta2, false, A2, M, K, lda, BM))) return rc;
  if (k_switch > 0) {
    if ((rc = make_map(&ta, false, A, M, k_switch, lda, BM))) return rc;
    if ((rc = make_map(&ta2, false, A2, M, K - k_switch, lda, BM))) return rc;
  }
  if ((rc = b_mn ? make_map_mn(&tb, B, N, K, ldb) : make_map(&tb, false, B, N, K, ldb, bn))) return rc;
  if (!dual && k_switch <= 0) ta2 = ta;
  float* dst = splits > 1 ? workspace : D;
  const int64_t dld = splits > 1 ? N : ldd;
  if (dld % 4 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 && !getenv("HHB_GEMM_NONPERSISTENT")) {
    CUtensorMap td;
    if ((rc = make_map_d(&td, dst, M, N, dld, splits))) return rc;
    // CTA pairs (cta_group::2, 256 x BN tiles) when there are enough rows
    if (bn >= 128 && M >= 512 && !getenv("HHB_GEMM_NO2SM")) {
      CUtensorMap tb2;
      if (!b_mn && (rc = make_map(&tb2, false, B, N, K, ldb, bn / 2))) return rc;
      if (b_mn) tb2 = tb;
      PArgs pa{};
      pa.M = M;
      pa.N = N;
      pa.m_tiles = int((M + 2 * BM - 1) / (2 * BM));
      pa.n_tiles = int((N + bn - 1) / bn);
      pa.kb_total = kb_total;
      pa.kb_per_split = (kb_total + splits - 1) / splits;
      pa.splits = splits;
      pa.tiles = pa.m_tiles * pa.n_tiles * splits;
      pa.idesc = instr_desc(false, bn, a_mn, b_mn, 2 * BM);
      pa.bias = splits > 1 ? nullptr : bias;
      pa.kb_switch = k_switch > 0 ? int(k_switch / 64) : 0;
      pa.n_fast = gemm_n_fast();
#define HHB_GEMM_2CASE(AM, BMN, DU)                                                              \
  if (a_mn == AM && b_mn == BMN && dual == DU)                                                   \
    rc = bn == 128 ? launch_2sm<128, AM, BMN, DU>(ta, ta2, tb2, td, pa, st)                      \
                   : launch_2sm<256, AM, BMN, DU>(ta, ta2, tb2, td, pa, st);
      HHB_GEMM_2CASE(false, false, false)
      HHB_GEMM_2CASE(false, false, true)
      HHB_GEMM_2CASE(false, true, false)
      HHB_GEMM_2CASE(false, true, true)
      HHB_GEMM_2CASE(true, false, false)
      HHB_GEMM_2CASE(true, false, true)
      HHB_GEMM_2CASE(true, true, false)
      HHB_GEMM_2CASE(true, true, true)
#undef HHB_GEMM_2CASE
      if (rc || splits == 1) return rc;
      launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits, int64_t(M * N), bias, D, ldd);
      return cuda_check("k_gemm_reduce launch");
    }
    PArgs pa{};
    pa.M = M;
    pa.N = N;
    pa.m_tiles = int((M + BM - 1) / BM);
    pa.n_tiles = int((N + bn - 1) / bn);
    pa.kb_total = kb_total;
    pa.kb_per_split = (kb_total + splits - 1) / splits;
    pa.splits = splits;
    pa.tiles = pa.m_tiles * pa.n_tiles * splits;
    pa.idesc = instr_desc(false, bn, a_mn, b_mn);
    pa.bias = splits > 1 ? nullptr : bias;
    pa.kb_switch = k_switch > 0 ? int(k_switch / 64) : 0;
    pa.n_fast = gemm_n_fast();
#define HHB_GEMM_PCASE(AM, BMN, DU)                                   \
  if (a_mn == AM && b_mn == BMN && dual == DU)                        \
    rc = launch_p_bn<AM, BMN, DU>(bn, ta, ta2, tb, td, pa, st);
    HHB_GEMM_PCASE(false, false, false)
    HHB_GEMM_PCASE(false, false, true)
    HHB_GEMM_PCASE(false, true, false)
    HHB_GEMM_PCASE(false, true, true)
    HHB_GEMM_PCASE(true, false, false)
    HHB_GEMM_PCASE(true, false, true)
    HHB_GEMM_PCASE(true, true, false)
    HHB_GEMM_PCASE(true, true, true)
#undef HHB_GEMM_PCASE
    if (rc || splits == 1) return rc;
    launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits, int64_t(M * N), bias, D, ldd);
    return cuda_check("k_gemm_reduce launch");
  }
  Args a{};
  a.M = M;
  a.N = N;
  a.K = K;
  a.kb_total = kb_total;
  a.kb_per_split = (kb_total + splits - 1) / splits;
  a.idesc = instr_desc(false, bn, a_mn, b_mn);
  a.kb_switch = k_switch > 0 ? int(k_switch / 64) : 0;
  if (splits > 1) {
    a.D = workspace;
    a.ldd = N;
    a.split_stride = M * N;
    a.bias = nullptr;
  } else {
    a.D = D;
    a.ldd = ldd;
    a.split_stride = 0;
    a.bias = bias;
  }
#define HHB_GEMM_CASE(AM, BMN, DU)                                   \
  if (a_mn == AM && b_mn == BMN && dual == DU)                       \
    rc = launch_bn<false, AM, BMN, DU>(bn, ta, ta2, tb, a, splits, st);
  HHB_GEMM_CASE(false, false, false)
  HHB_GEMM_CASE(false, false, true)
  HHB_GEMM_CASE(false, true, false)
  HHB_GEMM_CASE(false, true, true)
  HHB_GEMM_CASE(true, false, false)
  HHB_GEMM_CASE(true, false, true)
  HHB_GEMM_CASE(true, true, false)
  HHB_GEMM_CASE(true, true, true)
#undef HHB_GEMM_CASE
  if (rc || splits == 1) return rc;
  launch_pdl(k_gemm_reduce, dim3(grid_1d(M * N, 256)), dim3(256), 0, st, M, N, (const float*)workspace, splits, int64_t(M * N), bias, D, ldd);
  return cuda_check("k_gemm_reduce launch");
}

int hhb_transpose(int32_t kind, int64_t rows, int64_t cols, const void* src, int64_t lds, void* dst, int64_t ldd,
                  void* stream) {
  if (rows <= 0 || cols <= 0) return HHB_OK;
  const dim3 grid{unsigned((cols + 31) / 32), unsigned((rows + 31) / 32), 1u};
  const dim3 block{32u, 8u, 1u};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  using namespace hhb::gemm;
  using bf = __nv_bfloat16;
  const float* sf = static_cast<const float*>(src);
  const bf* sb = static_cast<const bf*>(src);
  switch (kind) {
    case 0: launch_pdl(k_transpose<float, float, TR_PLAIN>, dim3(grid), dim3(block), 0, st, rows, cols, sf, lds, (float*)dst, ldd); break;
    case 1: launch_pdl(k_transpose<float, bf, TR_PLAIN>, dim3(grid), dim3(block), 0, st, rows, cols, sf, lds, (bf*)dst, ldd); break;
    case 2: launch_pdl(k_transpose<bf, bf, TR_PLAIN>, dim3(grid), dim3(block), 0, st, rows, cols, sb, lds, (bf*)dst, ldd); break;
    case 3: launch_pdl(k_transpose<float, bf, TR_SPLIT>, dim3(grid), dim3(block), 0, st, rows, cols, sf, lds, (bf*)dst, ldd); break;
    case 4: launch_pdl(k_transpose<bf, bf, TR_DUP>, dim3(grid), dim3(block), 0, st, rows, cols, sb, lds, (bf*)dst, ldd); break;
    default: return fail(HHB_EINVAL, "transpose kind");
  }
  return cuda_check("k_transpose launch");
}

int hhb_split_rows_bf16(int64_t rows, int64_t cols, const float* src, int64_t lds, void* dst, int64_t ldd,
                        void* stream) {
  if (rows <= 0 || cols <= 0) return HHB_OK;
  if (ldd < 2 * cols) return fail(HHB_EINVAL, "ldd < 2*cols");
  const dim3 grid{unsigned((cols + 255) / 256), unsigned(rows < 65535 ? rows : 65535), 1u};
  launch_pdl(hhb::gemm::k_split_rows, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      rows, cols, src, lds, static_cast<__nv_bfloat16*>(dst), ldd);
  return cuda_check("k_split_rows launch");
}

int hhb_split3_bf16(int64_t rows, int64_t cols, const float* src, int64_t lds, void* dst, int64_t ldd,
                    int64_t slot, int32_t order, void* stream) {
  if (rows <= 0 || cols <= 0) return HHB_OK;
  if (order == 2 ? (slot < rows || ldd < cols) : (order != 0 && order != 1) || slot < cols || ldd < 3 * slot)
    return fail(HHB_EINVAL, "split3 shape/order");
  const bool vec = cols % 8 == 0 && lds % 4 == 0 && ldd % 8 == 0 && slot % 8 == 0 &&
                   reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0;
  if (vec) {
    const int64_t total = rows * (cols / 8);
    launch_pdl(hhb::gemm::k_split3_rows_v8, dim3(grid_1d(total, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
        rows, cols / 8, src, lds, static_cast<__nv_bfloat16*>(dst), ldd, slot, order);
    return cuda_check("k_split3_rows_v8 launch");
  }
  const dim3 grid{unsigned((cols + 255) / 256), unsigned(rows < 65535 ? rows : 65535), 1u};
  launch_pdl(hhb::gemm::k_split3_rows, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      rows, cols, src, lds, static_cast<__nv_bfloat16*>(dst), ldd, slot, order);
  return cuda_check("k_split3_rows launch");
}

int hhb_cast_bf16(int64_t n, const float* src, void* dst, void* stream) {
  if (n <= 0) return HHB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t done = 0;
  if (reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 && n >= 8) {
    const int64_t n8 = n / 8;
    launch_pdl(hhb::gemm::k_cast_bf16_v8, dim3(grid_1d(n8, 256)), dim3(256), 0, st, n8, reinterpret_cast<const float4*>(src),
                                                                  static_cast<uint4*>(dst));
    done = n8 * 8;
  }
  if (done < n)
    launch_pdl(hhb::gemm::k_cast_bf16, dim3(grid_1d(n - done, 256)), dim3(256), 0, st, n - done, src + done,
                                                                    static_cast<__nv_bfloat16*>(dst) + done);
  return cuda_check("k_cast_bf16 launch");
}

static int col_chunks(int64_t rows) {
  return int(rows < hhb::gemm::kColChunks * 8 ? (rows + 7) / 8 : hhb::gemm::kColChunks);
}

int64_t hhb_col_sum_scratch(int64_t rows, int64_t cols) { return rows > 0 && cols > 0 ? col_chunks(rows) * cols : 0; }

int hhb_col_sum(int64_t rows, int64_t cols, const float* src, int64_t ld, double* out, double* scratch,
                void* stream) {
  if (rows <= 0 || cols <= 0) return HHB_OK;
  if (!scratch) return fail(HHB_EINVAL, "col_sum needs hhb_col_sum_scratch doubles of scratch");
  using namespace hhb::gemm;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int chunks = col_chunks(rows);
  const dim3 grid{unsigned((cols + 31) / 32), unsigned(chunks), 1u};
  const dim3 block{32u, 8u, 1u};
  launch_pdl(k_col_sum_part, dim3(grid), dim3(block), 0, st, rows, cols, src, ld, scratch);
  launch_pdl(k_col_sum_final, dim3(unsigned((cols + 127) / 128)), dim3(128), 0, st, cols, chunks, scratch, out);
  return cuda_check("k_col_sum launch");
}

int hhb_col_sum_ex(int64_t rows, int64_t cols, const float* src, int64_t ld, double* out64, float* out32,
                   double* scratch, void* stream) {
  if (cols <= 0) return HHB_OK;
  using namespace hhb::gemm;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (rows <= kColOnePass) {
    launch_pdl(k_col_sum_one, dim3(unsigned((cols + 31) / 32)), dim3(dim3(32u, 8u, 1u)), 0, st, rows, cols, src, ld, out64, out32);
    return cuda_check("k_col_sum_one launch");
  }
  if (!scratch) return fail(HHB_EINVAL, "col_sum_ex needs hhb_col_sum_scratch doubles of scratch");
  const int chunks = col_chunks(rows);
  const dim3 grid{unsigned((cols + 31) / 32), unsigned(chunks), 1u};
  launch_pdl(k_col_sum_part, dim3(grid), dim3(dim3(32u, 8u, 1u)), 0, st, rows, cols, src, ld, scratch);
  launch_pdl(k_col_sum_final_set, dim3(unsigned((cols + 127) / 128)), dim3(128), 0, st, cols, chunks, scratch, out64, out32);
  return cuda_check("k_col_sum_ex launch");
}

int hhb_sum_f64(int64_t n, const double* x, double scale, double* out64, float* out32, void* stream) {
  if (n < 0 || (n > 0 && !x)) return fail(HHB_EINVAL, "sum_f64: bad input");
  launch_pdl(hhb::gemm::k_sum_f64, dim3(1), dim3(1024), 0, static_cast<cudaStream_t>(stream), n, x, scale, out64, out32);
  return cuda_check("k_sum_f64 launch");
}

}  // extern "C"
