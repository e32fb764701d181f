/*
 * hhb200.h -- C ABI of the B200-native Hodgkin-Huxley hot path.
 *
 * The reference (arXiv 2601.21407 desk-scale package `hhengine`) has no native
 * code and no FFI: its boundary is the Python module API of
 * hhengine.dynamics / hhengine.adjoint.  This header is the library that a
 * drop-in for that API binds (through ctypes); each entry
 * point names the reference function it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch / C++ types.
 *   - Array pointers are DEVICE pointers unless a comment says "host".
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  No call allocates device memory: the
 *     caller pre-allocates every buffer (the Workspace idea of
 *     dynamics.py:388-406).
 *   - Return value: HHB_OK (0) or an error code; hhb_last_error() returns a
 *     thread-local message.  No C++ exception crosses the ABI.
 *   - dtype selects the arithmetic: HHB_F32 (MUFU fast path, the throughput
 *     build) or HHB_F64 (reference-order arithmetic, the parity build).  All
 *     floating arrays of one call share that dtype.
 *   - Layouts are the reference's own: time-major series [T][ld] (Trace,
 *     dynamics.py:269-270) and gate-major state [n_gates][ld]
 *     (NeuronState, dynamics.py:254-256).  Spikes are bitmaps, one uint32
 *     word per 32 neurons, bit i of word w = neuron 32*w + i.
 */
#ifndef HHB200_H
#define HHB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HHB_ABI_VERSION 3
#define HHB_MAX_GATES 8
#define HHB_MAX_CHANNELS 8

enum hhb_status {
  HHB_OK = 0,
  HHB_EINVAL = 22,   /* bad shape / argument / parameter table */
  HHB_ENOTSUP = 95,  /* combination not compiled in */
  HHB_ECUDA = 1000,  /* CUDA launch or runtime error */
  HHB_ECOMM = 1001   /* NCCL error (spike exchange) */
};

enum hhb_dtype { HHB_F32 = 0, HHB_F64 = 1 };

/* RateFn.kind (dynamics.py:36-38) */
enum hhb_rate_kind { HHB_RATE_LINOID = 0, HHB_RATE_EXP = 1, HHB_RATE_SIGMOID = 2 };

/* SurrogateSpec.kind (adjoint.py:37-46) */
enum hhb_surrogate_kind { HHB_SUR_SIGMOID_DERIV = 0, HHB_SUR_RECTANGULAR = 1 };

/* RateFn(kind, a, v0, b)                                 dynamics.py:32-54 */
typedef struct {
  int32_t kind;
  int32_t reserved;
  double a, v0, b;
} hhb_rate_t;

/* GateSpec(name, alpha, beta, exponent), plus its owning channel index
 * (HHParams.gate_layout, dynamics.py:190-193)            dynamics.py:96-108 */
typedef struct {
  hhb_rate_t alpha, beta;
  int32_t exponent;
  int32_t channel;
} hhb_gate_t;

/* ChannelSpec(name, g_max, e_rev, gates): its gates are the contiguous run
 * gates[gate_begin .. gate_begin+gate_count) of hhb_params_t  dynamics.py:128-142 */
typedef struct {
  double g_max, e_rev;
  int32_t gate_begin, gate_count;
} hhb_channel_t;

/* HHParams (dynamics.py:162-188), flattened. Host pointer at every call. */
typedef struct {
  int32_t n_gates, n_channels;
  double c_m, dt, v_theta, v_rest, rate_scale;
  hhb_gate_t gates[HHB_MAX_GATES];
  hhb_channel_t channels[HHB_MAX_CHANNELS];
} hhb_params_t;

/* SurrogateSpec(kind, width)                             adjoint.py:33-48 */
typedef struct {
  int32_t kind;
  int32_t reserved;
  double width;
} hhb_surrogate_t;

int hhb_abi_version(void);
const char* hhb_last_error(void);
/* Validate a parameter table (the ConfigurationError checks of
 * dynamics.py:50-54, :106-108, :140-142, :178-188).  Host-only. */
int hhb_check_params(const hhb_params_t* params);

/*
 * hhb_forward -- replaces simulate() (dynamics.py:541-586) and hh_step()
 * (dynamics.py:443-529): runs n_steps fused HH steps for n neurons in one
 * launch with the state in registers.
 *
 *   v_in [n], g_in [n_gates][g_ld]          state before step 0
 *   v_fin, g_fin (same layout)              state after the last step; may
 *                                           alias v_in / g_in (in place)
 *   i_ext + (i_st, i_sn)                    current of neuron j at step t is
 *                                           i_ext[t*i_st + j*i_sn]; (ld,1) dense,
 *                                           (0,1) per-neuron constant, (1,0) per
 *                                           step scalar, (0,0) one scalar
 *   v_out [n_steps][v_ld]      or NULL      Trace.v_series (potential after step t)
 *   spk_out [n_steps][spk_ld]  or NULL      Trace.spike_series as bitmap words
 *   ckpt [ceil(T/K)][1+n_gates][ckpt_ld]    state BEFORE steps 0, K, 2K, ...
 *        or NULL, K = ckpt_every            (adjoint.py:330-336 stored states)
 *   first_bad (device int64)                atomicMin(step_base + t) over the
 *                                           first non-finite V' of every neuron;
 *                                           caller initialises it to INT64_MAX
 *                                           (NumericalOverflowError, dynamics.py:526-527)
 */
int hhb_forward(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                const void* v_in, const void* g_in, int64_t g_ld,
                void* v_fin, void* g_fin,
                const void* i_ext, int64_t i_st, int64_t i_sn,
                void* v_out, int64_t v_ld,
                uint32_t* spk_out, int64_t spk_ld,
                void* ckpt, int64_t ckpt_every, int64_t ckpt_ld,
                int64_t step_base, int64_t* first_bad, void* stream);

/* hhb_forward plus spk_val[n_steps][spk_val_ld] (dtype of V, NULL = off): the
 * spike flags as 0/1 values, the SNN layer's differentiable spike output,
 * written by the forward kernel itself (no bitmap round trip);
 * step_base_dev (NULL = off): *step_base_dev is added to step_base on the
 * device (first_bad indices inside a replayed CUDA graph); and sq_partials
 * (NULL = off): per-block partial sums of V'^2 over the launch, the fused
 * forward half of an MSE(V, 0) loss (learn.py:80-88) -- hhb_forward_partials(n)
 * doubles zeroed by the caller, summed by it in any fixed order. */
int hhb_forward_ex(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                   const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                   const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld,
                   uint32_t* spk_out, int64_t spk_ld, void* spk_val, int64_t spk_val_ld, void* ckpt,
                   int64_t ckpt_every, int64_t ckpt_ld, int64_t step_base, int64_t* first_bad,
                   const int64_t* step_base_dev, double* sq_partials, void* stream);
/* hhb_forward_ex plus spk_bf16[n_steps][spk_bf16_ld] (NULL = off): the spike
 * flags again as bf16 0/1 values (0x3F80 = 1.0), so a stacked layer's spikes
 * reach the next layer's bf16 tcgen05 GEMM as its A operand without a cast
 * pass (learn.py:210-211 applied to spikes, exact in bf16). */
int hhb_forward_ex2(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                    const void* v_in, const void* g_in, int64_t g_ld, void* v_fin, void* g_fin,
                    const void* i_ext, int64_t i_st, int64_t i_sn, void* v_out, int64_t v_ld,
                    uint32_t* spk_out, int64_t spk_ld, void* spk_val, int64_t spk_val_ld, void* ckpt,
                    int64_t ckpt_every, int64_t ckpt_ld, int64_t step_base, int64_t* first_bad,
                    const int64_t* step_base_dev, double* sq_partials, void* spk_bf16, int64_t spk_bf16_ld,
                    void* stream);
int64_t hhb_forward_partials(int64_t n);
/*
 * hhb_forward_poisson -- hhb_forward with the BASELINE config-2 stimulus
 * I[t][j] = amp * Poisson(lam) drawn inside the kernel (Philox-4x32-10 keyed by
 * (seed, neuron_base + j, (step_base + t) / 4)): bit-identical to running
 * hhb_poisson_current into a buffer and hhb_forward on it, without the
 * 4 B/neuron-step write and re-read.  Other arguments as hhb_forward.
 */
int hhb_forward_poisson(const hhb_params_t* params, int32_t dtype, int64_t n, int64_t n_steps,
                        const void* v_in, const void* g_in, int64_t g_ld,
                        void* v_fin, void* g_fin,
                        uint64_t seed, int64_t neuron_base, double lam, double amp,
                        void* v_out, int64_t v_ld,
                        uint32_t* spk_out, int64_t spk_ld,
                        void* ckpt, int64_t ckpt_every, int64_t ckpt_ld,
                        int64_t step_base, int64_t* first_bad, void* stream);

/*
 * hhb_backward -- replaces backward_through_time() (adjoint.py:281-365) and
 * hh_step_backward() (adjoint.py:102-194).  One launch runs the whole reverse
 * sweep: for each checkpoint segment, newest first, it recomputes the segment
 * states into seg_buf (skipped when ckpt_every == 1: full storage) and then
 * applies the exact adjoint step by step.
 *
 *   ckpt, ckpt_every, ckpt_ld           as written by hhb_forward
 *   seg_buf [ckpt_every][1+n_gates][ckpt_ld] scratch, may be NULL if ckpt_every == 1
 *   seed_v  [T][seed_v_ld]   or NULL    dL/dV of trace row t (added before step t)
 *   seed_spk[T][seed_spk_ld] or NULL    dL/dspike of trace row t
 *   adj_v [n], adj_g [n_gates][adj_g_ld] in: adjoint after the last step;
 *                                        out: adjoint of the state before step 0
 *   d_i [T][d_i_ld]          or NULL    dL/di_ext per neuron and step
 *   d_params [1+n_channels]  (double)   += {d_c_m, d_g_max[0..]}: deterministic
 *                                       two-pass reduction through `partials`
 *   partials  (double) hhb_backward_partials(n, dtype) doubles of scratch
 *   first_bad (device int64)            atomicMax(step_base + t) of the first
 *                                       non-finite adjoint in processing order;
 *                                       caller initialises it to -1
 *                                       (GradientOverflowError, adjoint.py:190-191)
 */
int hhb_backward(const hhb_params_t* params, const hhb_surrogate_t* surrogate, int32_t dtype,
                 int64_t n, int64_t n_steps,
                 const void* i_ext, int64_t i_st, int64_t i_sn,
                 const void* ckpt, int64_t ckpt_every, int64_t ckpt_ld, void* seg_buf,
                 const void* seed_v, int64_t seed_v_ld,
                 const void* seed_spk, int64_t seed_spk_ld,
                 void* adj_v, void* adj_g, int64_t adj_g_ld,
                 void* d_i, int64_t d_i_ld,
                 double* d_params, double* partials,
                 int64_t step_base, int64_t* first_bad, void* stream);
/* doubles of `partials` scratch hhb_backward needs for n neurons */
/* hhb_backward plus the SNN layer's outputs (float only, each optional):
 * d_i_hi / d_i_lo [n_steps][d_split_ld] uint16 bf16 bit patterns with
 * hi = bf16(dI) and lo = bf16(dI - hi) -- the operands of the bf16x2 gradient
 * GEMMs (hhb_gemm_ex), so dI never round-trips through fp32 for them; with
 * d_split_group > 0 neuron i sits at (i / group) * d_split_pitch + i % group
 * (rows of `group` neurons padded to a 16-byte pitch) -- and
 * d_i_sum[n] += sum over the steps of dI (the bias gradient before the
 * batch sum, learn.py:273); seed_v_scale (device float, NULL = 1): seed_v is
 * multiplied by *seed_v_scale as it is read -- with seed_v pointing at the V'
 * values themselves (e.g. the checkpoint v-planes one slot ahead), the fused
 * backward half of MSE(V, 0), seed = 2 V g / numel. */
int hhb_backward_ex(const hhb_params_t* params, const hhb_surrogate_t* surrogate, int32_t dtype,
                    int64_t n, int64_t n_steps, const void* i_ext, int64_t i_st, int64_t i_sn,
                    const void* ckpt, int64_t ckpt_every, int64_t ckpt_ld, void* seg_buf,
                    const void* seed_v, int64_t seed_v_ld, const void* seed_spk, int64_t seed_spk_ld,
                    void* adj_v, void* adj_g, int64_t adj_g_ld, void* d_i, int64_t d_i_ld,
                    double* d_params, double* partials, int64_t step_base, int64_t* first_bad,
                    void* d_i_hi, void* d_i_lo, int64_t d_split_ld, int64_t d_split_group,
                    int64_t d_split_pitch, float* d_i_sum, const float* seed_v_scale, void* stream);
int64_t hhb_backward_partials(int64_t n, int32_t dtype);

/* ---- elementary ops (dynamics.py:324-381, adjoint.py:60-66) ------------ */

/* gate_rates(): alpha, beta of one gate at n potentials, times rate_scale */
int hhb_gate_rates(const hhb_gate_t* gate, double rate_scale, int32_t dtype, int64_t n,
                   const void* v, void* alpha, void* beta, void* stream);
/* RateFn.__call__ (with_slope=0) or RateFn.deriv (with_slope=1) of one rate */
int hhb_rate_eval(const hhb_rate_t* rate, int32_t with_slope, int32_t dtype, int64_t n,
                  const void* v, void* out, void* stream);
/* gate_step(): exponential Euler p_inf + (p - p_inf) exp(-dt (alpha+beta)) */
int hhb_gate_step(int32_t dtype, int64_t n, const void* p, const void* alpha, const void* beta,
                  double dt, void* out, void* stream);
/* ionic_current(): sum_X g_X prod p^k (V - E_X) */
int hhb_ionic_current(const hhb_params_t* params, int32_t dtype, int64_t n, const void* v,
                      const void* g, int64_t g_ld, void* out, void* stream);
/* spike_detect(): v_prev < theta <= v_new, one byte per neuron */
int hhb_spike_detect(int32_t dtype, int64_t n, const void* v_prev, const void* v_new,
                     double theta, uint8_t* out, void* stream);
/* surrogate_grad() at threshold offsets u */
int hhb_surrogate_grad(const hhb_surrogate_t* surrogate, int32_t dtype, int64_t n,
                       const void* u, void* out, void* stream);

/* ---- data formats either side of the step ------------------------------ */

/* bitmap [T][words] -> bool bytes [T][n] (Trace.spike_series) */
int hhb_unpack_spikes(const uint32_t* bits, int64_t words_ld, int64_t n_steps, int64_t n,
                      uint8_t* out, int64_t out_ld, void* stream);
/* the same as float 0/1 (the SNN layer's spike output) */
int hhb_unpack_spikes_f32(const uint32_t* bits, int64_t words_ld, int64_t n_steps, int64_t n,
                          float* out, int64_t out_ld, void* stream);
/* Synthetic stimulus (BASELINE config 2): out[t][j] = amp * Poisson(lam), Philox-4x32-10
 * keyed by (seed, global neuron j + neuron_base, global step t + step_base) so a
 * sharded population draws the same numbers as an unsharded one. */
int hhb_poisson_current(int32_t dtype, int64_t n, int64_t n_steps, uint64_t seed,
                        int64_t neuron_base, int64_t step_base, double lam, double amp,
                        void* out, int64_t ld, void* stream);

/* ---- dense synaptic projection (tcgen05) ---------------------------------- */

enum hhb_gemm_in { HHB_GEMM_BF16 = 0, HHB_GEMM_TF32 = 1 };

/* D[M][ldd] (fp32) = A[M][K] . B[N][K]^T (+ bias[N]) on the 5th-gen tensor
 * cores (tcgen05.mma, fp32 accumulation in TMEM, TMA-fed 128B-swizzled smem).
 * Replaces DenseLayer.__call__ (learn.py:210-211) and the gradient einsum
 * (learn.py:272) of the HH readout/SNN layer.  A and B are K-major (row
 * pitch lda/ldb elements, 16-byte aligned): bf16 for HHB_GEMM_BF16, fp32
 * read as tf32 for HHB_GEMM_TF32.  splits > 1 splits K over CTAs into fp32
 * partial slices (workspace: hhb_gemm_workspace floats) summed in a fixed
 * order -- deterministic. */
int hhb_gemm(int32_t in_kind, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
             const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd,
             int32_t splits, float* workspace, void* stream);
int64_t hhb_gemm_workspace(int64_t M, int64_t N, int32_t splits);
/* bf16 generalisation of hhb_gemm for the layer gradients (learn.py:264-274):
 *   D[M][ldd] = (A (+ A2)) . B^T (+ bias)
 * HHB_GEMM_A_MN: A is stored MN-major, A[k][m] at A + k*lda + m (else
 * A[m][k] at A + m*lda + k); HHB_GEMM_B_MN likewise for B[k][n].  A2 (same
 * layout as A, or NULL) is accumulated into the same tensor-memory tile: with
 * A/A2 the bf16 hi/lo halves of an fp32 operand the product carries ~16
 * mantissa bits of it.  So dW = dI^T X and dX = dI W read dI, X and W in
 * their natural row-major layouts, without transposed or split copies. */
enum hhb_gemm_flags { HHB_GEMM_A_MN = 1, HHB_GEMM_B_MN = 2, HHB_GEMM_A_F32 = 4, HHB_GEMM_A_SPLIT = 8 };
/* HHB_GEMM_A_F32: A is fp32 (K-major, lda in floats), rounded to bf16 on chip
 * inside the GEMM (TMA -> converter warps -> tensor cores): D = bf16(A) . B^T
 * (+ bias), bit-identical to casting A first; with HHB_GEMM_A_SPLIT, A2 is
 * B_lo (bf16, B's layout) and D = A_hi.B + A_lo.B + A_hi.B_lo, A_hi/A_lo the
 * bf16 hi/lo split of A (the fp32-class projection of DenseLayer, learn.py:
 * 210-211, without the separate split pass).  K-major B, M >= 512. */
int hhb_gemm_ex(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2, int64_t lda,
                const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits,
                float* workspace, void* stream);
/* hhb_gemm_ex with k_switch > 0 (a multiple of 64 below K, K-major A): A2 is
 * not a second addend but the A source for k >= k_switch, read at
 * k - k_switch -- the K-concatenation [A | A2] of two operands without a
 * copy.  The fp32-class input gradient uses it: [dI_hi | dI_lo] then dI_hi
 * against [W_hi; W_hi; W_lo], three products in one GEMM. */
int hhb_gemm_ex2(int32_t flags, int64_t M, int64_t N, int64_t K, const void* A, const void* A2, int64_t lda,
                 const void* B, int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits,
                 float* workspace, int64_t k_switch, void* stream);
/* The fp32-A GEMM of hhb_gemm_ex (HHB_GEMM_A_F32 [| HHB_GEMM_A_SPLIT with
 * B_lo]) that also writes the operand it converted on chip: xs[m][k] = bf16
 * hi of A, xs[m][xs_slot + k] = lo (B_lo given) -- the layer's weight gradient
 * reads them, so the fp32-class projection needs no separate split pass.
 * xs NULL: not written.  K, xs_ld, xs_slot multiples of 8. */
int hhb_gemm_f32a(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const void* B, const void* B_lo,
                  int64_t ldb, const float* bias, float* D, int64_t ldd, int32_t splits, float* workspace,
                  void* xs, int64_t xs_ld, int64_t xs_slot, void* stream);
/* Weight-gradient form: D[m][n] = sum_k (A + A_lo)[k][m] . B_hi[k][n] (+ A[k][m] .
 * B_lo[k][n] when split_b), A / A_lo bf16 MN-major (A[k][m] at A + k*lda + m: the
 * hi / lo halves of the layer's dI), B fp32 MN-major (B[k][n] at B + k*ldb + n:
 * the layer input x), rounded (split_b: and split into bf16 hi / lo) on chip --
 * the dW of proj="bf16x3" (three products) or proj="bf16" (two) (learn.py:272)
 * in one GEMM over the fp32 x.  M >= 512, N > 128. */
int hhb_gemm_f32b(int64_t M, int64_t N, int64_t K, const void* A, const void* A_lo, int64_t lda, const float* B,
                  int64_t ldb, int32_t split_b, float* D, int64_t ldd, int32_t splits, float* workspace,
                  void* stream);
/* dst[c][r] = src[r][c]; kind 0: fp32->fp32, 1: fp32->bf16, 2: bf16->bf16,
 * 3: fp32 -> bf16 hi at [c][r] and lo = x - hi at [c][rows + r] (bf16x2 split),
 * 4: bf16 -> bf16 written to [c][r] and [c][rows + r].  Kinds 3 + 4 turn a
 * product with one fp32 operand into one bf16 GEMM with K doubled whose
 * result carries ~16 mantissa bits of that operand. */
int hhb_transpose(int32_t kind, int64_t rows, int64_t cols, const void* src, int64_t lds,
                  void* dst, int64_t ldd, void* stream);
/* row-wise bf16x2 split: dst[r][c] = hi(src[r][c]), dst[r][cols + c] = lo */
int hhb_split_rows_bf16(int64_t rows, int64_t cols, const float* src, int64_t lds, void* dst,
                        int64_t ldd, void* stream);
/* row-wise three-slot bf16 split (the fp32-class "bf16x3" projection):
 * slots of `slot` (>= cols) elements per row; order 0: [hi | lo | hi],
 * order 1: [hi | hi | lo]; order 2: three row blocks [hi; hi; lo] of `slot`
 * (>= rows) rows of pitch ldd (the input gradient's stacked B operand).  A bf16 GEMM over K = 3 slot of an order-0 A and
 * an order-1 B is x_h.W_h + x_l.W_h + x_h.W_l (~16 mantissa bits of both
 * operands; replaces the float64 x @ W.T of DenseLayer, learn.py:210-211). */
int hhb_split3_bf16(int64_t rows, int64_t cols, const float* src, int64_t lds, void* dst,
                    int64_t ldd, int64_t slot, int32_t order, void* stream);
int hhb_cast_bf16(int64_t n, const float* src, void* dst, void* stream);
/* out[c] += sum_r src[r][c] (bias gradient, learn.py:273), fixed-order two-pass
 * reduction through hhb_col_sum_scratch(rows, cols) doubles of scratch */
int hhb_col_sum(int64_t rows, int64_t cols, const float* src, int64_t ld, double* out,
                double* scratch, void* stream);
int64_t hhb_col_sum_scratch(int64_t rows, int64_t cols);
/* out64[c] / out32[c] = sum_r src[r][c] (assigned, either output may be NULL):
 * the bias gradient of an HH layer (learn.py:273, db = d_i.sum over (t, b)) in
 * one launch when rows <= 512 (the per-neuron BPTT sums of a batch), else two
 * through hhb_col_sum_scratch doubles of scratch; fixed order (deterministic). */
int hhb_col_sum_ex(int64_t rows, int64_t cols, const float* src, int64_t ld, double* out64, float* out32,
                   double* scratch, void* stream);
/* out64[0] / out32[0] = scale * sum of x[0..n) in a fixed order (one block):
 * the fused MSE(V, 0) loss of an HH layer from the forward kernel's per-block
 * partials (learn.py:80-84, mean of V^2) -- replaces sum + divide + cast. */
int hhb_sum_f64(int64_t n, const double* x, double scale, double* out64, float* out32, void* stream);

/* ---- LIF baseline (dynamics.py:227-244, :532-538; adjoint.py:197-227) ------ */

/* n_steps of n LIF neurons in one launch: v' = v + (dt/tau)(i - v), spike =
 * v' >= v_theta, v = spike ? v_reset : v'.  i_ext[t*i_st + j*i_sn]; v_out
 * [n_steps][n] and spk_out uint8 [n_steps][n] optional; v_fin [n]. */
int hhb_lif_forward(int32_t dtype, int64_t n, int64_t n_steps, double tau, double dt, double v_theta,
                    double v_reset, const void* v_in, const void* i_ext, int64_t i_st, int64_t i_sn,
                    void* v_out, uint8_t* spk_out, void* v_fin, void* stream);
/* lif_step_backward: d_v_pre = g_v_out ((1 - s) + (v_reset - v_pre) sg) +
 * g_spike sg (g_spike may be NULL), d_v_in = d_v_pre (1 - k), d_i = d_v_pre k;
 * *bad set >= 0 when d_v_in is non-finite (GradientOverflowError). */
int hhb_lif_backward(int32_t dtype, int64_t n, double tau, double dt, double v_theta, double v_reset,
                     const hhb_surrogate_t* surrogate, const void* v, const void* i_ext, int64_t i_sn,
                     const void* g_v_out, const void* g_spike, void* d_v_in, void* d_i, int64_t* bad,
                     void* stream);

/* ---- training plumbing (learn.py) ----------------------------- */

/* psp_filter (learn.py:52-55): y[t][c] = causal FIR of x[.][c] with taps[0..ntaps)
 * (device float64 array), in scipy.signal.lfilter's direct-form-II-transposed
 * operation order; x, y [steps][cols] of dtype. */
int hhb_psp_filter(int32_t dtype, int64_t steps, int64_t cols, int32_t ntaps, const double* taps_dev,
                   const void* x, void* y, void* stream);

/* ReadoutModel dendrite layer (learn.py:238-247, one output channel):
 * drive[t][b] = bias[0] + sum_c x(b,t,c) w[c], x(b,t,c) at x[b*x_sb + t*x_st + c];
 * drive is written time-major [steps][batch] (the HH i_series).  w, bias device. */
int hhb_readout_drive(int32_t dtype, int64_t batch, int64_t steps, int64_t n_in, const void* x, int64_t x_sb,
                      int64_t x_st, const void* w, const void* bias, void* drive, void* stream);
/* ReadoutModel.grads weight part (learn.py:269-273): d_w[c] = sum d_drive[t][b] x(b,t,c),
 * d_b[0] = sum d_drive; deterministic (fixed-order two-stage reduction) into a
 * caller workspace of hhb_readout_workspace(dtype, n_in) bytes. */
int64_t hhb_readout_workspace(int32_t dtype, int64_t n_in);
int hhb_readout_grad(int32_t dtype, int64_t batch, int64_t steps, int64_t n_in, const void* x, int64_t x_sb,
                     int64_t x_st, const void* d_drive, void* d_w, void* d_b, void* workspace, int64_t ws_bytes,
                     void* stream);

/* ---- multicompartment neurons (morphology.py) ---------------- */

/* T steps of `batch` independent multicompartment neurons on one compartment
 * graph (simulate_morphology, morphology.py:144-166): every step, compartment
 * c receives i_ext[t][c][b] + axial, axial = sum over edges e in order of
 * g_e (V_b - V_a) (+ for c == a, - for c == b) on the previous step's
 * potentials (axial_current, :115-124), then takes one HH step with its
 * channel table tables[table_of[c]] (morph_step, :127-141).  Layouts:
 * i_ext / v_out [n_steps][n_comp][batch], spk_out uint8 likewise, v [n_comp]
 * [batch], gates [n_comp][HHB_MAX_GATES][batch] (a compartment uses its first
 * n_gates rows).  n_steps == 0 writes the axial current of (v_in) into
 * ax_out [n_comp][batch] and nothing else.  Limits: 32 compartments, 64
 * edges, 4 distinct tables per call.  first_bad: atomicMin of the first
 * non-finite step (NumericalOverflowError). */
int hhb_morph_forward(int32_t dtype, int32_t n_tables, const hhb_params_t* tables, int32_t n_comp,
                      const int32_t* table_of, int32_t n_edges, const int32_t* edge_a,
                      const int32_t* edge_b, const double* g_axial, int64_t batch, int64_t n_steps,
                      const void* i_ext, const void* v_in, const void* g_in, void* v_fin, void* g_fin,
                      void* v_out, uint8_t* spk_out, void* ax_out, int64_t step_base, int64_t* first_bad,
                      void* stream);

/* ---- recurrent network (BASELINE config 5) ---------------------------------- */

/* Per-step input of the cortex network (cortex.py:283-301) for n local
 * neurons: arrived = ring[t % depth][i] * w_scale (int64 fixed point, row then
 * zeroed), psp = psp*decay + arrived + background, cur = psp (+ extra).
 * bg_mode 0: none; 1: bg[i] supplied (e.g. the reference RNG's sample);
 * 2: compound Poisson N*mu + sigma*sqrt(N)*z, N ~ Poisson(lam[i]) drawn with
 * Philox keyed by (seed, neuron_base + i, t). */
int hhb_cortex_input(int32_t dtype, int64_t n, int64_t t, int64_t depth, int64_t* ring, void* psp,
                     double decay, int32_t bg_mode, const void* bg, const double* lam, double mu,
                     double sigma, uint64_t seed, int64_t neuron_base, const void* extra, void* cur,
                     double w_scale, void* stream);
/* Delayed spike delivery (SpikeBuffer.enqueue, cortex.py:248-250, 304-308):
 * for every set bit s of bits[0..words) (global source ids) and every synapse
 * j in offsets[s] .. offsets[s+1]: ring[(t + delays[j]) % depth][targets[j]]
 * += weights_fx[j] (int64 atomics: order-independent, deterministic). */
int hhb_spike_deliver(int64_t words, const uint32_t* bits, const int64_t* offsets,
                      const int32_t* targets, const int32_t* weights_fx, const int32_t* delays,
                      int64_t t, int64_t depth, int64_t n_local, int64_t* ring, void* stream);
/* CUDA-graph forms: the step index is read from device memory t_dev (when
 * non-NULL, t is ignored), so one captured network step replays for every t;
 * hhb_cortex_tick adds 1 to *t_dev (the last node of a captured step). */
int hhb_cortex_input_dev(int32_t dtype, int64_t n, int64_t t, const int64_t* t_dev, int64_t depth,
                         int64_t* ring, void* psp, double decay, int32_t bg_mode, const void* bg,
                         const double* lam, double mu, double sigma, uint64_t seed, int64_t neuron_base,
                         const void* extra, void* cur, double w_scale, void* stream);
int hhb_spike_deliver_dev(int64_t words, const uint32_t* bits, const int64_t* offsets,
                          const int32_t* targets, const int32_t* weights_fx, const int32_t* delays,
                          int64_t t, const int64_t* t_dev, int64_t depth, int64_t n_local, int64_t* ring,
                          void* stream);
/* The whole network step loop of one rank in ONE cooperative launch
 * (cortex.py:273-310 x steps; float32 neurons, JIT module): ring drain + PSP +
 * Philox background (bg_mode 0 none / 2 philox, as hhb_cortex_input_dev), the
 * HH step, the spike bitmap and the synapse delivery; one block per
 * 256-neuron tile, one grid barrier per step (barrier: one device uint32 of
 * scratch), n <= 65536.  Synapse rows must be sorted by target: segments[s][k]
 * (int64, n_sources x (tiles + 1), tiles = ceil(n / 256)) is the index of the
 * first synapse of row s with target >= 256 k, so a tile delivers only its
 * own segment of each spiking row.  bits: [2][words] ping-pong, or with
 * record != 0 [steps][words] -- the spike words of every step.  timing
 * (NULL = off): [steps][tiles][4] %globaltimer stamps per block (step start,
 * spikes written, barrier passed, delivery done) for profiling.  Bit-identical to stepping
 * the same network with the per-step kernels; HHB_ENOTSUP when the JIT or
 * cooperative launches are unavailable. */
int hhb_cortex_run(const hhb_params_t* params, int64_t n, int64_t steps, int64_t t0, int64_t depth, int64_t* ring,
                   float* psp, double decay, int32_t bg_mode, const double* lam, double mu, double sigma,
                   uint64_t seed, int64_t neuron_base, double w_scale, float* v, float* g, int64_t g_ld,
                   uint32_t* bits, int32_t record, int64_t words, const int64_t* segments, int64_t tiles,
                   const int32_t* targets, const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad,
                   uint32_t* barrier, uint64_t* timing, void* stream);
/* Thalamic drive of run_network (cortex.py:398-429) drawn on the device: the
 * thalamic synapses in CSR by target (offsets [n + 1] local positions,
 * weights of the network's dtype); synapse k (global position id_base + k)
 * fires at step t in [t_on, t_off) iff word (k mod 4) of the Philox-4x32-10
 * block ((id_base + k) / 4, t) under key `seed` is < threshold (= lam 2^32,
 * the reference's rng.random() < lam).  The current of neuron i is the sum of
 * its firing synapses' weights in row order (deterministic, the same for any
 * sharding); it is added to that step's current only (not to the PSP). */
typedef struct {
  const int64_t* offsets;
  const void* weights;
  int64_t id_base;
  int64_t t_on, t_off;
  uint32_t threshold;
  uint32_t reserved;
  uint64_t seed;
} hhb_thalamic_t;
/* extra[i] = the thalamic current of step t (*t_dev if t_dev != NULL) for the
 * n local neurons; 0 outside [t_on, t_off).  Pass extra to hhb_cortex_input. */
int hhb_thalamic_drive(int32_t dtype, int64_t n, int64_t t, const int64_t* t_dev, const hhb_thalamic_t* thal,
                       void* extra, void* stream);
/* hhb_cortex_run with the thalamic drive inside the persistent kernel
 * (thal NULL = hhb_cortex_run); float32 weights. */
int hhb_cortex_run_ex(const hhb_params_t* params, int64_t n, int64_t steps, int64_t t0, int64_t depth, int64_t* ring,
                      float* psp, double decay, int32_t bg_mode, const double* lam, double mu, double sigma,
                      uint64_t seed, int64_t neuron_base, double w_scale, float* v, float* g, int64_t g_ld,
                      uint32_t* bits, int32_t record, int64_t words, const int64_t* segments, int64_t tiles,
                      const int32_t* targets, const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad,
                      uint32_t* barrier, uint64_t* timing, const hhb_thalamic_t* thal, void* stream);
/* hhb_cortex_run for `replicas` (1..16) independent copies of the network in
 * one launch (CortexReplicas): replica r's v / psp at r * ld (g rows: g_ld >=
 * replicas * ld), its ring at r * depth * ld, its spike words at r * words of
 * each step's [replicas][words] block, its background key seed + r. */
int hhb_cortex_run_replicas(const hhb_params_t* params, int64_t replicas, int64_t ld, int64_t n, int64_t steps,
                            int64_t t0, int64_t depth, int64_t* ring, float* psp, double decay, int32_t bg_mode,
                            const double* lam, double mu, double sigma, uint64_t seed, int64_t neuron_base,
                            double w_scale, float* v, float* g, int64_t g_ld, uint32_t* bits, int32_t record,
                            int64_t words, const int64_t* segments, int64_t tiles, const int32_t* targets,
                            const int32_t* weights_fx, const int32_t* delays, int64_t* first_bad, uint32_t* barrier,
                            uint64_t* timing, void* stream);

/* Spike raster -> event list (SpikeRecord, cortex.py:422-438):
 * bits [steps][words] (bit i of word w = neuron 32 w + i; neurons >= n ignored).
 * hhb_spike_event_counts writes each step's event count; with offsets = the
 * exclusive scan of the counts, hhb_spike_events writes the events sorted by
 * (step, neuron) -- NumPy nonzero's order over the unpacked raster. */
int hhb_spike_event_counts(int64_t steps, int64_t words, const uint32_t* bits, int64_t n, int64_t* counts,
                           void* stream);
int hhb_spike_events(int64_t steps, int64_t words, const uint32_t* bits, int64_t n, const int64_t* offsets,
                     int32_t* out_step, int32_t* out_neuron, void* stream);

int hhb_cortex_tick(int64_t* t_dev, void* stream);
/* hhb_spike_deliver_dev in two kernels for the sparse per-step case: one
 * block lists the spiking sources (ascending) with the prefix of their row
 * lengths, then every (spike, synapse) pair gets its own thread.  Same ring
 * (bit-identical: integer atomics).  scratch: hhb_spike_scratch(words * 32)
 * int64 of device memory. */
int hhb_spike_deliver_flat(int64_t words, const uint32_t* bits, const int64_t* offsets,
                           const int32_t* targets, const int32_t* weights_fx, const int32_t* delays,
                           int64_t t, const int64_t* t_dev, int64_t depth, int64_t n_local, int64_t* ring,
                           int64_t* scratch, void* stream);
int64_t hhb_spike_scratch(int64_t n_sources);

/* ---- multi-GPU spike exchange ----------------------------
 * Replaces the single-process visibility of every spike in step_network
 * (cortex.py:273-310, :304-308): with the network sharded by target neuron
 * over `world` GPUs, each step every rank contributes its words_per_rank
 * bitmap words and receives all of them (ncclAllGather on `stream`, NVLink /
 * NVSwitch inside a node; capturable into CUDA graphs).  NCCL is loaded at
 * run time; hhb_spk_exchange_available() is 0 without it (HHB_ENOTSUP). */
typedef struct hhb_exchange hhb_exchange_t;
int hhb_spk_exchange_available(void);
/* rank 0 creates the 128-byte id (host buffer) and shares it out of band */
int hhb_spk_exchange_unique_id(void* id, int64_t bytes);
int hhb_spk_exchange_init(const void* id, int32_t rank, int32_t world, int64_t words_per_rank,
                          hhb_exchange_t** out);
/* global_words[r * words_per_rank + i] = rank r's local_words[i] */
int hhb_spk_exchange_allgather(hhb_exchange_t* ex, const uint32_t* local_words, uint32_t* global_words,
                               void* stream);
/* spk_step: the all-gather fused with hhb_spike_deliver_flat of the gathered
 * bitmap into this rank's ring (words_global <= world * words_per_rank) */
int hhb_spk_step(hhb_exchange_t* ex, const uint32_t* local_words, uint32_t* global_words, int64_t words_global,
                 const int64_t* offsets, const int32_t* targets, const int32_t* weights_fx, const int32_t* delays,
                 int64_t t, const int64_t* t_dev, int64_t depth, int64_t n_local, int64_t* ring, int64_t* scratch,
                 void* stream);
/* HHB_OK, or HHB_ECOMM with the NCCL asynchronous error (ncclCommGetAsyncError) */
int hhb_spk_exchange_status(hhb_exchange_t* ex);
/* abort (after a timeout / error: unblocks pending collectives) or destroy; both free ex */
int hhb_spk_exchange_abort(hhb_exchange_t* ex);
int hhb_spk_exchange_destroy(hhb_exchange_t* ex);
/* `replicas` independent copies of one network on one GPU ("replicas x speed",
 * PAPER.md:193; SPEC data-parallel batching): per-replica state rows of n_pad
 * (= 32-aligned neuron count) neurons, ring [replicas][depth][n_pad], bitmap
 * [replicas][n_pad/32] words, Philox background keyed by (seed + replica,
 * neuron, step), step index on the device.  phase 0 = the input of every
 * replica (ring drain, PSP, background: cortex.py:283-301); phase 1 =
 * compaction + delivery of every replica's spikes (cortex.py:304-308); the HH
 * step of all replicas runs in between as one population (hhb_forward_ex).
 * scratch: replicas * hhb_spike_scratch(n_pad) int64. */
int hhb_cortex_step_batch(int32_t dtype, int64_t replicas, int64_t n_pad, int64_t words, const int64_t* t_dev,
                          int64_t depth, int64_t* ring, void* psp, double decay, const double* lam, double mu,
                          double sigma, uint64_t seed, void* cur, double w_scale, const uint32_t* bits,
                          const int64_t* offsets, const int32_t* targets, const int32_t* weights_fx,
                          const int32_t* delays, int64_t* scratch, int32_t phase, void* stream);

/* ---- runtime specialisation ----------------------------------------------- */

/* The float (HHB_F32) forward/backward kernels are generated per parameter
 * table (constants as immediates, rate kinds and exponents resolved) and
 * compiled with NVRTC for sm_100a on first use; the generic table-driven
 * kernels run when NVRTC is unavailable or HHB_NO_JIT=1.
 * hhb_jit_status: "ok", "not initialised" or the reason the JIT is off.
 * hhb_jit_source: writes the generated CUDA source for `params` into buf
 * (NUL-terminated, truncated to cap) and returns the full size + 1, or -1. */
/* out[i] = x[i] * (scale[0] * c), fp32, scale read on the device: the
 * autograd seed of a reduction loss, e.g. MSE's 2 (V - target) / n times the
 * incoming gradient (learn.py:86-88), in one pass with no host sync. */
int hhb_scale_f32(int64_t n, const float* x, const float* scale, double c, float* out, void* stream);
const char* hhb_jit_status(void);
/* compile-only NVRTC build (no device needed) of one generated module for
 * sm_100a: kind 0 forward + backward, 1 the persistent network kernel, 2 the
 * network kernel for 4 replicas, 16 + f the backward module specialised on
 * optional-stream flags f, -1 - f the forward module on output flags f.  Returns the cubin size (copied into buf when
 * cap suffices), -1 on error (hhb_last_error has the NVRTC log). */
int64_t hhb_jit_cubin(const hhb_params_t* params, int32_t kind, void* buf, int64_t cap);
int64_t hhb_jit_source(const hhb_params_t* params, char* buf, int64_t cap);

/* ---- measurement ---------------------------------------------------------- */

/* Pipe-throughput probe used by bench.py to measure the roofline denominator
 * of the SFU-bound kernels on the box itself: which = 0 runs independent
 * MUFU ex2 chains, which = 1 FFMA chains, which = 2 MUFU rcp chains, on
 * 148 * 8 blocks x 256 threads, `iters` iterations of 8 ops per thread.
 * Returns the number of operations issued in *ops (host). */
int hhb_pipe_probe(int32_t which, int64_t iters, float* sink, int64_t* ops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HHB200_H */
