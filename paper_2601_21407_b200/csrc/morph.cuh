// morph.cuh -- multicompartment neurons (reference hhengine/morphology.py,
// SURVEY §8 f3): compartments on a graph, each with its own channel table,
// coupled by the axial neighbour sum of the previous step's potentials
// (axial_current, morphology.py:115-124), then one HH step per compartment
// with i_ext + axial (morph_step, morphology.py:127-141), over T steps
// (simulate_morphology, :144-166).
//
// Time-fused, B200 layout: one block = 32 batch elements x C compartments,
// thread (lane, c); a warp is one compartment for 32 batch elements, so the
// table dispatch is warp-uniform and I/O is coalesced along the batch.  The
// potentials of the tile live in shared memory (double-buffered, one
// __syncthreads per step); each compartment walks the edge list in the
// reference's order (out[a] += flow, out[b] -= flow), so the float64 build
// reproduces NumPy's sums exactly.
#pragma once

#include "hh_host.cuh"

namespace hhb {
namespace morph {

constexpr int kMaxComp = 32;
constexpr int kMaxEdges = 64;
constexpr int kMaxTables = 4;

template <typename T>
struct Graph {
  int n_comp, n_edges;
  int table_of[kMaxComp];
  int ng_of[kMaxComp];
  int edge_a[kMaxEdges], edge_b[kMaxEdges];
  T g_axial[kMaxEdges];
  DevTable<T> tb[kMaxTables];
};

template <typename T>
struct Args {
  int64_t batch, steps;
  const T* i_ext;      // [steps][n_comp][batch]
  const T* v_in;       // [n_comp][batch]
  const T* g_in;       // [n_comp][kMaxGates][batch] (a compartment uses its first ng rows)
  T* v_fin;
  T* g_fin;
  T* v_out;            // [steps][n_comp][batch] or NULL
  uint8_t* spk_out;    // [steps][n_comp][batch] or NULL
  T* ax_out;           // steps == 0: the axial current of the input state, [n_comp][batch]
  int64_t step_base;
  long long* first_bad;
};

template <typename T, int NG>
__device__ __forceinline__ T step_ng(const DevTable<T>& tb, T v, T (&p)[kMaxGates], T cur) {
  return step_forward<T, NG>(tb, v, reinterpret_cast<T(&)[NG > 0 ? NG : 1]>(p), cur);
}

template <typename T>
__device__ __forceinline__ T step_any(int ng, const DevTable<T>& tb, T v, T (&p)[kMaxGates], T cur) {
  switch (ng) {
    case 0: return step_ng<T, 0>(tb, v, p, cur);
    case 1: return step_ng<T, 1>(tb, v, p, cur);
    case 2: return step_ng<T, 2>(tb, v, p, cur);
    case 3: return step_ng<T, 3>(tb, v, p, cur);
    case 4: return step_ng<T, 4>(tb, v, p, cur);
    case 5: return step_ng<T, 5>(tb, v, p, cur);
    case 6: return step_ng<T, 6>(tb, v, p, cur);
    case 7: return step_ng<T, 7>(tb, v, p, cur);
    default: return step_ng<T, 8>(tb, v, p, cur);
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) k_morph(const __grid_constant__ Graph<T> G, const Args<T> a) {
  __shared__ T vs[2][kMaxComp][32];
  const int lane = threadIdx.x, c = threadIdx.y;
  const int64_t b = int64_t(blockIdx.x) * 32 + lane;
  const bool on = b < a.batch;
  const int64_t bb = on ? b : 0;
  const int ng = G.ng_of[c];
  const DevTable<T>& tb = G.tb[G.table_of[c]];
  const int64_t cb = int64_t(c) * a.batch + bb;
  T v = a.v_in[cb];
  T p[kMaxGates];
#pragma unroll
  for (int g = 0; g < kMaxGates; ++g) p[g] = g < ng ? a.g_in[(int64_t(c) * kMaxGates + g) * a.batch + bb] : T(0);
  long long bad = LLONG_MAX;
  const int64_t srow = int64_t(G.n_comp) * a.batch;
  int buf = 0;
  const int64_t nsteps = a.steps > 0 ? a.steps : 1;
  for (int64_t t = 0; t < nsteps; ++t) {
    vs[buf][c][lane] = v;
    __syncthreads();
    // axial_current (morphology.py:115-124): edges in declaration order
    T ax = T(0);
    for (int e = 0; e < G.n_edges; ++e) {
      const int ea = G.edge_a[e], eb = G.edge_b[e];
      if (ea != c && eb != c) continue;
      const T flow = mul_(G.g_axial[e], sub_(vs[buf][eb][lane], vs[buf][ea][lane]));
      ax = (ea == c) ? add_(ax, flow) : sub_(ax, flow);
    }
    if (a.steps == 0) {          // axial_current only
      if (on) a.ax_out[cb] = ax;
      break;
    }
    const T cur = add_(a.i_ext[t * srow + cb], ax);
    const T vn = step_any<T>(ng, tb, v, p, cur);
    const bool spk = (v < tb.theta) && (vn >= tb.theta);       // spike_detect, dynamics.py:379-381
    if (!finite_(vn) && bad == LLONG_MAX && on) bad = a.step_base + t;
    v = vn;
    if (on) {
      if (a.v_out) a.v_out[t * srow + cb] = v;
      if (a.spk_out) a.spk_out[t * srow + cb] = spk ? 1 : 0;
    }
    buf ^= 1;
  }
  if (on && a.steps > 0) {
    a.v_fin[cb] = v;
    for (int g = 0; g < ng; ++g) a.g_fin[(int64_t(c) * kMaxGates + g) * a.batch + bb] = p[g];
  }
  if (bad != LLONG_MAX) atomicMin(a.first_bad, bad);
}

template <typename T>
int launch(int n_tables, const hhb_params_t* tables, int n_comp, const int32_t* table_of, int n_edges,
           const int32_t* edge_a, const int32_t* edge_b, const double* g_axial, const Args<T>& a,
           cudaStream_t st) {
  if (n_comp < 1 || n_comp > kMaxComp) return fail(HHB_EINVAL, "morphology: 1..32 compartments per neuron");
  if (n_edges < 0 || n_edges > kMaxEdges) return fail(HHB_EINVAL, "morphology: at most 64 edges");
  if (n_tables < 1 || n_tables > kMaxTables) return fail(HHB_EINVAL, "morphology: 1..4 distinct channel tables");
  Graph<T> G{};
  G.n_comp = n_comp;
  G.n_edges = n_edges;
  for (int k = 0; k < n_tables; ++k) G.tb[k] = pack_table<T>(&tables[k]);
  for (int c = 0; c < n_comp; ++c) {
    if (table_of[c] < 0 || table_of[c] >= n_tables) return fail(HHB_EINVAL, "morphology: bad table index");
    G.table_of[c] = table_of[c];
    G.ng_of[c] = tables[table_of[c]].n_gates;
  }
  for (int e = 0; e < n_edges; ++e) {
    if (edge_a[e] < 0 || edge_a[e] >= n_comp || edge_b[e] < 0 || edge_b[e] >= n_comp)
      return fail(HHB_EINVAL, "morphology: edge endpoint out of range");
    G.edge_a[e] = edge_a[e];
    G.edge_b[e] = edge_b[e];
    G.g_axial[e] = T(g_axial[e]);
  }
  const dim3 block{32u, unsigned(n_comp), 1u};
  const dim3 grid{unsigned((a.batch + 31) / 32), 1u, 1u};
  k_morph<T><<<grid, block, 0, st>>>(G, a);
  return cuda_check("k_morph launch");
}

}  // namespace morph
}  // namespace hhb
