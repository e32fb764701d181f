// morph_f64.cu -- float64 flavour of the multicompartment kernel (morph.cuh),
// built with -fmad=false like hh_f64.cu so its sums follow NumPy's rounding;
// also the C ABI of the morphology entry points.
#include "morph.cuh"

namespace hhb {
namespace morph {
int morph_f32(int n_tables, const hhb_params_t* tables, int n_comp, const int32_t* table_of, int n_edges,
              const int32_t* edge_a, const int32_t* edge_b, const double* g_axial, const Args<float>& a,
              cudaStream_t st);
}  // namespace morph
}  // namespace hhb

using namespace hhb;

extern "C" int hhb_morph_forward(int32_t dtype, int32_t n_tables, const hhb_params_t* tables, int32_t n_comp,
                                 const int32_t* table_of, int32_t n_edges, const int32_t* edge_a,
                                 const int32_t* edge_b, const double* g_axial, int64_t batch, int64_t n_steps,
                                 const void* i_ext, const void* v_in, const void* g_in, void* v_fin, void* g_fin,
                                 void* v_out, uint8_t* spk_out, void* ax_out, int64_t step_base,
                                 int64_t* first_bad, void* stream) {
  if (!tables || !table_of || (n_edges > 0 && (!edge_a || !edge_b || !g_axial)))
    return fail(HHB_EINVAL, "morphology: missing graph arrays");
  for (int k = 0; k < n_tables; ++k) {
    const int rc = hhb_check_params(&tables[k]);
    if (rc) return rc;
  }
  if (batch < 0 || n_steps < 0) return fail(HHB_EINVAL, "batch and n_steps must be >= 0");
  if (batch == 0) return HHB_OK;
  if (!v_in || !g_in || !first_bad) return fail(HHB_EINVAL, "morphology: v_in, g_in, first_bad required");
  if (n_steps > 0 && (!i_ext || !v_fin || !g_fin)) return fail(HHB_EINVAL, "morphology: i_ext, v_fin, g_fin required");
  if (n_steps == 0 && !ax_out) return fail(HHB_EINVAL, "morphology: n_steps == 0 computes ax_out, which is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HHB_F32) {
    morph::Args<float> a{batch, n_steps, (const float*)i_ext, (const float*)v_in, (const float*)g_in,
                         (float*)v_fin, (float*)g_fin, (float*)v_out, spk_out, (float*)ax_out, step_base,
                         reinterpret_cast<long long*>(first_bad)};
    return morph::morph_f32(n_tables, tables, n_comp, table_of, n_edges, edge_a, edge_b, g_axial, a, st);
  }
  if (dtype != HHB_F64) return fail(HHB_EINVAL, "dtype");
  morph::Args<double> a{batch, n_steps, (const double*)i_ext, (const double*)v_in, (const double*)g_in,
                        (double*)v_fin, (double*)g_fin, (double*)v_out, spk_out, (double*)ax_out, step_base,
                        reinterpret_cast<long long*>(first_bad)};
  return morph::launch<double>(n_tables, tables, n_comp, table_of, n_edges, edge_a, edge_b, g_axial, a, st);
}
