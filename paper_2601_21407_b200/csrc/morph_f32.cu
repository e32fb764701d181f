// morph_f32.cu -- float flavour of the multicompartment kernel (morph.cuh)
#include "morph.cuh"

namespace hhb {
namespace morph {
int morph_f32(int n_tables, const hhb_params_t* tables, int n_comp, const int32_t* table_of, int n_edges,
              const int32_t* edge_a, const int32_t* edge_b, const double* g_axial, const Args<float>& a,
              cudaStream_t st) {
  return launch<float>(n_tables, tables, n_comp, table_of, n_edges, edge_a, edge_b, g_axial, a, st);
}
}  // namespace morph
}  // namespace hhb
