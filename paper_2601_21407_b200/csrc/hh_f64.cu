// hh_f64.cu -- double flavour (the parity build).  Compiled with -fmad=false
// so every product and sum rounds separately, as NumPy does in the reference.
#include "hh_host.cuh"

namespace hhb {
HHB_DEFINE_FLAVOUR(double, 2)
}  // namespace hhb
