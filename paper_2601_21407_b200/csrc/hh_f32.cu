// hh_f32.cu -- float flavour (the throughput build): MUFU ex2/rcp, FMA on.
#include "hh_host.cuh"

namespace hhb {
HHB_DEFINE_FLAVOUR(float, 4)
}  // namespace hhb
