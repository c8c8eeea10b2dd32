// Bond-propagation non-local gates (apply_2q_bondprop, gate_apply.cpp:181-255).
// Placeholder until the carrier-SVD path lands: non-local gates are routed
// through SWAP chains (the default NonlocalMethod) instead.
#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

void apply_bondprop(State&, const cplx*, int, int, const mpsim_policy&, double*, long long*, int*) {
  fail(MPSIM_EINVAL, "bond propagation is not available in this build; use the SWAP method");
}

}  // namespace mpsim_gpu
