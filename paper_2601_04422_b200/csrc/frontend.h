// Host front end shared between frontend.cpp and statevec.cu.
#pragma once

#include <complex>
#include <vector>

namespace mpsim_gpu {

// One primitive op for the dense statevector backend: q1 = -1 for a
// one-qubit op; two-qubit ops have q0 < q1 and u in the (q0, q1) basis.
struct SvOp {
  int q0 = 0, q1 = -1;
  std::complex<double> u[16];
};

// sv_run (statevector.cpp:88-99) on the device; out receives the 2^n
// amplitudes. launches (nullable) = kernels launched.
void sv_run_device(int n, const std::vector<SvOp>& ops, int device, std::vector<std::complex<double>>& out,
                   long long* launches);

}  // namespace mpsim_gpu
