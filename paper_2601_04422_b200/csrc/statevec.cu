// Dense statevector backend of run_circuit (Backend::Statevector,
// runner.cpp:236-250 over sv_run, statevector.cpp:88-99): the raw primitive
// ops applied in order to a 2^n amplitude vector in HBM, qubit 0 = most
// significant bit (statevector.cpp:40-41, :58-59). HBM-bound: every gate
// streams the vector once (16 B read + 16 B write per amplitude).
#include <complex>
#include <vector>

#include "common.cuh"
#include "engine.h"
#include "frontend.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

struct SvU {
  cplx u[16];
};

// One thread per amplitude pair (i, i + stride): StateVector::apply_1q,
// statevector.cpp:29-46.
__global__ void __launch_bounds__(256) sv_1q_kernel(cplx* __restrict__ a, long long half, long long stride, SvU u) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < half;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = (t / stride) * 2 * stride + t % stride;
    const cplx a0 = a[i], a1 = a[i + stride];
    cplx n0 = cmul(u.u[0], a0), n1 = cmul(u.u[2], a0);
    cfma(n0, u.u[1], a1);
    cfma(n1, u.u[3], a1);
    a[i] = n0;
    a[i + stride] = n1;
  }
}

// One thread per 4-amplitude group with both gate bits clear:
// StateVector::apply_2q, statevector.cpp:48-75 (s0 = stride of the low-index
// qubit = row bit 1 of the 4x4 matrix, s1 < s0).
__global__ void __launch_bounds__(256) sv_2q_kernel(cplx* __restrict__ a, long long quarter, long long s0,
                                                    long long s1, SvU u) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < quarter;
       t += (long long)gridDim.x * blockDim.x) {
    // insert a zero bit at s1, then at s0
    long long i = (t / s1) * 2 * s1 + t % s1;
    i = (i / s0) * 2 * s0 + i % s0;
    const cplx x[4] = {a[i], a[i + s1], a[i + s0], a[i + s0 + s1]};
    cplx y[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      cplx acc = cmul(u.u[4 * r], x[0]);
#pragma unroll
      for (int c = 1; c < 4; ++c) cfma(acc, u.u[4 * r + c], x[c]);
      y[r] = acc;
    }
    a[i] = y[0];
    a[i + s1] = y[1];
    a[i + s0] = y[2];
    a[i + s0 + s1] = y[3];
  }
}

__global__ void sv_init_kernel(cplx* a, long long dim) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < dim;
       t += (long long)gridDim.x * blockDim.x)
    a[t] = make_double2(t == 0 ? 1.0 : 0.0, 0.0);
}

namespace {
#define SVCK(x)                                                                             \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

unsigned grid_for(long long work) {
  long long b = (work + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;  // grid-stride beyond 16 CTAs per SM
  return (unsigned)(b < 1 ? 1 : b);
}
}  // namespace

void sv_run_device(int n, const std::vector<SvOp>& ops, int device, std::vector<std::complex<double>>& out,
                   long long* launches) {
  DeviceGuard g(device);
  const long long dim = 1LL << n;
  cplx* a = nullptr;
  SVCK(cudaMalloc(&a, (size_t)dim * sizeof(cplx)));
  cudaStream_t st = nullptr;
  long long nl = 0;
  try {
    SVCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    sv_init_kernel<<<grid_for(dim), 256, 0, st>>>(a, dim);
    ++nl;
    for (const SvOp& op : ops) {
      SvU u;
      const int k = op.q1 >= 0 ? 16 : 4;
      for (int e = 0; e < k; ++e) u.u[e] = make_double2(op.u[e].real(), op.u[e].imag());
      if (op.q1 < 0) {
        sv_1q_kernel<<<grid_for(dim / 2), 256, 0, st>>>(a, dim / 2, 1LL << (n - 1 - op.q0), u);
      } else {
        sv_2q_kernel<<<grid_for(dim / 4), 256, 0, st>>>(a, dim / 4, 1LL << (n - 1 - op.q0),
                                                        1LL << (n - 1 - op.q1), u);
      }
      ++nl;
    }
    SVCK(cudaGetLastError());
    out.resize((size_t)dim);
    SVCK(cudaMemcpyAsync(out.data(), a, (size_t)dim * sizeof(cplx), cudaMemcpyDeviceToHost, st));
    SVCK(cudaStreamSynchronize(st));
  } catch (...) {
    if (st) cudaStreamDestroy(st);
    cudaFree(a);
    throw;
  }
  cudaStreamDestroy(st);
  cudaFree(a);
  if (launches) *launches = nl;
}

}  // namespace mpsim_gpu
