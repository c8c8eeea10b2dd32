// Bond-propagation non-local gates (apply_2q_bondprop, gate_apply.cpp:181-255)
// on the GPU. The 4x4 gate is split by SVD across the control|target cut
// (prop <= 4 operator-Schmidt terms); the left factor opens a carrier bond at
// q0, every intermediate site absorbs the carrier with one truncating SVD
// (the same batched Jacobi kernels as the local path), and the right factor
// closes it at q1. Exactly q1 - q0 truncating SVDs, as in the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

struct Small4 {
  cplx m[16];  // row-major 4x4 (left: (p0',p0) x kappa ; right: kappa x (p1',p1))
};

// X/X0 of the Jacobi operand from a row-major device matrix A (rows x cols).
// Orientation 0: vector v = column v of A; 1: vector v = conj(row v of A).
__global__ void load_matrix_kernel(const cplx* __restrict__ A, long long lda, int rows, int cols, int xtrans,
                                   cplx* __restrict__ X, long long ldx, int xsplit, int f, cplx* __restrict__ X0,
                                   long long ldx0, double* frob2) {
  double fr = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)rows * cols;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    const cplx v = A[(long long)r * lda + c];
    const cplx vc = make_double2(v.x, -v.y);
    const long long xv = xtrans == 0 ? c : r, xe = xtrans == 0 ? r : c;
    const cplx xval = xtrans == 0 ? v : vc;
    (void)xsplit;  // every workspace operand is split planes (common.cuh)
    xs_set(X + xv * ldx, ldx, xe, xval);
    if (f == 0) xs_set(X0 + (long long)c * ldx0, ldx0, r, v);
    else xs_set(X0 + (long long)r * ldx0, ldx0, c, vc);
    fr += cabs2(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fr += __shfl_xor_sync(0xffffffffu, fr, o);
  if (threadIdx.x % 32 == 0) atomicAdd(frob2, fr);
}

void launch_load_matrix(const cplx* A, long long lda, int rows, int cols, int xtrans, cplx* X, long long ldx,
                        int xsplit, int f, cplx* X0, long long ldx0, double* frob2, cudaStream_t st) {
  long long blocks = ((long long)rows * cols + 255) / 256;
  blocks = std::max(1LL, std::min(blocks, 2048LL));
  load_matrix_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, lda, rows, cols, xtrans, X, ldx, xsplit, f, X0, ldx0,
                                                       frob2);
}

// Open (gate_apply.cpp:210-215):
// out[(l,p0')][(kappa,b)] = sum_p site[(l*2+p)*chi + b] * left[(p0',p)][kappa]
__global__ void bp_open_kernel(const cplx* __restrict__ site, int chi, int dl, int b0, Small4 left, int prop,
                               cplx* __restrict__ out) {
  const int N = prop * b0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)dl * 2 * N;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / N), col = (int)(i % N);
    const int l = row / 2, po = row % 2, kk = col / b0, b = col % b0;
    cplx acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int pi = 0; pi < 2; ++pi) cfma(acc, site[(long long)(l * 2 + pi) * chi + b], left.m[(po * 2 + pi) * 4 + kk]);
    out[i] = acc;
  }
}

// Close (gate_apply.cpp:248-251):
// site[(a*2+p1')*chi + r] = sum_{kappa,p1} target[(a*prop+kappa)][p1*dr + r] * right[kappa][(p1',p1)]
__global__ void bp_close_kernel(const cplx* __restrict__ target, int k, int prop, int dr, Small4 right,
                                cplx* __restrict__ site, int chi) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * 2 * dr;
       i += (long long)gridDim.x * blockDim.x) {
    const int a = (int)(i / (2 * dr)), e = (int)(i % (2 * dr));
    const int po = e / dr, r = e % dr;
    cplx acc = make_double2(0.0, 0.0);
    for (int kk = 0; kk < prop; ++kk)
#pragma unroll
      for (int pi = 0; pi < 2; ++pi)
        cfma(acc, target[(long long)(a * prop + kk) * 2 * dr + pi * dr + r], right.m[kk * 4 + po * 2 + pi]);
    site[(long long)(a * 2 + po) * chi + r] = acc;
  }
}

namespace {

unsigned grid_for(long long n) { return (unsigned)std::max(1LL, std::min((n + 255) / 256, 4096LL)); }

// One truncating SVD of a row-major device matrix A (M x N): U -> u_out (ldu),
// S V^dag -> v_out (k x N, ld N). Returns the GateOut.
GateOut svd_into(State& s, const cplx* A, int M, int N, const mpsim_policy& pol, cplx* u_out, long long ldu,
                 cplx* v_out) {
  GateDesc d{};
  d.dl = std::max(1, M / 2);
  d.dm = 1;
  d.dr = std::max(1, N / 2);
  d.trans = M >= N ? 0 : 1;
  d.m = std::max(M, N);
  d.n = std::min(M, N);
  d.n_pad = ((d.n + kP - 1) / kP) * kP;
  d.m_pad = ((d.m + kE - 1) / kE) * kE;
  d.nb = d.n_pad / kW;
  d.max_bond = pol.max_bond;
  d.cutoff = pol.cutoff;
  desc_layout(d, 0, use_qr_precondition(d.n));
  d.u_out = u_out;
  d.ldu = ldu;
  d.v_out = v_out;
  d.ldv = N;
  d.vsplit = N;
  d.vsplit_ld = 0;
  std::vector<GateOut> outs;
  run_two_chunk(s, {d}, outs, A, N);
  if (outs[0].status != 0)
    fail(MPSIM_ENUMERIC, "singular value decomposition did not converge for (" + std::to_string(M) + "," +
                             std::to_string(N) + ") matrix");
  return outs[0];
}

void gemm(State& s, int M, int N, int K, const cplx* A, long long lda, const cplx* B, long long ldb, cplx* C,
          long long ldc) {
  GemmArgs g{M, N, K, A, lda, 0, B, ldb, 0, C, ldc, make_double2(1.0, 0.0), 0};
  launch_cgemm(g, s.st);
  ++s.launches;
}

}  // namespace

void apply_bondprop(State& s, const cplx* u, int q0, int q1, const mpsim_policy& pol, double* w_out,
                    long long* k_out, int* svd_out) {
  DeviceGuard g(s.device);
  // Gate split (gate_apply.cpp:198-206): split[(p0',p0),(p1',p1)] = u[2p0'+p1'][2p0+p1], unbounded SVD.
  double split[32];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int c = 0; c < 2; ++c)
        for (int e = 0; e < 2; ++e) {
          const cplx v = u[(a * 2 + b) * 4 + c * 2 + e];
          const int idx = (a * 2 + c) * 4 + b * 2 + e;
          split[2 * idx] = v.x;
          split[2 * idx + 1] = v.y;
        }
  int64_t prop64 = 0;
  double sv[4], uu[32], vd[32], wg = 0.0;
  if (mpsim_gpu_svd(4, 4, split, MPSIM_UNBOUNDED, 0.0, s.device, &prop64, sv, uu, vd, &wg) != MPSIM_OK)
    fail(MPSIM_ENUMERIC, last_error_slot());
  const int prop = (int)prop64;
  Small4 left{}, right{};
  for (int r = 0; r < 4; ++r)
    for (int kk = 0; kk < prop; ++kk) left.m[r * 4 + kk] = make_double2(uu[2 * (r * prop + kk)], uu[2 * (r * prop + kk) + 1]);
  for (int kk = 0; kk < prop; ++kk)
    for (int c = 0; c < 4; ++c)
      right.m[kk * 4 + c] = make_double2(sv[kk] * vd[2 * (kk * 4 + c)], sv[kk] * vd[2 * (kk * 4 + c) + 1]);

  double w = 0.0;
  long long newb = 1;
  int svd = 0;
  DeviceBuf mat, car, car2, tgt;
  // ---- open at q0 (gate_apply.cpp:208-225)
  const int dl0 = (int)s.sdl[q0], b0 = (int)s.sdr[q0];
  {
    const long long need = std::min<long long>(std::min<long long>(2LL * dl0, (long long)prop * b0), pol.max_bond);
    if (need > s.chi) {
      int c = 1;
      while (c < need) c <<= 1;
      s.grow(c);
    }
  }
  mat.ensure(sizeof(cplx) * (size_t)2 * dl0 * prop * b0);
  bp_open_kernel<<<grid_for(2LL * dl0 * prop * b0), 256, 0, s.st>>>(s.sites + (long long)q0 * s.stride, s.chi, dl0, b0,
                                                                      left, prop, (cplx*)mat.p);
  ++s.launches;
  car.ensure(sizeof(cplx) * (size_t)std::min(2 * dl0, prop * b0) * prop * b0);
  GateOut o = svd_into(s, (const cplx*)mat.p, 2 * dl0, prop * b0, pol, s.sites + (long long)q0 * s.stride, s.chi,
                       (cplx*)car.p);
  int k = o.k;
  s.sdr[q0] = k;
  s.bonds[(size_t)q0 + 1] = k;
  w += o.w;
  newb = std::max<long long>(newb, k);
  ++svd;
  int bprev = b0;
  // ---- push through q0+1 .. q1-1 (gate_apply.cpp:227-246)
  for (int site = q0 + 1; site < q1; ++site) {
    const int br = (int)s.sdr[site];
    const int M = 2 * k, N = prop * br;
    const long long need = std::min<long long>(std::min<long long>(M, N), pol.max_bond);
    if (need > s.chi) {
      int c = 1;
      while (c < need) c <<= 1;
      s.grow(c);
    }
    const cplx* T = s.sites + (long long)site * s.stride;
    mat.ensure(sizeof(cplx) * (size_t)M * N);
    cplx* A = (cplx*)mat.p;
    // arranged[(a,p)][(kappa,r)] = sum_b carrier[a][(kappa,b)] T[(b,p),r]
    for (int kk = 0; kk < prop; ++kk)
      for (int p = 0; p < 2; ++p)
        gemm(s, k, br, bprev, (const cplx*)car.p + (long long)kk * bprev, (long long)prop * bprev,
             T + (long long)p * s.chi, 2LL * s.chi, A + (long long)p * N + (long long)kk * br, 2LL * N);
    car2.ensure(sizeof(cplx) * (size_t)std::min(M, N) * N);
    o = svd_into(s, A, M, N, pol, s.sites + (long long)site * s.stride, s.chi, (cplx*)car2.p);
    const int k2 = o.k;
    s.sdl[site] = k;
    s.sdr[site] = k2;
    s.bonds[(size_t)site + 1] = k2;
    w += o.w;
    newb = std::max<long long>(newb, k2);
    ++svd;
    std::swap(car, car2);
    k = k2;
    bprev = br;
  }
  // ---- close at q1 (gate_apply.cpp:248-253)
  const int dr1 = (int)s.sdr[q1];
  if (k > s.chi) {
    int c = 1;
    while (c < k) c <<= 1;
    s.grow(c);
  }
  tgt.ensure(sizeof(cplx) * (size_t)k * prop * 2 * dr1);
  cplx* S1 = s.sites + (long long)q1 * s.stride;
  for (int p = 0; p < 2; ++p)
    gemm(s, k * prop, dr1, bprev, (const cplx*)car.p, bprev, S1 + (long long)p * s.chi, 2LL * s.chi,
         (cplx*)tgt.p + (long long)p * dr1, 2LL * dr1);
  bp_close_kernel<<<grid_for(2LL * k * dr1), 256, 0, s.st>>>((const cplx*)tgt.p, k, prop, dr1, right, S1, s.chi);
  ++s.launches;
  cudaError_t e = cudaStreamSynchronize(s.st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) fail(MPSIM_ECUDA, std::string("bond propagation: ") + cudaGetErrorString(e));
  s.sdl[q1] = k;
  // update_center(q0, q1) (gate_apply.cpp:252)
  if (s.center >= 0) s.center = (s.center >= q0 && s.center <= q1) ? q1 : -1;
  *w_out = w;
  *k_out = newb;
  *svd_out = svd;
  for (DeviceBuf* b : {&mat, &car, &car2, &tgt}) b->release();
}

}  // namespace mpsim_gpu
