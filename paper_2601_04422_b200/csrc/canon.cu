// Orthogonality-centre moves on the GPU: the QR sweeps of move_center
// (mps.cpp:57-95, :171-187), built on the blocked Householder QR of qr.cu.
#include <algorithm>
#include <cmath>
#include <string>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

void launch_qr_panel(cplx* A, long long lda, int m, int c0, int jb, cplx* P, cplx* V, cplx* T, cplx* tau,
                     cudaStream_t st);
void launch_set_identity(cplx* Y, long long ld, int m, int k, cudaStream_t st);
void launch_copy_matrix(const cplx* src, long long ld_s, cplx* dst, long long ld_d, int rows, int cols, int op,
                        cudaStream_t st);
void launch_site_adjoint(const cplx* site, int chi, int dl, int dr, cplx* A, long long lda, cudaStream_t st);
void launch_site_from_adjoint(const cplx* Q, long long ldq, int k, int dr, cplx* site, int chi, cudaStream_t st);
void launch_sum_abs2(const cplx* A, long long lda, int rows, int cols, double* out, cudaStream_t st);
void launch_cgemm(const GemmArgs&, cudaStream_t);

namespace {

constexpr int kQB = 32;

struct QrWork {
  DeviceBuf W, P, Vall, Tall, tau, W1, W2, Q, R, tmp, nrm;
};

void gemm(State& s, int M, int N, int K, const cplx* A, long long lda, int opA, const cplx* B, long long ldb,
          int opB, cplx* C, long long ldc, double alpha, int acc) {
  GemmArgs g{M, N, K, A, lda, opA, B, ldb, opB, C, ldc, make_double2(alpha, 0.0), acc};
  launch_cgemm(g, s.st);
  ++s.launches;
}

// Householder QR of W (m x n, row-major, ld n), destroyed. Q (m x k, ldq) and
// R (k x n, ldr), k = min(m, n) (thin_qr: Q = householderQ * I(m, k)).
int thin_qr(State& s, QrWork& w, cplx* W, int m, int n, cplx* Q, long long ldq, cplx* R, long long ldr) {
  const int k = std::min(m, n);
  const int np = (k + kQB - 1) / kQB;
  w.P.ensure(sizeof(cplx) * (size_t)m * kQB);
  w.Vall.ensure(sizeof(cplx) * (size_t)np * m * kQB);
  w.Tall.ensure(sizeof(cplx) * (size_t)np * kQB * kQB);
  w.tau.ensure(sizeof(cplx) * (size_t)std::max(k, 1));
  w.W1.ensure(sizeof(cplx) * (size_t)kQB * std::max(n, k));
  w.W2.ensure(sizeof(cplx) * (size_t)kQB * std::max(n, k));
  cplx* Vall = (cplx*)w.Vall.p;
  cplx* Tall = (cplx*)w.Tall.p;
  cplx* W1 = (cplx*)w.W1.p;
  cplx* W2 = (cplx*)w.W2.p;
  for (int p = 0; p < np; ++p) {
    const int c0 = p * kQB, jb = std::min(kQB, k - c0), L = m - c0;
    cplx* V = Vall + (long long)p * m * kQB;
    cplx* T = Tall + (long long)p * kQB * kQB;
    launch_qr_panel(W, n, m, c0, jb, (cplx*)w.P.p, V, T, (cplx*)w.tau.p, s.st);
    ++s.launches;
    const int n2 = n - c0 - jb;
    if (n2 > 0) {  // A2 <- (I - V T^H V^H) A2
      cplx* A2 = W + (long long)c0 * n + c0 + jb;
      gemm(s, kQB, n2, L, V, kQB, 1, A2, n, 0, W1, n2, 1.0, 0);
      gemm(s, kQB, n2, kQB, T, kQB, 1, W1, n2, 0, W2, n2, 1.0, 0);
      gemm(s, L, n2, kQB, V, kQB, 0, W2, n2, 0, A2, n, -1.0, 1);
    }
  }
  if (R) {
    launch_copy_matrix(W, n, R, ldr, k, n, 2, s.st);
    ++s.launches;
  }
  // Q = H_1 ... H_np [I; 0]
  launch_set_identity(Q, ldq, m, k, s.st);
  ++s.launches;
  for (int p = np - 1; p >= 0; --p) {
    const int c0 = p * kQB, L = m - c0;
    cplx* V = Vall + (long long)p * m * kQB;
    cplx* T = Tall + (long long)p * kQB * kQB;
    cplx* Y2 = Q + (long long)c0 * ldq;
    gemm(s, kQB, k, L, V, kQB, 1, Y2, ldq, 0, W1, k, 1.0, 0);
    gemm(s, kQB, k, kQB, T, kQB, 0, W1, k, 0, W2, k, 1.0, 0);
    gemm(s, L, k, kQB, V, kQB, 0, W2, k, 0, Y2, ldq, -1.0, 1);
  }
  return k;
}

#define CKC(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// sweep_left_of (mps.cpp:69-80): site i = Q (Dl,2,k), site i+1 = R * site i+1.
void left_step(State& s, QrWork& w, int i) {
  const int dl = (int)s.sdl[i], dr = (int)s.sdr[i];
  const int m = 2 * dl, n = dr;
  cplx* site = s.sites + (long long)i * s.stride;
  cplx* next = s.sites + (long long)(i + 1) * s.stride;
  w.W.ensure(sizeof(cplx) * (size_t)m * n);
  w.R.ensure(sizeof(cplx) * (size_t)std::min(m, n) * n);
  w.tmp.ensure(sizeof(cplx) * (size_t)s.stride);
  cplx* W = (cplx*)w.W.p;
  launch_copy_matrix(site, s.chi, W, n, m, n, 0, s.st);
  ++s.launches;
  const int k = thin_qr(s, w, W, m, n, site, s.chi, (cplx*)w.R.p, n);
  const int dr2 = (int)s.sdr[i + 1];
  cplx* tmp = (cplx*)w.tmp.p;
  for (int p = 0; p < 2; ++p)
    gemm(s, k, dr2, n, (cplx*)w.R.p, n, 0, next + (long long)p * s.chi, 2LL * s.chi, 0, tmp + (long long)p * s.chi,
         2LL * s.chi, 1.0, 0);
  CKC(cudaMemcpy2DAsync(next, sizeof(cplx) * s.chi, tmp, sizeof(cplx) * s.chi, sizeof(cplx) * dr2, (size_t)k * 2,
                        cudaMemcpyDeviceToDevice, s.st));
  s.sdr[i] = k;
  s.sdl[i + 1] = k;
  s.bonds[(size_t)i + 1] = k;
}

// sweep_right_of (mps.cpp:84-95): QR of site_i^H (2Dr x Dl); site i = Q^H,
// site i-1 = site i-1 * R^H.
void right_step(State& s, QrWork& w, int i) {
  const int dl = (int)s.sdl[i], dr = (int)s.sdr[i];
  const int m = 2 * dr, n = dl, k = std::min(m, n);
  cplx* site = s.sites + (long long)i * s.stride;
  cplx* prev = s.sites + (long long)(i - 1) * s.stride;
  w.W.ensure(sizeof(cplx) * (size_t)m * n);
  w.R.ensure(sizeof(cplx) * (size_t)k * n);
  w.Q.ensure(sizeof(cplx) * (size_t)m * k);
  w.tmp.ensure(sizeof(cplx) * (size_t)s.stride);
  cplx* W = (cplx*)w.W.p;
  launch_site_adjoint(site, s.chi, dl, dr, W, n, s.st);
  ++s.launches;
  thin_qr(s, w, W, m, n, (cplx*)w.Q.p, k, (cplx*)w.R.p, n);
  launch_site_from_adjoint((cplx*)w.Q.p, k, k, dr, site, s.chi, s.st);
  ++s.launches;
  const int dl2 = (int)s.sdl[i - 1];
  cplx* tmp = (cplx*)w.tmp.p;
  gemm(s, 2 * dl2, k, n, prev, s.chi, 0, (cplx*)w.R.p, n, 1, tmp, s.chi, 1.0, 0);
  CKC(cudaMemcpy2DAsync(prev, sizeof(cplx) * s.chi, tmp, sizeof(cplx) * s.chi, sizeof(cplx) * k, (size_t)2 * dl2,
                        cudaMemcpyDeviceToDevice, s.st));
  s.sdl[i] = k;
  s.sdr[i - 1] = k;
  s.bonds[(size_t)i] = k;
}

thread_local std::string g_err_canon;

}  // namespace

// Pieces of move_center for site-sharded chains: left steps
// i = i0 .. i1 - 1 (site i -> Q, R absorbed into i + 1) or right steps
// i = i1 .. i0 (site i -> Q^H, R^H absorbed into i - 1, i0 >= 1) over the
// local slots, the boundary step run by the left shard on its ghost slot.
void sweep_left_impl(State& s, int i0, int i1) {
  if (i0 < 0 || i1 > s.n - 1 || i0 > i1) fail(MPSIM_EINVAL, "left sweep range out of bounds");
  DeviceGuard g(s.device);
  QrWork w;
  for (int i = i0; i < i1; ++i) left_step(s, w, i);
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
  for (DeviceBuf* b : {&w.W, &w.P, &w.Vall, &w.Tall, &w.tau, &w.W1, &w.W2, &w.Q, &w.R, &w.tmp, &w.nrm}) b->release();
  s.center = -1;
}

void sweep_right_impl(State& s, int i0, int i1) {
  if (i0 < 1 || i1 > s.n - 1 || i0 > i1 + 1) fail(MPSIM_EINVAL, "right sweep range out of bounds");
  DeviceGuard g(s.device);
  QrWork w;
  for (int i = i1; i >= i0; --i) right_step(s, w, i);
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
  for (DeviceBuf* b : {&w.W, &w.P, &w.Vall, &w.Tall, &w.tau, &w.W1, &w.W2, &w.Q, &w.R, &w.tmp, &w.nrm}) b->release();
  s.center = -1;
}

double site_norm2_impl(State& s, int i) {
  if (i < 0 || i >= s.n) fail(MPSIM_EINVAL, "site index out of range");
  DeviceGuard g(s.device);
  DeviceBuf nrm;
  nrm.ensure(sizeof(double));
  launch_sum_abs2(s.sites + (long long)i * s.stride, s.chi, (int)(2 * s.sdl[i]), (int)s.sdr[i], (double*)nrm.p, s.st);
  ++s.launches;
  double n2 = 0.0;
  CKC(cudaMemcpyAsync(&n2, nrm.p, sizeof(double), cudaMemcpyDeviceToHost, s.st));
  CKC(cudaStreamSynchronize(s.st));
  nrm.release();
  return n2;
}

void move_center_impl(State& s, int c) {
  if (c < 0 || c >= s.n) fail(MPSIM_EINVAL, "center out of range");
  DeviceGuard g(s.device);
  QrWork w;
  for (int i = 0; i < c; ++i) left_step(s, w, i);
  for (int i = s.n - 1; i > c; --i) right_step(s, w, i);
  w.nrm.ensure(sizeof(double));
  launch_sum_abs2(s.sites + (long long)c * s.stride, s.chi, (int)(2 * s.sdl[c]), (int)s.sdr[c], (double*)w.nrm.p, s.st);
  ++s.launches;
  double n2 = 0.0;
  CKC(cudaMemcpyAsync(&n2, w.nrm.p, sizeof(double), cudaMemcpyDeviceToHost, s.st));
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
  for (DeviceBuf* b : {&w.W, &w.P, &w.Vall, &w.Tall, &w.tau, &w.W1, &w.W2, &w.Q, &w.R, &w.tmp, &w.nrm}) b->release();
  if (std::sqrt(n2) < 1e-14) fail(MPSIM_ENUMERIC, "cannot canonicalize a zero-norm state");
  s.center = c;
}

}  // namespace mpsim_gpu
