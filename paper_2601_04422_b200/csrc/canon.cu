// Orthogonality-centre moves on the GPU: the QR sweeps of move_center
// (mps.cpp:57-95, :171-187), built on the blocked Householder QR of qr.cu.
#include <algorithm>
#include <cmath>
#include <string>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

#define CKC(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define CK_CANON CKC

void launch_qr_panel(cplx* A, long long lda, int m, int c0, int jb, cplx* P, cplx* V, cplx* T, cplx* tau,
                     cudaStream_t st);
void launch_set_identity(cplx* Y, long long ld, int m, int k, cudaStream_t st);
void launch_copy_matrix(const cplx* src, long long ld_s, cplx* dst, long long ld_d, int rows, int cols, int op,
                        cudaStream_t st);
void launch_site_adjoint(const cplx* site, int chi, int dl, int dr, cplx* A, long long lda, cudaStream_t st);
void launch_site_from_adjoint(const cplx* Q, long long ldq, int k, int dr, cplx* site, int chi, cudaStream_t st);
void launch_sum_abs2(const cplx* A, long long lda, int rows, int cols, double* out, cudaStream_t st);
void launch_cgemm(const GemmArgs&, cudaStream_t);
void launch_qr_factor(const GateDesc*, int, int, int, cplx*, cplx*, long long, cplx*, int, int, cudaStream_t);
void launch_qr_apply(const GateDesc*, int, int, int, cplx*, const cplx*, long long, const cplx*, int, const int*,
                     long long, const GateOut*, cudaStream_t);
bool site_qr_supported(int m, int n);
int site_qr(State& s, cplx* site, int dl, int dr, int right, DeviceBuf& Abuf, DeviceBuf& Vbuf, DeviceBuf& Tbuf,
            DeviceBuf& Qbuf, cplx* R, cudaStream_t aux, cudaEvent_t* evs, int set);

// ---- tensor-core QR of one site (the gate path's QR machinery, qr_pre.cu:
// 4-CTA cluster panels with the panel held on chip, DMMA trailing updates and
// DMMA Q formation) for the large sites of a centre move. Operand layout:
// columns of the site matrix as split-plane vectors (common.cuh).

// left (right = 0): A_c[r] = site[r chi + c], r < 2 dl, c < dr (the (2Dl x Dr)
// matricisation); right: A_l[e] = conj(site[(l 2 + p) chi + r]), e = p dr + r
// (the (Dl x 2Dr)^H one). Rows m .. ld are zeroed.
__global__ void site_to_qr_kernel(const cplx* __restrict__ site, int chi, int dl, int dr, int right,
                                  cplx* __restrict__ A, long long ld, int n) {
  const int m = right ? 2 * dr : 2 * dl;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * ld;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ld), r = (int)(i % ld);
    cplx v = make_double2(0.0, 0.0);
    if (r < m) {
      if (!right) {
        v = site[(long long)r * chi + c];
      } else {
        const int p = r / dr, rr = r % dr;
        v = site[(long long)(c * 2 + p) * chi + rr];
        v.y = -v.y;
      }
    }
    xs_set(A + (long long)c * ld, ld, r, v);
  }
}

// R (k x n, row-major) = the upper triangle of the factored operand
__global__ void qr_extract_r_kernel(const cplx* __restrict__ A, long long ld, int k, int n, cplx* __restrict__ R) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * n;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / n), c = (int)(i % n);
    R[i] = j <= c ? xs_get(A + (long long)c * ld, ld, j) : make_double2(0.0, 0.0);
  }
}

// X (n vectors of length m_pad) = I, order = identity, out.k = k: the inputs
// of launch_qr_apply that make it form Q = Q1 [I_k; 0] in the QR area.
__global__ void qr_identity_kernel(cplx* __restrict__ X, long long m_pad, int n, int n_pad, int* __restrict__ order,
                                   GateOut* __restrict__ out, int k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n_pad * m_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / m_pad), r = (int)(i % m_pad);
    xs_set(X + (long long)j * m_pad, m_pad, r, make_double2(j == r && j < n ? 1.0 : 0.0, 0.0));
    if (r == 0) order[j] = j;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    GateOut o;
    o.k = k;
    o.status = 0;
    o.w = 0.0;
    o.scale = 1.0;
    *out = o;
  }
}

// site <- Q (left: rows r < 2 dl, columns j < k) or Q^H (right: site[(j 2 + p)
// chi + r] = conj(Q_j[p dr + r]))
__global__ void q_to_site_kernel(const cplx* __restrict__ Z, long long ld, int k, int dl, int dr, int right,
                                 cplx* __restrict__ site, int chi) {
  const int m = right ? 2 * dr : 2 * dl;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * m;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / m), r = (int)(i % m);
    cplx v = xs_get(Z + (long long)j * ld, ld, r);
    if (!right) {
      site[(long long)r * chi + j] = v;
    } else {
      const int p = r / dr, rr = r % dr;
      v.y = -v.y;
      site[(long long)(j * 2 + p) * chi + rr] = v;
    }
  }
}

namespace {

constexpr int kQB = 32;

struct QrWork {
  DeviceBuf W, P, Vall, Tall, tau, W1, W2, Q, R, tmp, nrm;
  DeviceBuf ws, vbuf, tbuf, desc, order, out;  // cluster-panel path (qr_pre.cu)
  DeviceBuf V2[2], T2[2];                      // site QR (qr_site.cu): alternate reflector sets
  int set = 0;
};

// The site QRs' Q formations run on s.aux: the sweep's last step joins them
// back into s.st (every public entry point ends with this before its sync).
void join_aux(State& s) {
  if (!s.aux) return;
  CK_CANON(cudaEventRecord(s.evq[0], s.aux));
  CK_CANON(cudaStreamWaitEvent(s.st, s.evq[0], 0));
}

unsigned grid_of(long long n) { return (unsigned)std::max(1LL, std::min((n + 255) / 256, 8LL * 148)); }

// Site QRs: up to 1024 rows, the latency-shaped kernels of qr_site.cu
// (register-resident 8-column panels, look-ahead updates on a second
// stream); up to 2048 rows, the gate path's cluster panels + DMMA updates
// (qr_pre.cu); small or wide sites keep the streaming panel of qr.cu.
bool tc_qr(int m, int n) { return n >= 64 && m >= n && m <= 2048; }

int fast_site_qr(State& s, QrWork& w, cplx* site, int dl, int dr, int right) {
  if (!s.aux) {
    CK_CANON(cudaStreamCreateWithFlags(&s.aux, cudaStreamNonBlocking));
    for (cudaEvent_t& e : s.evq) CK_CANON(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr, k = std::min(m, n);
  w.R.ensure(sizeof(cplx) * (size_t)k * n);
  const int set = w.set;
  w.set ^= 1;
  return site_qr(s, site, dl, dr, right, w.W, w.V2[set], w.T2[set], w.Q, (cplx*)w.R.p, s.aux, s.evq, set);
}

// Factor the site's matricisation with the qr_pre.cu machinery: R (k x n,
// row-major) into w.R, Q written back into the site (Q or Q^H per side).
int tc_site_qr(State& s, QrWork& w, cplx* site, int dl, int dr, int right) {
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr, k = std::min(m, n);
  GateDesc d{};
  d.q = 0;
  d.n = n;
  d.n_pad = (n + kP - 1) / kP * kP;
  d.nb = d.n_pad / kW;
  d.qr_m = m;
  d.qr_m_pad = (m + kE - 1) / kE * kE;
  d.m = n;
  d.m_pad = (n + kE - 1) / kE * kE;
  d.pre = 1;
  d.ws_off = 0;                                          // X (form_rh / identity)
  d.qr_off = (long long)d.n_pad * d.m_pad;                 // the QR operand
  const long long elems = d.qr_off + (long long)d.n_pad * d.qr_m_pad;
  const int npan = d.n_pad / kQB;
  w.ws.ensure(sizeof(cplx) * (size_t)elems);
  w.vbuf.ensure(sizeof(cplx) * (size_t)npan * kQB * d.qr_m_pad);
  w.tbuf.ensure(sizeof(cplx) * (size_t)npan * kQB * kQB);
  w.desc.ensure(sizeof(GateDesc));
  w.order.ensure(sizeof(int) * (size_t)d.n_pad);
  w.out.ensure(sizeof(GateOut));
  w.R.ensure(sizeof(cplx) * (size_t)k * n);
  cplx* ws = (cplx*)w.ws.p;
  cudaStream_t st = s.st;
  CK_CANON(cudaMemcpyAsync(w.desc.p, &d, sizeof(GateDesc), cudaMemcpyHostToDevice, st));
  const GateDesc* dd = (const GateDesc*)w.desc.p;
  site_to_qr_kernel<<<grid_of((long long)n * d.qr_m_pad), 256, 0, st>>>(site, s.chi, dl, dr, right, ws + d.qr_off,
                                                                         d.qr_m_pad, n);
  // zero padding vectors n .. n_pad of the operand
  if (d.n_pad > n)
    CK_CANON(cudaMemsetAsync(ws + d.qr_off + (long long)n * d.qr_m_pad, 0,
                             sizeof(cplx) * (size_t)(d.n_pad - n) * d.qr_m_pad, st));
  launch_qr_factor(dd, 1, d.n_pad, d.m_pad, ws, (cplx*)w.vbuf.p, d.qr_m_pad, (cplx*)w.tbuf.p, npan, 0, st);
  qr_extract_r_kernel<<<grid_of((long long)k * n), 256, 0, st>>>(ws + d.qr_off, d.qr_m_pad, k, n, (cplx*)w.R.p);
  qr_identity_kernel<<<grid_of((long long)d.n_pad * d.m_pad), 256, 0, st>>>(ws, d.m_pad, n, d.n_pad,
                                                                             (int*)w.order.p, (GateOut*)w.out.p, k);
  launch_qr_apply(dd, 1, d.n_pad, (int)d.qr_m_pad, ws, (const cplx*)w.vbuf.p, d.qr_m_pad, (const cplx*)w.tbuf.p, npan,
                  (const int*)w.order.p, d.n_pad, (const GateOut*)w.out.p, st);
  q_to_site_kernel<<<grid_of((long long)k * m), 256, 0, st>>>(ws + d.qr_off, d.qr_m_pad, k, dl, dr, right, site,
                                                              s.chi);
  s.launches += 4 + 2 * npan + 1 + npan + 1;
  return k;
}

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


// sweep_left_of (mps.cpp:69-80): site i = Q (Dl,2,k), site i+1 = R * site i+1.
void left_step(State& s, QrWork& w, int i) {
  const int dl = (int)s.sdl[i], dr = (int)s.sdr[i];
  const int m = 2 * dl, n = dr;
  cplx* site = s.sites + (long long)i * s.stride;
  cplx* next = s.sites + (long long)(i + 1) * s.stride;
  w.W.ensure(sizeof(cplx) * (size_t)m * n);
  w.R.ensure(sizeof(cplx) * (size_t)std::min(m, n) * n);
  w.tmp.ensure(sizeof(cplx) * (size_t)s.stride);
  int k;
  if (site_qr_supported(m, n)) {
    k = fast_site_qr(s, w, site, dl, dr, 0);
  } else if (tc_qr(m, n)) {
    k = tc_site_qr(s, w, site, dl, dr, 0);
  } else {
    cplx* W = (cplx*)w.W.p;
    launch_copy_matrix(site, s.chi, W, n, m, n, 0, s.st);
    ++s.launches;
    k = thin_qr(s, w, W, m, n, site, s.chi, (cplx*)w.R.p, n);
  }
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
  if (site_qr_supported(m, n)) {
    fast_site_qr(s, w, site, dl, dr, 1);
  } else if (tc_qr(m, n)) {
    tc_site_qr(s, w, site, dl, dr, 1);
  } else {
    cplx* W = (cplx*)w.W.p;
    launch_site_adjoint(site, s.chi, dl, dr, W, n, s.st);
    ++s.launches;
    thin_qr(s, w, W, m, n, (cplx*)w.Q.p, k, (cplx*)w.R.p, n);
    launch_site_from_adjoint((cplx*)w.Q.p, k, k, dr, site, s.chi, s.st);
    ++s.launches;
  }
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
  join_aux(s);
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
  s.center = -1;
}

void sweep_right_impl(State& s, int i0, int i1) {
  if (i0 < 1 || i1 > s.n - 1 || i0 > i1 + 1) fail(MPSIM_EINVAL, "right sweep range out of bounds");
  DeviceGuard g(s.device);
  QrWork w;
  for (int i = i1; i >= i0; --i) right_step(s, w, i);
  join_aux(s);
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
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
  join_aux(s);
  CKC(cudaStreamSynchronize(s.st));
  nrm.release();
  return n2;
}

void move_center_impl(State& s, int c) {
  NvtxRange nv("mpsim: move_center (QR sweeps)");
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
  join_aux(s);
  CKC(cudaStreamSynchronize(s.st));
  CKC(cudaGetLastError());
  if (std::sqrt(n2) < 1e-14) fail(MPSIM_ENUMERIC, "cannot canonicalize a zero-norm state");
  s.center = c;
}

}  // namespace mpsim_gpu
