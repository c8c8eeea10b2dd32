// Shared device-side definitions for the B200 MPS gate-application engine.
//
// Data layout in HBM:
//   * Site store: n_sites slots of (chi_cap x 2 x chi_cap) complex128, row-major
//     (l, p, r) with r fastest — the reference's site layout (tensor.hpp:139-148,
//     "(l*2+p)*Dr + r") with the leading dimension padded to chi_cap. Real bond
//     dimensions live in the host-side bond array (mps.hpp:72-74).
//   * Jacobi workspace, per two-qubit gate: X (n_pad vectors x m_pad elements,
//     vector-major, complex128) and a pristine copy X0 of the same matrix.
//     X = theta (vectors = columns (p1',r)) when 2Dl >= 2Dr, else X = theta^H
//     (vectors = conjugated rows (l,p0')), so the vector count is
//     n = min(2Dl, 2Dr) — the number of singular values the reference's thin
//     SVD returns (svd.hpp:95).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

namespace mpsim_gpu {

// A/B switches of sweep policy and kernel variants (MPSIM_QR, MPSIM_JACOBI,
// MPSIM_CROSS*, ...): read from the environment only in an A/B build
// (make AB=1 -> -DMPSIM_AB_KNOBS). The product library ignores them, so a stray
// variable cannot change numerics of the drop-in path.
inline const char* ab_knob(const char* name) {
#ifdef MPSIM_AB_KNOBS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

typedef double2 cplx;

// Block-Jacobi geometry: W vectors per block, a pair of blocks = 2W vectors,
// E elements per streamed chunk.
constexpr int kW = 16;
constexpr int kP = 2 * kW;  // vectors per block pair
constexpr int kE = 64;      // element chunk
constexpr int kPad = 33;    // padded smem row (complex) for [e][vector] tiles
// Per-gate singular-value sorts (de Rijk order, truncation) run in one CTA
// with the keys in shared memory: 12 bytes per vector -> 16384 vectors
// (bond dimensions up to 8192).
constexpr int kMaxSortN = 16384;

// One two-qubit gate of a batched layer launch.
struct GateDesc {
  int q;            // left site; the gate acts on (q, q+1)
  int dl, dm, dr;   // bond dims left of q, between q and q+1, right of q+1
  int m, n;         // vector length / vector count of X (n = min(2dl, 2dr))
  int trans;        // 0: X = theta ; 1: X = theta^H
  int n_pad, m_pad; // n_pad multiple of kP, m_pad multiple of kE
  int nb;           // blocks of kW vectors (n_pad / kW), even
  long long ws_off; // offset (complex elements) of X in the workspace; X0 follows
  // Output addressing of the two factors:
  //   U (M x k):       u_out[e * ldu + j]
  //   S V^dag (k x N): v_out[j * ldv + (v / vsplit) * vsplit_ld + v % vsplit]
  // For an MPS gate U is site q viewed as (2Dl x chi) and S V^dag is site
  // q+1 viewed as (k, 2, Dr) with padded rows (vsplit = Dr, vsplit_ld = chi).
  cplx* u_out;
  cplx* v_out;
  long long ldu, ldv, vsplit_ld;
  int vsplit, pad2;
  long long max_bond;
  double cutoff;
  cplx u[16];       // 4x4 gate, (low, high) basis, row = 2*p_low + p_high (circuit.hpp:20-22)
  // Factor formula of the split epilogue (split.cu): f = 0: the converged X
  // holds sigma * (left singular vectors); f = 1: it holds sigma * (right
  // singular vectors)^*. X0 (the pristine operand the other factor is
  // contracted with) has n0 vectors of length m, stride x0_ld.
  int f, n0;
  long long x0_off, x0_ld;
  // QR preconditioning (qr_pre.cu), pre = 1: theta -> QR operand (n vectors
  // of length qr_m, stride qr_m_pad at qr_off, orientation trans) = Q R; the
  // Jacobi operand X is R^H (n vectors of length m = n) and f = trans ^ 1.
  // pre = 2: a second step R^H = Q2 R2 (in the y2 area), Jacobi on R2^H, then
  // Z = Q1 [X; 0] in the QR area holds sigma * (left vectors): f = trans.
  // pre = 4 (A/B): two more steps, R2^H = Q3 R3 (y3 area), R3^H = Q4 R4 (y4
  // area), Jacobi on R4^H; theta = Q1 Q3 R4^H (Q2 Q4)^H, so Z = Q1 [Q3 X; 0].
  int pre, qr_m;
  long long qr_off, qr_m_pad, y2_off;
  long long y3_off, y4_off;
  int zsrc_ordered;  // Z formation reads its source in kept order (no permutation)
  int pad4;
};

// Workspace layout of one descriptor starting at `off` (complex elements);
// returns the span. Without preconditioning: X (n_pad x m_pad) then X0 (same).
// pre = 1: X = R^H (n_pad x m_pad, m = n), X0 (n0 = qr_m vectors x m_pad), the
// QR operand (n_pad x qr_m_pad). pre = 2: X = R2^H (n_pad x m_pad, m = n), X0
// (n vectors x qr_m_pad, orientation trans), the QR operand / Z, the y2 area.
// The descriptor holds the Jacobi-phase view; phase_desc() (engine.cu) derives
// the others.
inline long long desc_layout(GateDesc& d, long long off, int pre) {
  d.pre = pre;
  d.ws_off = off;
  d.y2_off = 0;
  d.y3_off = 0;
  d.y4_off = 0;
  d.zsrc_ordered = 0;
  if (pre == 0) {
    d.f = d.trans;
    d.n0 = d.n;
    d.x0_ld = d.m_pad;
    d.x0_off = off + (long long)d.n_pad * d.m_pad;
    d.qr_m = 0;
    d.qr_m_pad = 0;
    d.qr_off = 0;
    return 2LL * d.n_pad * d.m_pad;
  }
  d.qr_m = d.m;
  d.qr_m_pad = d.m_pad;
  d.m = d.n;
  d.m_pad = ((d.n + kE - 1) / kE) * kE;
  d.x0_off = off + (long long)d.n_pad * d.m_pad;
  if (pre == 1) {
    d.f = d.trans ^ 1;
    d.n0 = d.qr_m;
    d.x0_ld = d.m_pad;
    d.qr_off = d.x0_off + (long long)d.n0 * d.x0_ld;
    return (long long)d.n_pad * d.m_pad + (long long)d.n0 * d.x0_ld + (long long)d.n_pad * d.qr_m_pad;
  }
  d.f = d.trans;
  d.n0 = d.n;
  d.x0_ld = d.qr_m_pad;
  d.qr_off = d.x0_off + (long long)d.n_pad * d.x0_ld;
  d.y2_off = d.qr_off + (long long)d.n_pad * d.qr_m_pad;
  if (pre == 4) {
    d.y3_off = d.y2_off + (long long)d.n_pad * d.m_pad;
    d.y4_off = d.y3_off + (long long)d.n_pad * d.m_pad;
    return 4LL * d.n_pad * d.m_pad + 2LL * d.n_pad * d.qr_m_pad;
  }
  return 2LL * d.n_pad * d.m_pad + 2LL * d.n_pad * d.qr_m_pad;
}

// Per-gate outputs of the split epilogue.
struct GateOut {
  int k;            // kept rank (new bond)
  int status;       // 0 ok, 3 numeric (non-convergence / non-finite)
  double w;         // discarded weight (pre-rescale, gate_apply.cpp:143)
  double scale;     // 1/sqrt(1-w) if w > 0 else 1 (gate_apply.cpp:44-51)
};

// One single-qubit gate.
struct Gate1Desc {
  int q, dl, dr, pad;
  cplx u[4];
};

struct GemmArgs {
  int M, N, K;
  const cplx* A;
  long long lda;
  int opA;  // 0: A[i][k] = A[i*lda+k]; 1: A[i][k] = conj(A[k*lda+i])
  const cplx* B;
  long long ldb;
  int opB;  // 0: B[k][j] = B[k*ldb+j]; 1: B[k][j] = conj(B[j*ldb+k])
  cplx* C;
  long long ldc;
  cplx alpha;
  int accumulate;  // C = alpha*op(A)op(B) (+ C if accumulate)
};

__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfmac(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// acc += a * b with every product and sum rounded separately (no contraction).
__device__ __forceinline__ void cmac_rn(cplx& acc, cplx a, cplx b) {
  const double re = __dadd_rn(__dmul_rn(a.x, b.x), -__dmul_rn(a.y, b.y));
  const double im = __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x));
  acc.x = __dadd_rn(acc.x, re);
  acc.y = __dadd_rn(acc.y, im);
}
__device__ __forceinline__ cplx conjc(cplx a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }

// Every workspace operand (the Jacobi X, X0, the QR operand / Z, the y2 area,
// the QR reflectors) keeps each vector as split planes inside its m_pad-complex
// slot: Re in doubles [0, m_pad), Im in [m_pad, 2 m_pad) — so two rows of one
// plane are one 16-byte cp.async into vector-major shared memory
// (jacobi_split.cu, pair_gemm.cuh).
__device__ __forceinline__ cplx xs_get(const cplx* vec, long long m_pad, long long e) {
  const double* d = reinterpret_cast<const double*>(vec);
  return make_double2(d[e], d[m_pad + e]);
}
__device__ __forceinline__ void xs_set(cplx* vec, long long m_pad, long long e, cplx v) {
  double* d = reinterpret_cast<double*>(vec);
  d[e] = v.x;
  d[m_pad + e] = v.y;
}

}  // namespace mpsim_gpu
