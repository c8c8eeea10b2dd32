// Split epilogue of a batched two-qubit layer: singular values, the
// reference truncation rule, renormalisation and the write-back of
//   site q   <- U        (Dl, 2, k)   (gate_apply.cpp:136)
//   site q+1 <- S V^dag  (k, 2, Dr)   (gate_apply.cpp:137-138, scale_rows :54-64)
// After the Jacobi sweeps the vectors of X are orthogonal: X = U_X Sigma.
//   f = 0 (X = theta, or R^H of theta^H = QR):  U = X/sigma,  S V^dag = U^H theta = (X/sigma)^H X0
//   f = 1 (X = theta^H, or R^H of theta = QR):  S V^dag = X^H, U = theta X Sigma^-2 = X0^H X / sigma^2
// so one "cross-Gram" kernel (C = P^H Q over vector-major operands) produces
// whichever factor is not a plain copy. With two-step QR preconditioning
// (pre = 2) X is Z = Q1 [X_kept; 0], already in descending-sigma order.
#include <float.h>

#include "common.cuh"
#include "pair_gemm.cuh"

namespace mpsim_gpu {

// ---- vector norms: one warp per vector, coalesced along the element axis.
__global__ void __launch_bounds__(256) norms_kernel(const GateDesc* __restrict__ gates,
                                                    const cplx* __restrict__ ws,
                                                    double* __restrict__ sigma, long long sig_stride) {
  const GateDesc& g = gates[blockIdx.y];
  const int v = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (v >= g.n) return;
  const cplx* x = ws + g.ws_off + (long long)v * g.m_pad;
  double s = 0.0;
  for (int e = lane; e < g.m; e += 32) s += cabs2(xs_get(x, g.m_pad, e));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sigma[blockIdx.y * sig_stride + v] = sqrt(s);
}

// ---- sort descending + truncation rule (svd.hpp:48-74) + renorm factor.
// One CTA (1024 threads) per gate; its keys sit in dynamic shared memory
// (12 bytes per value, n <= kMaxSortN).
__global__ void __launch_bounds__(1024) truncate_kernel(const GateDesc* __restrict__ gates,
                                                        double* __restrict__ sigma,
                                                        int* __restrict__ order, long long sig_stride,
                                                        GateOut* __restrict__ out,
                                                        const double* __restrict__ frob2, double floor_rel2) {
  const GateDesc& g = gates[blockIdx.y];
  // Singular values at the rounding-noise level of ||theta||_F are exact
  // zeros of a structurally rank-deficient theta (Clifford gates on product
  // states, SWAPs): report them as 0 so svd.hpp:58's cutoff-0 rule trims them
  // the way an exact-arithmetic decomposition (and LAPACK/Eigen on such
  // structured inputs) does. Below any cutoff >= 1e-25 this changes nothing.
  const double floor2 = floor_rel2 * frob2[blockIdx.y];
  __shared__ int bad;
  const int n = g.n;
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  extern __shared__ double sort_smem[];
  double* key = sort_smem;
  int* idx = reinterpret_cast<int*>(sort_smem + n2);
  double* sg = sigma + blockIdx.y * sig_stride;
  int* od = order + blockIdx.y * sig_stride;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    double v = i < n ? sg[i] : -1.0;
    if (i < n && v * v <= floor2) v = 0.0;
    if (i < n && !(v <= DBL_MAX)) bad = 1;  // NaN or inf
    key[i] = v;
    idx[i] = i;
  }
  __syncthreads();
  // Bitonic sort: descending key, ascending index on ties.
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const double ki = key[i], kj = key[j];
          const int ii = idx[i], ij = idx[j];
          // "i before j" in the final order
          const bool i_first = (ki > kj) || (ki == kj && ii < ij);
          if (desc != i_first) {
            key[i] = kj;
            key[j] = ki;
            idx[i] = ij;
            idx[j] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sg[i] = key[i];
    od[i] = idx[i];
  }
  if (threadIdx.x == 0) {
    // Same accumulation order as the reference loop.
    double total = 0.0;
    for (int i = 0; i < n; ++i) total += key[i] * key[i];
    long long keep = n;
    if (total > 0.0) {
      double tail = 0.0;
      while (keep > 1 && tail + key[keep - 1] * key[keep - 1] <= g.cutoff * total) {
        tail += key[keep - 1] * key[keep - 1];
        --keep;
      }
    } else {
      keep = 1;
    }
    const long long cap = g.max_bond < 1 ? 1 : g.max_bond;
    if (keep > cap) keep = cap;
    double dropped = 0.0;
    for (long long i = keep; i < n; ++i) dropped += key[i] * key[i];
    const double w = total > 0.0 ? dropped / total : 0.0;
    GateOut o;
    o.k = (int)keep;
    o.w = w;
    o.scale = w > 0.0 ? 1.0 / sqrt(1.0 - w) : 1.0;  // gate_apply.cpp:44-51
    o.status = bad ? 3 : 0;
    out[blockIdx.y] = o;
  }
}

// Element e of vector j of the converged operand: the Jacobi X or, with
// two-step QR preconditioning, Z = Q1 [X; 0] (both split planes).
__device__ __forceinline__ cplx x_elem(const GateDesc& g, const cplx* X, int j, int e) {
  return xs_get(X + (long long)j * g.m_pad, g.m_pad, e);
}

// ---- plain-copy factor.
//  trans 0: site q   [e*chi + j]                 = X[o_j][e] / sigma_j   (e < m = 2dl, j < k)
//  trans 1: site q+1 [j*2chi + p1*chi + r]       = scale * conj(X[o_j][e]), e = p1*dr + r
__global__ void __launch_bounds__(256) copy_factor_kernel(const GateDesc* __restrict__ gates,
                                                          const cplx* __restrict__ ws,
                                                          const double* __restrict__ sigma,
                                                          const int* __restrict__ order, long long sig_stride,
                                                          const GateOut* __restrict__ out) {
  const GateDesc& g = gates[blockIdx.z];
  const GateOut o = out[blockIdx.z];
  const int k = o.k;
  const int j0 = blockIdx.y * 32, e0 = blockIdx.x * 32;
  if (j0 >= k || e0 >= g.m) return;
  const double* sg = sigma + blockIdx.z * sig_stride;
  const int* od = order + blockIdx.z * sig_stride;
  const cplx* X = ws + g.ws_off;
  __shared__ cplx tile[32][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  if (g.f == 0) {
    // Read along e (coalesced), write along j (coalesced) through a transpose.
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj, e = e0 + tx;
      cplx v = make_double2(0.0, 0.0);
      if (j < k && e < g.m) {
        const double s = sg[j];
        if (s > 0.0) {
          const cplx x = x_elem(g, X, g.pre >= 2 ? j : od[j], e);
          v = make_double2(x.x / s, x.y / s);
        } else {
          v = make_double2(e == j ? 1.0 : 0.0, 0.0);  // zero matrix: any unit column
        }
      }
      tile[jj][tx] = v;
    }
    __syncthreads();
    for (int ee = ty; ee < 32; ee += 8) {
      const int e = e0 + ee, j = j0 + tx;
      if (e < g.m && j < k) g.u_out[(long long)e * g.ldu + j] = tile[tx][ee];
    }
  } else {
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj, e = e0 + tx;
      if (j < k && e < g.m) {
        const cplx x = x_elem(g, X, g.pre >= 2 ? j : od[j], e);
        const long long off = (long long)j * g.ldv + (long long)(e / g.vsplit) * g.vsplit_ld + e % g.vsplit;
        g.v_out[off] = make_double2(o.scale * x.x, -o.scale * x.y);
      }
    }
  }
}

// ---- cross-Gram factor, C[a][b] = sum_e conj(P_a[e]) Q_b[e], on DMMA
// (pair_gemm.cuh), one 32 x 32 block of C per CTA.
//  f = 0: a = j (X, sigma order), b = v (X0): site q+1[(j*2+p1)*chi + r] = scale/sigma_j * C, v = p1*dr + r
//  f = 1: a = v (X0), b = j (X, sigma order): site q  [v*chi + j]        = C / sigma_j^2
struct CrossSmem {
  union {
    double buf[2][pg::kBuf];
    double Wx[64 * 65];
  } u;
  cplx W[32 * 33];
};

__global__ void __launch_bounds__(256, 2) cross_gram_kernel(const GateDesc* __restrict__ gates,
                                                            const cplx* __restrict__ ws,
                                                            const double* __restrict__ sigma,
                                                            const int* __restrict__ order, long long sig_stride,
                                                            const GateOut* __restrict__ out,
                                                            const double* __restrict__ frob2, double floor_rel2) {
  const GateDesc& g = gates[blockIdx.z];
  const GateOut o = out[blockIdx.z];
  const int k = o.k;
  // Kept vectors at the rounding-noise level (sigma^2 <= floor, see
  // jacobi.cu) were never orthogonalised against the large ones, so the
  // cross-Gram formula is meaningless for them: they contribute an exact
  // zero (their true weight is below 64 eps ||theta||_F).
  const double floor2 = floor_rel2 * frob2[blockIdx.z];
  const int n_a = g.f == 0 ? k : g.n0;
  const int n_b = g.f == 0 ? g.n0 : k;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  if (a0 >= n_a || b0 >= n_b) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CrossSmem& S = *reinterpret_cast<CrossSmem*>(smem_raw);
  const double* sg = sigma + blockIdx.z * sig_stride;
  const int* od = order + blockIdx.z * sig_stride;
  const cplx* X = ws + g.ws_off;
  const cplx* X0 = ws + g.x0_off;
  const int t = threadIdx.x;
  auto xvec = [&](int j) { return X + (long long)(g.pre >= 2 ? j : od[j]) * g.m_pad; };
  auto x0vec = [&](int v) { return X0 + (long long)v * g.x0_ld; };
  // padding vectors (beyond n_a / n_b) load a valid vector, results discarded
  auto pa = [&](int v) { const int a = min(a0 + v, n_a - 1); return g.f == 0 ? xvec(a) : x0vec(a); };
  auto qb = [&](int v) { const int b = min(b0 + v, n_b - 1); return g.f == 0 ? x0vec(b) : xvec(b); };
  pg::Loader ld;
  ld.init(pa, qb, g.f == 0 ? g.m_pad : g.x0_ld, g.f == 0 ? g.x0_ld : g.m_pad, t);
  pg::cross_gram(ld, S.u.buf, S.u.Wx, S.W, 33, 0, g.m_pad, t);
  for (int idx = t; idx < 32 * 32; idx += 256) {
    const int ai = a0 + idx / 32, bi = b0 + idx % 32;
    if (ai >= n_a || bi >= n_b) continue;
    const cplx c = S.W[(idx / 32) * 33 + idx % 32];
    if (g.f == 0) {
      const double s = sg[ai];
      const double f = s * s > floor2 && s > 0.0 ? o.scale / s : 0.0;
      const long long off = (long long)ai * g.ldv + (long long)(bi / g.vsplit) * g.vsplit_ld + bi % g.vsplit;
      g.v_out[off] = make_double2(f * c.x, f * c.y);
    } else {
      const double s = sg[bi];
      cplx v;
      if (s * s > floor2 && s > 0.0) {
        const double f = 1.0 / (s * s);
        v = make_double2(f * c.x, f * c.y);
      } else {
        v = make_double2(s == 0.0 && ai == bi ? 1.0 : 0.0, 0.0);
      }
      g.u_out[(long long)ai * g.ldu + bi] = v;
    }
  }
}

// ---- orthonormalisation of the kept vectors (first order, in place).
// The converged Jacobi vectors are orthogonal only to the sweep tolerance
// (relative off-diagonals <= 4 eps max(sqrt(m), 32)), so the split
// U (U^H theta) [f = 0] or (theta V Sigma^-2)(Sigma V^H) [f = 1] reproduces
// theta only to that tolerance per gate, and the excess compounds over a
// circuit (measured on the C4 window: ~1e-11 by the first truncating gate).
// With Y the kept normalised vectors and E = Y^H Y - I (FP64, ~1e-14),
// Y <- Y (I - E / 2) makes them orthonormal to O(E^2); both split formulas
// then apply the exact projector onto span(Y). In terms of the sigma-scaled
// operand: X_j <- X_j - sum_i X_i F[i][j], F[i][j] = E[i][j] sigma_j /
// (2 sigma_i); the product is a first-order term, computed in FP32.
__global__ void __launch_bounds__(256, 2) ortho_gram_kernel(const GateDesc* __restrict__ gates,
                                                            const cplx* __restrict__ ws,
                                                            const double* __restrict__ sigma,
                                                            const int* __restrict__ order, long long sig_stride,
                                                            const GateOut* __restrict__ out,
                                                            const double* __restrict__ frob2, double floor_rel2,
                                                            float2* __restrict__ fbuf, int kcap) {
  const GateDesc& g = gates[blockIdx.z];
  const int k = out[blockIdx.z].k;
  const int a0 = blockIdx.y * 32, b0 = blockIdx.x * 32;
  if (a0 >= k || b0 >= k) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CrossSmem& S = *reinterpret_cast<CrossSmem*>(smem_raw);
  const double floor2 = floor_rel2 * frob2[blockIdx.z];
  const double* sg = sigma + blockIdx.z * sig_stride;
  const int* od = order + blockIdx.z * sig_stride;
  const cplx* X = ws + g.ws_off;
  const int t = threadIdx.x;
  auto xvec = [&](int j) { return X + (long long)(g.pre >= 2 ? j : od[j]) * g.m_pad; };
  auto pa = [&](int v) { return xvec(min(a0 + v, k - 1)); };
  auto qb = [&](int v) { return xvec(min(b0 + v, k - 1)); };
  pg::Loader ld;
  ld.init(pa, qb, g.m_pad, g.m_pad, t);
  pg::cross_gram(ld, S.u.buf, S.u.Wx, S.W, 33, 0, g.m_pad, t);
  float2* F = fbuf + (long long)blockIdx.z * kcap * kcap;
  for (int idx = t; idx < 32 * 32; idx += 256) {
    const int i = a0 + idx / 32, j = b0 + idx % 32;
    if (i >= k || j >= k) continue;
    const double si = sg[i], sj = sg[j];
    float2 f = make_float2(0.0f, 0.0f);
    if (si * si > floor2 && sj * sj > floor2) {
      const cplx c = S.W[(idx / 32) * 33 + idx % 32];
      const double e_re = c.x / (si * sj) - (i == j ? 1.0 : 0.0), e_im = i == j ? 0.0 : c.y / (si * sj);
      const double r = 0.5 * sj / si;
      f = make_float2((float)(r * e_re), (float)(r * e_im));
    }
    F[(long long)i * kcap + j] = f;
  }
}

// T_j[e] = sum_i X_i[e] F[i][j] (FP32) for a 32 x 32 tile of (rows e, kept j).
__global__ void __launch_bounds__(256) ortho_tmul_kernel(const GateDesc* __restrict__ gates,
                                                         const cplx* __restrict__ ws,
                                                         const int* __restrict__ order, long long sig_stride,
                                                         const GateOut* __restrict__ out,
                                                         const float2* __restrict__ fbuf, int kcap,
                                                         float2* __restrict__ tbuf, long long tstride) {
  const GateDesc& g = gates[blockIdx.z];
  const int k = out[blockIdx.z].k;
  const int e0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (j0 >= k || e0 >= g.m) return;
  __shared__ float2 xs[32][33], fs[32][33];
  const int* od = order + blockIdx.z * sig_stride;
  const cplx* X = ws + g.ws_off;
  const float2* F = fbuf + (long long)blockIdx.z * kcap * kcap;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int i0 = 0; i0 < k; i0 += 32) {
    for (int ii = ty; ii < 32; ii += 8) {
      const int i = i0 + ii, e = e0 + tx;
      float2 xv = make_float2(0.f, 0.f);
      if (i < k && e < g.m) {
        const cplx x = xs_get(X + (long long)(g.pre >= 2 ? i : od[i]) * g.m_pad, g.m_pad, e);
        xv = make_float2((float)x.x, (float)x.y);
      }
      xs[ii][tx] = xv;  // [i][e]
      fs[ii][tx] = (i < k && j0 + tx < k) ? F[(long long)i * kcap + j0 + tx] : make_float2(0.f, 0.f);  // [i][j]
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < 32; ++ii) {
      const float2 x = xs[ii][tx];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float2 f = fs[ii][ty + 8 * h];
        acc[h].x = fmaf(x.x, f.x, fmaf(-x.y, f.y, acc[h].x));
        acc[h].y = fmaf(x.x, f.y, fmaf(x.y, f.x, acc[h].y));
      }
    }
    __syncthreads();
  }
  float2* T = tbuf + blockIdx.z * tstride;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int j = j0 + ty + 8 * h, e = e0 + tx;
    if (j < k && e < g.m) T[(long long)j * g.m_pad + e] = acc[h];
  }
}

// X_j[e] -= T_j[e] over the kept vectors.
__global__ void __launch_bounds__(256) ortho_apply_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                          const int* __restrict__ order, long long sig_stride,
                                                          const GateOut* __restrict__ out,
                                                          const float2* __restrict__ tbuf, long long tstride) {
  const GateDesc& g = gates[blockIdx.z];
  const int k = out[blockIdx.z].k;
  const int j = blockIdx.y, e = blockIdx.x * 256 + threadIdx.x;
  if (j >= k || e >= g.m) return;
  const int* od = order + blockIdx.z * sig_stride;
  double* x = reinterpret_cast<double*>(ws + g.ws_off + (long long)(g.pre >= 2 ? j : od[j]) * g.m_pad);
  const float2 d = tbuf[blockIdx.z * tstride + (long long)j * g.m_pad + e];
  x[e] -= (double)d.x;
  x[g.m_pad + e] -= (double)d.y;
}

void launch_orthonormalize(const GateDesc* d_gates, int n_gates, int max_m, int kcap, cplx* ws, const double* sigma,
                           const int* order, long long sig_stride, const GateOut* d_out, const double* frob2,
                           double floor_rel2, float2* fbuf, float2* tbuf, long long tstride, cudaStream_t st) {
  const int kb = (kcap + 31) / 32;
  ortho_gram_kernel<<<dim3(kb, kb, n_gates), 256, sizeof(CrossSmem), st>>>(d_gates, ws, sigma, order, sig_stride,
                                                                          d_out, frob2, floor_rel2, fbuf, kcap);
  ortho_tmul_kernel<<<dim3((max_m + 31) / 32, kb, n_gates), 256, 0, st>>>(d_gates, ws, order, sig_stride, d_out,
                                                                         fbuf, kcap, tbuf, tstride);
  ortho_apply_kernel<<<dim3((max_m + 255) / 256, kcap, n_gates), 256, 0, st>>>(d_gates, ws, order, sig_stride,
                                                                             d_out, tbuf, tstride);
}

void split_init() {
  cudaFuncSetAttribute(cross_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CrossSmem));
  cudaFuncSetAttribute(ortho_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CrossSmem));
}

void launch_norms(const GateDesc* d_gates, int n_gates, int max_n, const cplx* ws, double* sigma,
                  long long sig_stride, cudaStream_t st) {
  norms_kernel<<<dim3((max_n + 7) / 8, n_gates), 256, 0, st>>>(d_gates, ws, sigma, sig_stride);
}

void launch_truncate(const GateDesc* d_gates, int n_gates, double* sigma, int* order, long long sig_stride,
                     GateOut* d_out, const double* frob2, double floor_rel2, int max_n, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(truncate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSortN * 12);
    init = true;
  }
  int p2 = 1;
  while (p2 < max_n) p2 <<= 1;
  truncate_kernel<<<dim3(1, n_gates), 1024, (size_t)p2 * 12, st>>>(d_gates, sigma, order, sig_stride, d_out, frob2, floor_rel2);
}

void launch_write_factors(const GateDesc* d_gates, int n_gates, int max_m, int max_n, int max_n0, const cplx* ws,
                          const double* sigma, const int* order, long long sig_stride, const GateOut* d_out,
                          const double* frob2, double floor_rel2, cudaStream_t st) {
  // k <= n, so n bounds every tile count.
  copy_factor_kernel<<<dim3((max_m + 31) / 32, (max_n + 31) / 32, n_gates), 256, 0, st>>>(
      d_gates, ws, sigma, order, sig_stride, d_out);
  cross_gram_kernel<<<dim3((max_n0 + 31) / 32, (max_n0 + 31) / 32, n_gates), 256, sizeof(CrossSmem), st>>>(
      d_gates, ws, sigma, order, sig_stride, d_out, frob2, floor_rel2);
}

}  // namespace mpsim_gpu
