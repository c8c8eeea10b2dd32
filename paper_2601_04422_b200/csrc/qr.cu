// Blocked Householder QR for orthogonality-centre moves (thin_qr, mps.cpp:57-65;
// sweep_left_of / sweep_right_of, mps.cpp:69-95).
//
// A (m x n, row-major, ld) is factored in place LAPACK-style (zgeqrf): panels
// of 32 columns are factored by one CTA (Householder vectors below the
// diagonal, R on and above it, tau, and the compact-WY T factor of the panel,
// Q_panel = I - V T V^H); the trailing matrix is updated with three complex
// GEMMs, A2 <- (I - V T^H V^H) A2. The thin Q (m x k, k = min(m, n)) is then
// formed by applying the block reflectors to [I; 0] in reverse order.
#include <cstdlib>

#include "common.cuh"

namespace mpsim_gpu {

constexpr int kQB = 32;  // panel width

// acc += sum over rows r0, r0 + 32, ... < L of conj(a[r]) b[r] (cfmac), in
// that order, with four rows' loads in flight per lane (the panel lives in
// L2, so a one-load-at-a-time loop is latency bound).
__device__ __forceinline__ void dot_rows(cplx& acc, const cplx* a, const cplx* b, int r0, int L) {
  int r = r0;
  for (; r + 96 < L; r += 128) {
    cplx aa[4], bb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      aa[q] = a[r + 32 * q];
      bb[q] = b[r + 32 * q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) cfmac(acc, aa[q], bb[q]);
  }
  for (; r < L; r += 32) cfmac(acc, a[r], b[r]);
}

// Factor panel columns [c0, c0 + jb) of A (row-major, ld), rows [c0, m).
// Writes: A (R part + Householder vectors below the diagonal), V (explicit,
// row-major (m - c0) x kQB, unit diagonal, zeros above), T (kQB x kQB,
// row-major, upper triangular), tau[c0 + j].
__global__ void __launch_bounds__(1024) qr_panel_kernel(cplx* __restrict__ A, long long lda, int m, int c0, int jb,
                                                        cplx* __restrict__ P, cplx* __restrict__ V,
                                                        cplx* __restrict__ T, cplx* __restrict__ tau,
                                                        int chunked) {
  const int L = m - c0;  // rows in the panel
  const int t = threadIdx.x, warp = t / 32, lane = t % 32, nw = blockDim.x / 32;
  // P: column-major panel copy, column j at P + j * L.
  for (int idx = t; idx < L * jb; idx += blockDim.x) {
    const int r = idx / jb, j = idx % jb;
    P[(long long)j * L + r] = A[(long long)(c0 + r) * lda + c0 + j];
  }
  __shared__ double red[32];
  __shared__ cplx s_tau, s_beta, s_alpha;
  __shared__ cplx z[kQB];
  __shared__ cplx part[kQB][kQB];  // partial column dots per (column, row chunk)
  __shared__ cplx Ts[kQB][kQB + 1];
  for (int i = t; i < kQB * (kQB + 1); i += blockDim.x) Ts[i / (kQB + 1)][i % (kQB + 1)] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    cplx* x = P + (long long)j * L;
    // ||x[j+1:]||^2
    double s = 0.0;
    for (int r = j + 1 + t; r < L; r += blockDim.x) s += cabs2(x[r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (t == 0) {
      double xn2 = 0.0;
      for (int w = 0; w < nw; ++w) xn2 += red[w];
      const cplx alpha = x[j];
      cplx tv = make_double2(0.0, 0.0), beta = alpha;
      if (!(xn2 == 0.0 && alpha.y == 0.0)) {  // zlarfg
        const double b = -copysign(sqrt(cabs2(alpha) + xn2), alpha.x);
        tv = make_double2((b - alpha.x) / b, -alpha.y / b);
        beta = make_double2(b, 0.0);
      }
      s_tau = tv;
      s_beta = beta;
      s_alpha = alpha;
    }
    __syncthreads();
    const cplx tv = s_tau, beta = s_beta, alpha = s_alpha;
    if (tv.x != 0.0 || tv.y != 0.0) {
      // v = x / (alpha - beta) below the diagonal
      const cplx d = make_double2(alpha.x - beta.x, alpha.y - beta.y);
      const double dd = cabs2(d);
      const cplx inv = make_double2(d.x / dd, -d.y / dd);
      for (int r = j + 1 + t; r < L; r += blockDim.x) x[r] = cmul(x[r], inv);
    }
    if (t == 0) {  // row j is not touched by the scaling (alpha was staged)
      x[j] = beta;
      tau[c0 + j] = tv;
    }
    __syncthreads();
    // Phase A, one round of warp items: the dots v^H y of the columns the
    // reflector updates (column, row chunk) and the zlarft dots V[:, l]^H v
    // of T's column j (l < j, forward); ncols + j < 32 warps, so the chunks
    // are sized to keep all items in one round. Partial dots meet in shared
    // memory and are summed in chunk order (deterministic).
    const int ncols = jb - j - 1;
    const bool refl = tv.x != 0.0 || tv.y != 0.0;
    const int GA = chunked ? max(1, (nw - j) / max(ncols, 1)) : 1;
    const int CHA = ((L - j - 1 + GA - 1) / GA + 31) / 32 * 32;
    const int itemsU = (refl && ncols > 0) ? ncols * GA : 0;
    for (int it = warp; it < itemsU + j; it += nw) {
      cplx w = make_double2(0.0, 0.0);
      if (it < itemsU) {
        const int ci = it / GA, g = it % GA;
        const cplx* y = P + (long long)(j + 1 + ci) * L;
        const int rb = j + 1 + g * CHA, re = min(L, rb + CHA);
        if (g == 0 && lane == 0) w = y[j];
        dot_rows(w, x, y, rb + lane, re);
      } else {
        // v_j has an implicit 1 at row j and zeros above; v_l has its stored entries below l.
        const cplx* vl = P + (long long)(it - itemsU) * L;
        if (lane == 0) w = conjc(vl[j]);
        dot_rows(w, vl, x, j + 1 + lane, L);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w.x += __shfl_xor_sync(0xffffffffu, w.x, o);
        w.y += __shfl_xor_sync(0xffffffffu, w.y, o);
      }
      if (lane == 0) {
        if (it < itemsU) part[it / GA][it % GA] = w;
        else z[it - itemsU] = w;
      }
    }
    __syncthreads();
    // T column j: T[0:j, j] = -tau_j T[0:j, 0:j] (V[:, 0:j]^H v_j)  (zlarft, forward)
    if (t < j) {
      cplx acc = make_double2(0.0, 0.0);
      for (int l = t; l < j; ++l) cfma(acc, Ts[t][l], z[l]);
      const cplx v = cmul(acc, tv);
      Ts[t][j] = make_double2(-v.x, -v.y);
    }
    // Phase B: apply H^H = I - conj(tau) v v^H to columns j+1..jb-1, every
    // warp one (column, row chunk) item so late columns use the whole CTA.
    if (itemsU > 0) {
      const int GB = chunked ? max(1, nw / ncols) : 1;
      const int CHB = ((L - j - 1 + GB - 1) / GB + 31) / 32 * 32;
      for (int it = warp; it < ncols * GB; it += nw) {
        const int ci = it / GB, g = it % GB;
        cplx* y = P + (long long)(j + 1 + ci) * L;
        const int rb = j + 1 + g * CHB, re = min(L, rb + CHB);
        cplx w = part[ci][0];
        for (int q = 1; q < GA; ++q) w = cadd(w, part[ci][q]);
        const cplx f = cmul(conjc(tv), w);  // conj(tau) * (v^H y)
        if (g == 0 && lane == 0) y[j] = make_double2(y[j].x - f.x, y[j].y - f.y);
        int r = rb + lane;
        for (; r + 96 < re; r += 128) {  // four rows in flight per lane (x, y distinct columns)
          cplx xa[4], ya[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            xa[q] = x[r + 32 * q];
            ya[q] = y[r + 32 * q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const cplx u = cmul(xa[q], f);
            y[r + 32 * q] = make_double2(ya[q].x - u.x, ya[q].y - u.y);
          }
        }
        for (; r < re; r += 32) {
          const cplx u = cmul(x[r], f);
          y[r] = make_double2(y[r].x - u.x, y[r].y - u.y);
        }
      }
    }
    if (t == 0) Ts[j][j] = tv;
    __syncthreads();
  }
  // write back the panel, the explicit V and T
  for (int idx = t; idx < L * jb; idx += blockDim.x) {
    const int r = idx / jb, j = idx % jb;
    const cplx p = P[(long long)j * L + r];
    A[(long long)(c0 + r) * lda + c0 + j] = p;
    V[(long long)r * kQB + j] = r > j ? p : make_double2(r == j ? 1.0 : 0.0, 0.0);
  }
  for (int idx = t; idx < L * (kQB - jb); idx += blockDim.x) {
    const int r = idx / (kQB - jb), j = jb + idx % (kQB - jb);
    V[(long long)r * kQB + j] = make_double2(0.0, 0.0);
  }
  for (int idx = t; idx < kQB * kQB; idx += blockDim.x) T[idx] = Ts[idx / kQB][idx % kQB];
}

// Y (m x k, row-major ld) = [I_k; 0]
__global__ void set_identity_kernel(cplx* Y, long long ld, int m, int k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)m * k;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / k), c = (int)(i % k);
    Y[(long long)r * ld + c] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
}

// dst (rows x cols, ld_d) = op(src): op 0 copy, 1 conjugate transpose
// (src is cols x rows then), 2 upper-triangular copy (zeros below diagonal).
__global__ void copy_matrix_kernel(const cplx* __restrict__ src, long long ld_s, cplx* __restrict__ dst,
                                   long long ld_d, int rows, int cols, int op) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)rows * cols;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    cplx v;
    if (op == 1) {
      v = src[(long long)c * ld_s + r];
      v.y = -v.y;
    } else {
      v = src[(long long)r * ld_s + c];
      if (op == 2 && c < r) v = make_double2(0.0, 0.0);
    }
    dst[(long long)r * ld_d + c] = v;
  }
}

// Right-sweep operand: A[e][l] = conj(site[(l*2+p)*chi + r]), e = p*dr + r
// (the (Dl x 2Dr)^H matricisation, mps.cpp:84-95).
__global__ void site_adjoint_kernel(const cplx* __restrict__ site, int chi, int dl, int dr, cplx* __restrict__ A,
                                    long long lda) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)dl * 2 * dr;
       i += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(i / (2 * dr)), e = (int)(i % (2 * dr));
    const int p = e / dr, r = e % dr;
    cplx v = site[(long long)(l * 2 + p) * chi + r];
    v.y = -v.y;
    A[(long long)e * lda + l] = v;
  }
}

// site[(j*2+p)*chi + r] = conj(Q[e][j]), e = p*dr + r, j < k  (site i <- Q^H)
__global__ void site_from_adjoint_kernel(const cplx* __restrict__ Q, long long ldq, int k, int dr,
                                         cplx* __restrict__ site, int chi) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * 2 * dr;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / (2 * dr)), e = (int)(i % (2 * dr));
    const int p = e / dr, r = e % dr;
    cplx v = Q[(long long)e * ldq + j];
    v.y = -v.y;
    site[(long long)(j * 2 + p) * chi + r] = v;
  }
}

__global__ void sum_abs2_kernel(const cplx* __restrict__ A, long long lda, int rows, int cols, double* out) {
  double s = 0.0;
  for (long long i = threadIdx.x; i < (long long)rows * cols; i += blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    s += cabs2(A[(long long)r * lda + c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) t += red[w];
    *out = t;
  }
}

static unsigned blocks_for(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 4096) b = 4096;
  return (unsigned)b;
}

void launch_qr_panel(cplx* A, long long lda, int m, int c0, int jb, cplx* P, cplx* V, cplx* T, cplx* tau,
                     cudaStream_t st) {
  static const int chunked = [] {  // MPSIM_QR_PANEL_CHUNKED=0: one warp per column, no row chunks (A/B)
    const char* v = ab_knob("MPSIM_QR_PANEL_CHUNKED");
    return v != nullptr && v[0] == '0' ? 0 : 1;
  }();
  qr_panel_kernel<<<1, 1024, 0, st>>>(A, lda, m, c0, jb, P, V, T, tau, chunked);
}
void launch_set_identity(cplx* Y, long long ld, int m, int k, cudaStream_t st) {
  set_identity_kernel<<<blocks_for((long long)m * k), 256, 0, st>>>(Y, ld, m, k);
}
void launch_copy_matrix(const cplx* src, long long ld_s, cplx* dst, long long ld_d, int rows, int cols, int op,
                        cudaStream_t st) {
  copy_matrix_kernel<<<blocks_for((long long)rows * cols), 256, 0, st>>>(src, ld_s, dst, ld_d, rows, cols, op);
}
void launch_site_adjoint(const cplx* site, int chi, int dl, int dr, cplx* A, long long lda, cudaStream_t st) {
  site_adjoint_kernel<<<blocks_for((long long)dl * 2 * dr), 256, 0, st>>>(site, chi, dl, dr, A, lda);
}
void launch_site_from_adjoint(const cplx* Q, long long ldq, int k, int dr, cplx* site, int chi, cudaStream_t st) {
  site_from_adjoint_kernel<<<blocks_for((long long)k * 2 * dr), 256, 0, st>>>(Q, ldq, k, dr, site, chi);
}
void launch_sum_abs2(const cplx* A, long long lda, int rows, int cols, double* out, cudaStream_t st) {
  sum_abs2_kernel<<<1, 1024, 0, st>>>(A, lda, rows, cols, out);
}

}  // namespace mpsim_gpu
