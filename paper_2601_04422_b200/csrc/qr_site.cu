// Householder QR of one tall site matrix for the centre moves (thin_qr,
// mps.cpp:57-65, in sweep_left_of / sweep_right_of, mps.cpp:69-95), shaped
// for latency: a centre move is a chain of site QRs where each site waits for
// the previous one's R, so nothing batches and the cost is the length of the
// dependent reflector chain (one per column).
//
//   site_panel_kernel   one CTA of 8 warps factors an 8-column panel; warp w
//                       holds column w in registers (32 rows per lane, m <=
//                       1024), so the column norm and every v^H x_c are warp
//                       reductions and a reflector costs one block barrier
//                       (publishing v); writes R, the explicit V and the
//                       compact-WY T (zlarft, Q_p = I - V T V^H).
//   site_update_kernel  A_b <- Q_p^H A_b (trailing columns) or Q_p A_b (Q
//                       formation, reflectors applied last to first), 8
//                       columns per CTA, rows streamed through shared memory.
// Look-ahead: the update of the next panel's own 8 columns runs first, so
// the next panel factors while the rest of the trailing matrix updates on a
// second stream; Q formation runs on that stream too (only R gates the next
// site). Any exact QR gives the same state; only k = min(m, n) is fixed by
// the reference (mps.cpp:57-65), and the reflector convention is zlarfg's.
#include <algorithm>
#include <cmath>
#include <string>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

namespace {

constexpr int kSW = 8;     // panel width (warps per panel CTA)
constexpr int kSL = 32;    // rows per lane: m <= 32 * 32 = 1024
constexpr int kUR = 64;    // rows per streamed chunk in the update

__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

struct PanelSmemS {
  cplx vs[kSW][kSL * 32];  // explicit reflectors, rows [c0, m) relative to c0
  cplx taus[kSW];
  cplx gv[kSW][kSW];       // v_i^H v_j (i < j) for zlarft
};

}  // namespace

// A: column-major complex (lda), rows [0, m). Factors columns [c0, c0 + jb)
// over rows [c0, m); R goes on and above the diagonal, the columns below it
// are left as zlarfg leaves them (unused). V (ldv, rows relative to c0,
// 8 columns, unit diagonal, zeros above and for columns >= jb) and T (8 x 8
// row-major, upper triangular) describe Q_p = I - V T V^H.
__global__ void __launch_bounds__(256, 1) site_panel_kernel(cplx* __restrict__ A, int lda, int m, int c0, int jb,
                                                            cplx* __restrict__ V, int ldv, cplx* __restrict__ T) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PanelSmemS& S = *reinterpret_cast<PanelSmemS*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int L = m - c0;  // rows in the panel
  cplx a[kSL];
  const cplx* col = A + (long long)(c0 + warp) * lda + c0;
#pragma unroll
  for (int s = 0; s < kSL; ++s) {
    const int r = lane + 32 * s;
    a[s] = (warp < jb && r < L) ? col[r] : make_double2(0.0, 0.0);
  }
  for (int j = 0; j < jb; ++j) {
    if (warp == j) {
      // zlarfg on rows >= j of this column (row j is lane j, slot 0: j < 8)
      double sn = 0.0;
#pragma unroll
      for (int s = 0; s < kSL; ++s) {
        const int r = lane + 32 * s;
        if (r > j && r < L) sn += cabs2(a[s]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sn += __shfl_xor_sync(0xffffffffu, sn, o);
      const cplx al = make_double2(__shfl_sync(0xffffffffu, a[0].x, j), __shfl_sync(0xffffffffu, a[0].y, j));
      cplx tau = make_double2(0.0, 0.0), inv = make_double2(0.0, 0.0);
      double beta = al.x;
      if (!(sn == 0.0 && al.y == 0.0)) {
        beta = -copysign(sqrt(cabs2(al) + sn), al.x);
        tau = make_double2((beta - al.x) / beta, -al.y / beta);
        const cplx d = make_double2(al.x - beta, al.y);
        const double dd = cabs2(d);
        inv = make_double2(d.x / dd, -d.y / dd);
      }
      const bool refl = tau.x != 0.0 || tau.y != 0.0;
#pragma unroll
      for (int s = 0; s < kSL; ++s) {
        const int r = lane + 32 * s;
        cplx v = make_double2(0.0, 0.0);
        if (r == j) {
          v = make_double2(1.0, 0.0);
          if (refl) a[s] = make_double2(beta, 0.0);
        } else if (r > j && r < L && refl) {
          v = cmul(a[s], inv);
          a[s] = v;
        }
        S.vs[j][r] = v;
      }
      if (lane == 0) S.taus[j] = tau;
    }
    __syncthreads();  // v_j and tau_j published
    const cplx tau = S.taus[j];
    if (warp > j && warp < jb && (tau.x != 0.0 || tau.y != 0.0)) {
      cplx d = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < kSL; ++s) {
        const int r = lane + 32 * s;
        if (r >= j && r < L) cfmac(d, S.vs[j][r], a[s]);
      }
      d = warp_sum(d);
      const cplx coef = cmul(make_double2(tau.x, -tau.y), d);  // H^H x = x - conj(tau) v (v^H x)
#pragma unroll
      for (int s = 0; s < kSL; ++s) {
        const int r = lane + 32 * s;
        if (r >= j && r < L) {
          const cplx u = cmul(S.vs[j][r], coef);
          a[s].x -= u.x;
          a[s].y -= u.y;
        }
      }
    } else if (warp < j) {
      cplx d = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < kSL; ++s) {
        const int r = lane + 32 * s;
        if (r >= j && r < L) cfmac(d, S.vs[warp][r], S.vs[j][r]);
      }
      d = warp_sum(d);
      if (lane == 0) S.gv[warp][j] = d;
    }
  }
  __syncthreads();
  // R (and the reflector storage below it) back to A; explicit V
  cplx* colw = A + (long long)(c0 + warp) * lda + c0;
#pragma unroll
  for (int s = 0; s < kSL; ++s) {
    const int r = lane + 32 * s;
    if (warp < jb && r < L) colw[r] = a[s];
  }
  for (int idx = t; idx < kSW * L; idx += 256) {
    const int jj = idx / L, r = idx % L;
    V[(long long)jj * ldv + r] = jj < jb ? S.vs[jj][r] : make_double2(0.0, 0.0);
  }
  if (warp == 0) {  // zlarft, forward columnwise: T[j][j] = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] gv[0:j, j]
    __shared__ cplx Ts[kSW][kSW];
    for (int j = 0; j < kSW; ++j) {
      cplx v = make_double2(0.0, 0.0);
      if (lane < j && j < jb) {
        for (int q = lane; q < j; ++q) cfma(v, Ts[lane][q], S.gv[q][j]);
        const cplx tj = S.taus[j];
        v = make_double2(-(tj.x * v.x - tj.y * v.y), -(tj.x * v.y + tj.y * v.x));
      } else if (lane == j && j < jb) {
        v = S.taus[j];
      }
      if (lane < kSW) Ts[lane][j] = (lane <= j && j < jb) ? v : make_double2(0.0, 0.0);
      __syncwarp();
    }
    if (lane < kSW)
      for (int j = 0; j < kSW; ++j) T[lane * kSW + j] = Ts[lane][j];
  }
}

// A_b <- (I - V op(T) V^H) A_b for columns [cb, cb + 8) of the CTA, rows
// [c0, m): adjoint = 1 uses T^H (Q_p^H, the trailing update), 0 uses T
// (Q_p, Q formation). Columns [col0, col1) are updated, 8 per CTA.
__global__ void __launch_bounds__(256) site_update_kernel(cplx* __restrict__ A, int lda, int m, int c0, int col0,
                                                          int col1, const cplx* __restrict__ V, int ldv,
                                                          const cplx* __restrict__ T, int adjoint) {
  const int cb = col0 + kSW * blockIdx.x;
  if (cb >= col1) return;
  const int nc = min(kSW, col1 - cb);
  const int L = m - c0;
  __shared__ cplx Vc[kUR][kSW + 1];
  __shared__ cplx Ac[kUR][kSW + 1];
  __shared__ cplx W[4][kSW][kSW];  // partial V^H A per row quarter
  __shared__ cplx W2[kSW][kSW];
  const int t = threadIdx.x;
  // pass 1: W = V^H A_b, thread (i, c, quarter q) sums rows q, q + 4, ... of each chunk
  const int q = t >> 6, ic = t & 63, i = ic >> 3, c = ic & 7;
  cplx w = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < L; r0 += kUR) {
    for (int idx = t; idx < kUR * kSW; idx += 256) {
      const int rr = idx / kSW, cc = idx % kSW, r = r0 + rr;
      Vc[rr][cc] = r < L ? V[(long long)cc * ldv + r] : make_double2(0.0, 0.0);
      Ac[rr][cc] = (r < L && cc < nc) ? A[(long long)(cb + cc) * lda + c0 + r] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = q; rr < kUR; rr += 4) cfmac(w, Vc[rr][i], Ac[rr][c]);
    __syncthreads();
  }
  W[q][i][c] = w;
  __syncthreads();
  if (t < 64) {  // W2 = op(T) W, with the quarters summed in order (deterministic)
    cplx acc = make_double2(0.0, 0.0);
    for (int k = 0; k < kSW; ++k) {
      const cplx wk = cadd(cadd(W[0][k][c], W[1][k][c]), cadd(W[2][k][c], W[3][k][c]));
      const cplx tk = adjoint ? conjc(T[k * kSW + i]) : T[i * kSW + k];
      cfma(acc, tk, wk);
    }
    W2[i][c] = acc;
  }
  __syncthreads();
  // pass 2: A_b -= V W2
  for (int r0 = 0; r0 < L; r0 += kUR) {
    for (int idx = t; idx < kUR * kSW; idx += 256) {
      const int rr = idx / kSW, cc = idx % kSW, r = r0 + rr;
      Vc[rr][cc] = r < L ? V[(long long)cc * ldv + r] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int idx = t; idx < kUR * kSW; idx += 256) {
      const int rr = idx / kSW, cc = idx % kSW, r = r0 + rr;
      if (r < L && cc < nc) {
        cplx* p = A + (long long)(cb + cc) * lda + c0 + r;
        cplx v = *p;
#pragma unroll
        for (int k = 0; k < kSW; ++k) {
          const cplx u = cmul(Vc[rr][k], W2[k][cc]);
          v.x -= u.x;
          v.y -= u.y;
        }
        *p = v;
      }
    }
    __syncthreads();
  }
}

// left (right = 0): A_c[r] = site[r chi + c] (r < 2 dl, c < dr); right:
// A_l[e] = conj(site[(l 2 + p) chi + r]), e = p dr + r. Column-major, lda.
__global__ void site_matrix_kernel(const cplx* __restrict__ site, int chi, int dl, int dr, int right,
                                   cplx* __restrict__ A, int lda) {
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * m;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / m), r = (int)(i % m);
    cplx v;
    if (!right) {
      v = site[(long long)r * chi + c];
    } else {
      const int p = r / dr, rr = r % dr;
      v = site[(long long)(c * 2 + p) * chi + rr];
      v.y = -v.y;
    }
    A[(long long)c * lda + r] = v;
  }
}

// R (k x n, row-major) from the factored A; Q (m x k, column-major, ldq) = [I_k; 0]
__global__ void site_r_and_identity_kernel(const cplx* __restrict__ A, int lda, int m, int n, int k,
                                           cplx* __restrict__ R, cplx* __restrict__ Q, int ldq) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * n;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / n), c = (int)(i % n);
    R[i] = j <= c ? A[(long long)c * lda + j] : make_double2(0.0, 0.0);
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * m;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / m), r = (int)(i % m);
    Q[(long long)c * ldq + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
}

// site <- Q (left: site[r chi + j], r < 2 dl) or Q^H (right: site[(j 2 + p) chi
// + r] = conj(Q[j][p dr + r])), j < k
__global__ void site_from_q_kernel(const cplx* __restrict__ Q, int ldq, int k, int dl, int dr, int right,
                                   cplx* __restrict__ site, int chi) {
  const int m = right ? 2 * dr : 2 * dl;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)k * m;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / m), r = (int)(i % m);
    cplx v = Q[(long long)j * ldq + r];
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
unsigned grid_of(long long n) { return (unsigned)std::max(1LL, std::min((n + 255) / 256, 8LL * 148)); }
#define CKQ(x)                                                                             \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
}  // namespace

bool site_qr_supported(int m, int n) { return m >= n && m <= kSL * 32 && n >= 16; }

// QR of the site's matricisation (left: (2 Dl x Dr); right: (Dl x 2 Dr)^H):
// R (k x n, row-major) into R, Q (or Q^H) written into the site. Work
// buffers grow as needed. Launched on s.st (panels, look-ahead updates) and
// aux (trailing updates, Q formation); on return aux has been joined back
// into s.st.
int site_qr(State& s, cplx* site, int dl, int dr, int right, DeviceBuf& Abuf, DeviceBuf& Vbuf, DeviceBuf& Tbuf,
            DeviceBuf& Qbuf, cplx* R, cudaStream_t aux, cudaEvent_t* evs) {
  static bool init = false;
  if (!init) {
    CKQ(cudaFuncSetAttribute(site_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(PanelSmemS)));
    init = true;
  }
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr, k = std::min(m, n);
  const int lda = (m + 31) / 32 * 32;
  const int np = (k + kSW - 1) / kSW;
  Abuf.ensure(sizeof(cplx) * (size_t)lda * n);
  Vbuf.ensure(sizeof(cplx) * (size_t)np * kSW * lda);
  Tbuf.ensure(sizeof(cplx) * (size_t)np * kSW * kSW);
  Qbuf.ensure(sizeof(cplx) * (size_t)lda * k);
  cplx* A = (cplx*)Abuf.p;
  cplx* Vall = (cplx*)Vbuf.p;
  cplx* Tall = (cplx*)Tbuf.p;
  cplx* Q = (cplx*)Qbuf.p;
  cudaStream_t st = s.st;
  site_matrix_kernel<<<grid_of((long long)n * m), 256, 0, st>>>(site, s.chi, dl, dr, right, A, lda);
  ++s.launches;
  // Panel p runs on st concurrently with the trailing update of panel p - 1
  // beyond panel p's columns (aux). Panel p's own columns were updated on st
  // (look-ahead) after st waited for aux: Householder updates of a column
  // apply in panel order.
  auto join = [&](cudaStream_t from, cudaStream_t to, cudaEvent_t e) {
    CKQ(cudaEventRecord(e, from));
    CKQ(cudaStreamWaitEvent(to, e, 0));
  };
  for (int p = 0; p < np; ++p) {
    const int c0 = p * kSW, jb = std::min(kSW, k - c0);
    cplx* V = Vall + (long long)p * kSW * lda;
    cplx* T = Tall + (long long)p * kSW * kSW;
    site_panel_kernel<<<1, 256, sizeof(PanelSmemS), st>>>(A, lda, m, c0, jb, V, lda, T);
    ++s.launches;
    const int c1 = c0 + kSW;
    if (c1 >= n) continue;
    const int la = std::min(n, c1 + kSW);
    if (la < n) join(st, aux, evs[0]);  // aux: the rest of panel p's update needs V_p, T_p
    join(aux, st, evs[1]);              // st: panel p - 1's aux update reached these columns first
    site_update_kernel<<<1, 256, 0, st>>>(A, lda, m, c0, c1, la, V, lda, T, 1);
    ++s.launches;
    if (la < n) {
      site_update_kernel<<<(n - la + kSW - 1) / kSW, 256, 0, aux>>>(A, lda, m, c0, la, n, V, lda, T, 1);
      ++s.launches;
    }
  }
  join(aux, st, evs[1]);  // the factorisation is complete on st
  site_r_and_identity_kernel<<<grid_of((long long)k * std::max(n, m)), 256, 0, st>>>(A, lda, m, n, k, R, Q, lda);
  ++s.launches;
  // Q = H_0 ... H_{np-1} [I; 0], last reflector block first (columns >= c0)
  for (int p = np - 1; p >= 0; --p) {
    const int c0 = p * kSW;
    site_update_kernel<<<(k - c0 + kSW - 1) / kSW, 256, 0, st>>>(Q, lda, m, c0, c0, k,
                                                                 Vall + (long long)p * kSW * lda, lda,
                                                                 Tall + (long long)p * kSW * kSW, 0);
    ++s.launches;
  }
  site_from_q_kernel<<<grid_of((long long)k * m), 256, 0, st>>>(Q, lda, k, dl, dr, right, site, s.chi);
  ++s.launches;
  return k;
}

}  // namespace mpsim_gpu
