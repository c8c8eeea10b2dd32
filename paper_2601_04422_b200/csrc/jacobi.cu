// Batched block one-sided Jacobi SVD (the truncated-SVD step of
// apply_2q_local, svd.hpp:93-108, replacing Eigen::BDCSVD).
//
// X (m x n, vector-major) is orthogonalised in place: each sweep visits every
// pair of kW-vector blocks once, in a round-robin tournament so that the
// nb/2 pairs of a round are disjoint and run as independent CTAs (one launch
// per round covers every gate of the layer). A CTA
//   1. streams its 2W vectors through shared memory to form the Gram block
//      G = X_P^H X_P (2W x 2W),
//   2. skips the pair if every off-diagonal |G_ij| <= tol * sqrt(G_ii G_jj)
//      (the one-sided Jacobi convergence test, relative, so tiny columns are
//      judged against their own norm),
//   3. diagonalises G in shared memory with cyclic two-sided Jacobi (parallel
//      ordering, complex rotations, relative off-diagonal threshold; relatively
//      accurate for the well-scaled Gram blocks that occur near convergence),
//      sorting the eigenvectors by descending eigenvalue,
//   4. streams the vectors again and applies X_P <- X_P R.
// Exactly-zero off-diagonals are never rotated, so exactly-zero columns stay
// exactly zero and their singular values are exact zeros — what the cutoff-0
// trimming rule of svd.hpp:58 relies on (test_tensor.cpp:336-341).
#include "common.cuh"

namespace mpsim_gpu {

struct JacobiSmem {
  cplx T[kE * kPad];  // [e][vector] streaming tile
  cplx G[kP * kPad];  // Gram / EVD working matrix
  cplx R[kP * kPad];  // accumulated eigenvectors
  double cs[kP / 2], sn[kP / 2];
  cplx ph[kP / 2];
  int pp[kP / 2], pq[kP / 2];
  int perm[kP];
  int any;
};

__device__ __forceinline__ void pair_of(int step, int k, int M, int& a, int& b) {
  // Round-robin tournament over M+1 players (M odd); player M is fixed.
  if (k == 0) {
    a = step;
    b = M;
  } else {
    a = (step + k) % M;
    b = (step - k + M) % M;
  }
}

__global__ void __launch_bounds__(256, 2) jacobi_round_kernel(const GateDesc* __restrict__ gates,
                                                           cplx* __restrict__ ws,
                                                           const int* __restrict__ active,
                                                           int* __restrict__ rotated, int round,
                                                           double tol, double tol_in, int max_in,
                                                           const double* __restrict__ frob2,
                                                           double floor_rel2,
                                                           const int* __restrict__ perm,
                                                           long long perm_stride) {
  const int gi = blockIdx.y;
  if (!active[gi]) return;
  const GateDesc& g = gates[gi];
  const int nb = g.nb;
  if (round >= nb - 1 || (int)blockIdx.x >= nb / 2) return;
  int ba, bb;
  pair_of(round, blockIdx.x, nb - 1, ba, bb);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiSmem& S = *reinterpret_cast<JacobiSmem*>(smem_raw);
  const int t = threadIdx.x;
  const long long mp = g.m_pad;
  cplx* X = ws + g.ws_off;
  // Slot -> vector map of this sweep (de Rijk ordering: vectors sorted by
  // decreasing norm at the start of every sweep).
  const int* pm = perm + gi * perm_stride;
  auto vec = [&](int i) -> cplx* {
    const int slot = i < kW ? ba * kW + i : bb * kW + (i - kW);
    return X + (long long)pm[slot] * mp;
  };
#ifdef MPSIM_BOUNDS_CHECK
  if (threadIdx.x == 0 && ((long long)(bb > ba ? bb : ba) * kW + kW > g.n_pad || g.ws_off < 0)) {
    printf("jacobi OOB: gate %d ba %d bb %d nb %d n_pad %d ws_off %lld\n", gi, ba, bb, nb, g.n_pad, g.ws_off);
    asm volatile("trap;");
  }
#endif

  // ---- 1. Gram block
  // Split-K over 4 thread groups; each group of 64 threads holds the whole
  // 32x32 block as 4x4 register tiles (8 shared loads per 16 complex MACs).
  const int kg = t / 64, tg = t % 64, ti = tg / 8, tj = tg % 8;
  cplx acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
#pragma unroll
    for (int s = 0; s < (kP * kE) / 256; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      S.T[ee * kPad + vi] = vec(vi)[e0 + ee];
    }
    __syncthreads();
#pragma unroll 4
    for (int ee = kg; ee < kE; ee += 4) {
      const cplx* row = S.T + ee * kPad;
      cplx av[4], bv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) av[x] = row[ti + 8 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = row[tj + 8 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) cfmac(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();
  }
  // Reduce the four partial Gram blocks group by group.
  for (int grp = 0; grp < 4; ++grp) {
    if (kg == grp) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          cplx* gp = S.G + (ti + 8 * x) * kPad + tj + 8 * y;
          *gp = grp == 0 ? acc[x][y] : cadd(*gp, acc[x][y]);
        }
    }
    __syncthreads();
  }
  const int ip = t / 16, jp = t % 16;

  // ---- 2. convergence test on the true columns (tol scales with sqrt(m),
  // the dot-product rounding level, like LAPACK zgesvj's ctol = sqrt(m)).
  // Columns whose squared norm is below floor (~(64 eps)^2 ||X||_F^2) are
  // rounding noise of an (exactly) rank-deficient matrix: they are left out
  // of the test so noise cannot stall convergence. Their singular values are
  // below any cutoff the reference rule can resolve against ||theta||^2.
  // The rotation X_P R mixes 2W vectors, so orthogonality below ~eps*2W is not
  // reachable; the threshold is tol * max(sqrt(m), 2W).
  const double tolg = tol * fmax(sqrt((double)g.m), (double)kP);
  const double floor2 = floor_rel2 * frob2[gi];
  bool need = false;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int i = 2 * ip + a, j = 2 * jp + b;
      if (i < j) {
        const double gij = sqrt(cabs2(S.G[i * kPad + j]));
        const double gii = S.G[i * kPad + i].x, gjj = S.G[j * kPad + j].x;
        if (gij > 0.0 && gij > tolg * sqrt(gii * gjj) && fmin(gii, gjj) > floor2) need = true;
      }
    }
  if (!__syncthreads_or(need)) return;

  // ---- 3. EVD of the Gram block (cyclic Jacobi, parallel order)
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int i = 2 * ip + a, j = 2 * jp + b;
      S.R[i * kPad + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    }
  // Clean the diagonal to be exactly real.
  if (t < kP) S.G[t * kPad + t].y = 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < max_in; ++sweep) {
    if (t == 0) S.any = 0;
    __syncthreads();
    for (int step = 0; step < kP - 1; ++step) {
      if (t < kP / 2) {
        int p, q;
        pair_of(step, t, kP - 1, p, q);
        const double a = S.G[p * kPad + p].x, b = S.G[q * kPad + q].x;
        const cplx gpq = S.G[p * kPad + q];
        const double c = sqrt(cabs2(gpq));
        double cs = 1.0, sn = 0.0;
        cplx ph = make_double2(1.0, 0.0);
        if (c > 0.0 && c > tol_in * sqrt(fabs(a * b)) && fmin(a, b) > floor2) {
          ph = make_double2(gpq.x / c, -gpq.y / c);  // e^{-i phi}
          const double zeta = (b - a) / (2.0 * c);
          const double az = fabs(zeta);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) /
                            (az > 1e100 ? 2.0 * az : az + sqrt(1.0 + zeta * zeta));
          cs = 1.0 / sqrt(1.0 + tt * tt);
          sn = cs * tt;
          S.any = 1;
        }
        S.cs[t] = cs;
        S.sn[t] = sn;
        S.ph[t] = ph;
        S.pp[t] = p;
        S.pq[t] = q;
      }
      __syncthreads();
      // Column update B = G J and R <- R J: items (row i, pair k).
      // J = [[cs, sn], [-ph sn, ph cs]] on (p, q).
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int item = t + 256 * s;
        const int i = item / (kP / 2), k = item % (kP / 2);
        const double cs = S.cs[k], sn = S.sn[k];
        if (sn != 0.0) {
          const cplx ph = S.ph[k];
          const int p = S.pp[k], q = S.pq[k];
          const cplx phs = make_double2(ph.x * sn, ph.y * sn), phc = make_double2(ph.x * cs, ph.y * cs);
          {
            cplx* M = S.G + i * kPad;
            const cplx xp = M[p], xq = M[q];
            cplx np_ = make_double2(xp.x * cs, xp.y * cs), nq = make_double2(xp.x * sn, xp.y * sn);
            const cplx t1 = cmul(xq, phs), t2 = cmul(xq, phc);
            np_.x -= t1.x; np_.y -= t1.y;
            nq.x += t2.x; nq.y += t2.y;
            M[p] = np_;
            M[q] = nq;
          }
          {
            cplx* M = S.R + i * kPad;
            const cplx xp = M[p], xq = M[q];
            cplx np_ = make_double2(xp.x * cs, xp.y * cs), nq = make_double2(xp.x * sn, xp.y * sn);
            const cplx t1 = cmul(xq, phs), t2 = cmul(xq, phc);
            np_.x -= t1.x; np_.y -= t1.y;
            nq.x += t2.x; nq.y += t2.y;
            M[p] = np_;
            M[q] = nq;
          }
        }
      }
      __syncthreads();
      // Row update G <- J^H B: items (pair k, column j).
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int item = t + 256 * s;
        const int k = item / kP, j = item % kP;
        const double cs = S.cs[k], sn = S.sn[k];
        if (sn != 0.0) {
          const cplx phc_ = conjc(S.ph[k]);
          const int p = S.pp[k], q = S.pq[k];
          const cplx bp = S.G[p * kPad + j], bq = S.G[q * kPad + j];
          // new_p = cs bp - conj(ph) sn bq ; new_q = sn bp + conj(ph) cs bq
          const cplx t1 = cmul(bq, phc_);
          S.G[p * kPad + j] = make_double2(cs * bp.x - sn * t1.x, cs * bp.y - sn * t1.y);
          S.G[q * kPad + j] = make_double2(sn * bp.x + cs * t1.x, sn * bp.y + cs * t1.y);
        }
      }
      __syncthreads();
      if (t < kP / 2 && S.sn[t] != 0.0) {
        const int p = S.pp[t], q = S.pq[t];
        S.G[p * kPad + q] = make_double2(0.0, 0.0);
        S.G[q * kPad + p] = make_double2(0.0, 0.0);
        S.G[p * kPad + p].y = 0.0;
        S.G[q * kPad + q].y = 0.0;
      }
      __syncthreads();
    }
    // Every thread must read the flag before thread 0 clears it for the next
    // sweep, or the CTA would diverge at the barriers.
    const int any = S.any;
    __syncthreads();
    if (!any) break;
  }
  // The eigenvector order is NOT sorted: R stays a product of small-angle
  // (|t| <= 1) rotations, close to the identity near convergence. Sorting
  // would permute R and break the uniformly-bounded-cosine property that
  // block Jacobi needs to converge (observed: linear convergence and
  // restarts when sorted). Singular values are sorted once in the epilogue.
  if (t < kP) S.perm[t] = t;
  __syncthreads();

  // ---- 4. apply X_P <- X_P R
  const int jq = t % 16, eq = t / 16;
  const int j0 = S.perm[2 * jq], j1 = S.perm[2 * jq + 1];
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
#pragma unroll
    for (int s = 0; s < (kP * kE) / 256; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      S.T[ee * kPad + vi] = vec(vi)[e0 + ee];
    }
    __syncthreads();
    cplx o[4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a) o[a][0] = o[a][1] = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int i = 0; i < kP; ++i) {
      const cplx r0 = S.R[i * kPad + j0], r1 = S.R[i * kPad + j1];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const cplx x = S.T[(eq + 16 * a) * kPad + i];
        cfma(o[a][0], x, r0);
        cfma(o[a][1], x, r1);
      }
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      S.T[(eq + 16 * a) * kPad + 2 * jq] = o[a][0];
      S.T[(eq + 16 * a) * kPad + 2 * jq + 1] = o[a][1];
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < (kP * kE) / 256; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      vec(vi)[e0 + ee] = S.T[ee * kPad + vi];
    }
    __syncthreads();
  }
  if (t == 0) rotated[gi] = 1;
}

size_t jacobi_smem_bytes() { return sizeof(JacobiSmem); }

void jacobi_init() {
  cudaFuncSetAttribute(jacobi_round_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(JacobiSmem));
}

void launch_jacobi_round(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws,
                         const int* d_active, int* d_rotated, int round, double tol, double tol_in,
                         int max_in, const double* frob2, double floor_rel2, const int* perm,
                         long long perm_stride, double* /*maxoff: DMMA kernel only*/, cudaStream_t st) {
  jacobi_round_kernel<<<dim3(max_pairs, n_gates), 256, sizeof(JacobiSmem), st>>>(
      d_gates, ws, d_active, d_rotated, round, tol, tol_in, max_in, frob2, floor_rel2, perm, perm_stride);
}

// ---- de Rijk ordering: per gate, sort the n_pad vector slots by decreasing
// norm (zero padding last). One CTA per gate; n_pad <= 2048.
__global__ void __launch_bounds__(1024) derijk_kernel(const GateDesc* __restrict__ gates,
                                                      const cplx* __restrict__ ws, const int* __restrict__ active,
                                                      int* __restrict__ perm, long long perm_stride) {
  const int gi = blockIdx.x;
  const GateDesc& g = gates[gi];
  if (!active[gi]) return;
  __shared__ double key[2048];
  __shared__ int idx[2048];
  const int n2 = g.n_pad;  // multiple of 32; pad to a power of two below
  int p2 = 1;
  while (p2 < n2) p2 <<= 1;
  const cplx* X = ws + g.ws_off;
  // norms: one warp per vector
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int v = warp; v < p2; v += blockDim.x / 32) {
    double s = -1.0;
    if (v < g.n) {
      s = 0.0;
      const cplx* x = X + (long long)v * g.m_pad;
      for (int e = lane; e < g.m; e += 32) s += cabs2(x[e]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    } else if (v < n2) {
      s = -0.5;  // zero padding vectors: after every real vector
    }
    if (lane == 0) {
      key[v] = s;
      idx[v] = v;
    }
  }
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const double ki = key[i], kj = key[j];
          const int ii = idx[i], ij = idx[j];
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
  for (int i = threadIdx.x; i < n2; i += blockDim.x) perm[gi * perm_stride + i] = idx[i];
}

void launch_derijk(const GateDesc* d_gates, int n_gates, const cplx* ws, const int* d_active, int* perm,
                   long long perm_stride, cudaStream_t st) {
  derijk_kernel<<<n_gates, 1024, 0, st>>>(d_gates, ws, d_active, perm, perm_stride);
}

}  // namespace mpsim_gpu
