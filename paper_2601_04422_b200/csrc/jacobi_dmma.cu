// Block one-sided Jacobi round on the FP64 tensor path (DMMA): same algorithm
// as jacobi_round_kernel (jacobi.cu), with the two streaming GEMMs of a pair
// visit on mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) instead of DFMA:
//   Gram      G_ext = X_ext^T X_ext   (64 x 64 real, X_ext = [Re X_P | Im X_P])
//             -> G = (A + D) + i (B - C) over its 32x32 quadrants
//   rotation  X_ext <- X_ext R_ext, R_ext = [[Re R, Im R], [-Im R, Re R]]
// The pair block streams through shared memory as split real/imaginary
// planes with a 36-double row pitch, which makes every DMMA fragment load
// (A: row = lane/4, col = lane%4; B: row = lane%4, col = lane/4) bank-conflict
// free. Each warp keeps its slice of R_ext in registers for the whole visit.
#include "common.cuh"
#include "evd.cuh"

namespace mpsim_gpu {

constexpr int kPitch = 36;  // doubles per smem row (== 4 mod 16: conflict-free fragments)

struct JacobiDmmaSmem {
  union {
    struct {
      double Tr[kE * kPitch];
      double Ti[kE * kPitch];
    } t;
    double Gx[64 * 65];  // real 64x64 Gram (after the chunk loop)
  } u;
  cplx G[kP * kPad];
  cplx R[kP * kPad];
  EvdScratch sc;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256, 2) jacobi_round_dmma_kernel(
    const GateDesc* __restrict__ gates, cplx* __restrict__ ws, const int* __restrict__ active,
    int* __restrict__ rotated, int round, double tol, double tol_in, int max_in, const double* __restrict__ frob2,
    double floor_rel2, const int* __restrict__ perm, long long perm_stride) {
  const int gi = blockIdx.y;
  if (!active[gi]) return;
  const GateDesc& g = gates[gi];
  const int nb = g.nb;
  if (round >= nb - 1 || (int)blockIdx.x >= nb / 2) return;
  int ba, bb;
  rr_pair(round, blockIdx.x, nb - 1, ba, bb);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacobiDmmaSmem& S = *reinterpret_cast<JacobiDmmaSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  const long long mp = g.m_pad;
  cplx* X = ws + g.ws_off;
  const int* pm = perm + gi * perm_stride;
  auto vec = [&](int i) -> cplx* {
    const int slot = i < kW ? ba * kW + i : bb * kW + (i - kW);
    return X + (long long)pm[slot] * mp;
  };
  double* Tr = S.u.t.Tr;
  double* Ti = S.u.t.Ti;
  // X_ext[e][c]: c < 32 -> Re, c >= 32 -> Im of vector c % 32
  auto xext = [&](int e, int c) -> double { return (c < kP ? Tr : Ti)[e * kPitch + (c & (kP - 1))]; };
  // Register double-buffering: the next chunk's global loads are issued
  // before the current chunk's DMMA work, so their latency overlaps compute.
  constexpr int kPer = (kP * kE) / 256;
  cplx pre[kPer];
  auto fetch = [&](int e0) {
#pragma unroll
    for (int s = 0; s < kPer; ++s) pre[s] = vec((t + 256 * s) / kE)[e0 + (t + 256 * s) % kE];
  };
  auto stage = [&]() {
#pragma unroll
    for (int s = 0; s < kPer; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      Tr[ee * kPitch + vi] = pre[s].x;
      Ti[ee * kPitch + vi] = pre[s].y;
    }
  };

  // ---- 1. Gram on DMMA: warp tile = rows [16*(warp/2), +16) x cols [32*(warp%2), +32) of G_ext
  const int r0 = 16 * (warp / 2), c0 = 32 * (warp % 2);
  const int fr = lane / 4, fk = lane % 4;  // A-fragment row / B-fragment col, and k index
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  fetch(0);
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
    stage();
    __syncthreads();
    if (e0 + kE < g.m_pad) fetch(e0 + kE);
#pragma unroll 4
    for (int ks = 0; ks < kE / 4; ++ks) {
      const int e = 4 * ks + fk;
      double av[2], bv[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = xext(e, r0 + 8 * a + fr);  // A[m = c][k = e] = X_ext[e][c]
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = xext(e, c0 + 8 * b + fr);  // B[k = e][n = c'] = X_ext[e][c']
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
    __syncthreads();
  }
  // scatter the real 64x64 Gram (aliases the chunk planes), then combine
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = r0 + 8 * a + fr, col = c0 + 8 * b + fk * 2 + v;
        S.u.Gx[row * 65 + col] = acc[a][b][v];
      }
  __syncthreads();
  for (int idx = t; idx < kP * kP; idx += 256) {
    const int i = idx / kP, j = idx % kP;
    const double* Gx = S.u.Gx;
    S.G[i * kPad + j] = make_double2(Gx[i * 65 + j] + Gx[(kP + i) * 65 + kP + j],
                                     Gx[i * 65 + kP + j] - Gx[(kP + i) * 65 + j]);
  }
  __syncthreads();

  // ---- 2. convergence test, 3. pair EVD (shared with the SIMT kernel)
  const double tolg = tol * fmax(sqrt((double)g.m), (double)kP);
  const double floor2 = floor_rel2 * frob2[gi];
  if (!pair_needs_rotation(S.G, t, tolg, floor2)) return;
  pair_evd(S.G, S.R, S.sc, t, tol_in, floor2, max_in);

  // ---- 4. rotation on DMMA: warp owns output column tile [8*warp, +8) of X_ext R_ext
  double bfrag[16];
  {
    const int jext = 8 * warp + fr;  // B[k = c_ext][n = j_ext]: n = lane / 4
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int cext = 4 * s + fk;
      const int c = cext & (kP - 1), j = jext & (kP - 1);
      const cplx r = S.R[c * kPad + j];
      double v;
      if (cext < kP) v = jext < kP ? r.x : r.y;   // [[Re R, Im R],
      else v = jext < kP ? -r.y : r.x;            //  [-Im R, Re R]]
      bfrag[s] = v;
    }
  }
  fetch(0);
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
    stage();
    __syncthreads();
    if (e0 + kE < g.m_pad) fetch(e0 + kE);
    double o[kE / 8][2];
#pragma unroll
    for (int rt = 0; rt < kE / 8; ++rt) o[rt][0] = o[rt][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
#pragma unroll
      for (int rt = 0; rt < kE / 8; ++rt) {
        const double av = xext(8 * rt + fr, 4 * s + fk);  // A[m = e][k = c_ext]
        dmma(o[rt][0], o[rt][1], av, bfrag[s]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int rt = 0; rt < kE / 8; ++rt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = 8 * rt + fr, jext = 8 * warp + 2 * fk + v;
        (jext < kP ? Tr : Ti)[e * kPitch + (jext & (kP - 1))] = o[rt][v];
      }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < (kP * kE) / 256; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      vec(vi)[e0 + ee] = make_double2(Tr[ee * kPitch + vi], Ti[ee * kPitch + vi]);
    }
    __syncthreads();
  }
  if (t == 0) rotated[gi] = 1;
}

size_t jacobi_dmma_smem_bytes() { return sizeof(JacobiDmmaSmem); }

void jacobi_dmma_init() {
  cudaFuncSetAttribute(jacobi_round_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(JacobiDmmaSmem));
}

void launch_jacobi_round_dmma(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                              int* d_rotated, int round, double tol, double tol_in, int max_in, const double* frob2,
                              double floor_rel2, const int* perm, long long perm_stride, cudaStream_t st) {
  jacobi_round_dmma_kernel<<<dim3(max_pairs, n_gates), 256, sizeof(JacobiDmmaSmem), st>>>(
      d_gates, ws, d_active, d_rotated, round, tol, tol_in, max_in, frob2, floor_rel2, perm, perm_stride);
}

}  // namespace mpsim_gpu
