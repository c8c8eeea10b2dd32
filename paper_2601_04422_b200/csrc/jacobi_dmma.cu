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

// (256, 2): 124 registers, no spills. (256, 3) fits 80 registers with spills
// and measured no faster at chi=512.
__global__ void __launch_bounds__(256, 2) jacobi_round_dmma_kernel(
    const GateDesc* __restrict__ gates, cplx* __restrict__ ws, const int* __restrict__ active,
    int* __restrict__ rotated, int round, double tol, double tol_in, int max_in, const double* __restrict__ frob2,
    double floor_rel2, const int* __restrict__ perm, long long perm_stride, double* __restrict__ maxoff) {
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
  // (Register double-buffering of the next chunk was measured: no gain at
  // chi=512, more spills; the chunk is loaded synchronously.)
  auto load_chunk = [&](int e0) {
#pragma unroll
    for (int s = 0; s < (kP * kE) / 256; ++s) {
      const int idx = t + 256 * s;
      const int vi = idx / kE, ee = idx % kE;
      const cplx v = vec(vi)[e0 + ee];
      Tr[ee * kPitch + vi] = v.x;
      Ti[ee * kPitch + vi] = v.y;
    }
  };

  // ---- 1. Gram on DMMA. Of the real 64x64 G_ext = [[A, B], [B^T, D]] only
  // the upper 8x8 tiles of A and D and all of B are needed (36 of 64 tiles):
  // Re G = A + D, Im G = B - B^T. Warps 0-3: tile row w of B (4 tiles);
  // warps 4-7: tile row r of A plus tile row 3-r of D (5 tiles).
  const int fr = lane / 4, fk = lane % 4;  // A-fragment row / B-fragment col, and k index
  int trow[5], tcol[5];
  int nt;
  if (warp < 4) {
    nt = 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      trow[i] = warp;
      tcol[i] = 4 + i;
    }
    trow[4] = tcol[4] = 0;
  } else {
    const int r = warp - 4;
    nt = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      // first 4 - r tiles: A row r, cols r..3 ; then r + 1 tiles: D row 3 - r, cols 3-r..3
      const int na = 4 - r;
      if (i < na) {
        trow[i] = r;
        tcol[i] = r + i;
      } else {
        trow[i] = 4 + (3 - r);
        tcol[i] = 4 + (3 - r) + (i - na);
      }
    }
    nt = 5;
  }
  double acc[5][2];
#pragma unroll
  for (int i = 0; i < 5; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
    load_chunk(e0);
    __syncthreads();
#pragma unroll 4
    for (int ks = 0; ks < kE / 4; ++ks) {
      const int e = 4 * ks + fk;
      double a_first = xext(e, 8 * trow[0] + fr), a_last = xext(e, 8 * trow[4] + fr);
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        if (i < nt) {
          const double av = trow[i] == trow[0] ? a_first : a_last;   // A[m = c][k = e] = X_ext[e][c]
          const double bv = xext(e, 8 * tcol[i] + fr);                 // B[k = e][n = c'] = X_ext[e][c']
          dmma(acc[i][0], acc[i][1], av, bv);
        }
      }
    }
    __syncthreads();
  }
  // scatter the computed tiles of G_ext (aliases the chunk planes), then combine
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (i < nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int row = 8 * trow[i] + fr, col = 8 * tcol[i] + fk * 2 + v;
        S.u.Gx[row * 65 + col] = acc[i][v];
      }
  __syncthreads();
  for (int idx = t; idx < kP * kP; idx += 256) {
    const int i = idx / kP, j = idx % kP;
    if (i > j) continue;
    const double* Gx = S.u.Gx;
    const double re = Gx[i * 65 + j] + Gx[(kP + i) * 65 + kP + j];
    const double im = Gx[i * 65 + kP + j] - Gx[j * 65 + kP + i];
    S.G[i * kPad + j] = make_double2(re, i == j ? 0.0 : im);
    if (i != j) S.G[j * kPad + i] = make_double2(re, -im);
  }
  __syncthreads();

  // ---- 2. convergence test, 3. pair EVD (shared with the SIMT kernel)
  const double tolg = tol * fmax(sqrt((double)g.m), (double)kP);
  const double floor2 = floor_rel2 * frob2[gi];
  if (!pair_needs_rotation(S.G, t, tolg, floor2, maxoff + gi)) return;
  // (16-thread parameters + fused block update, two barriers per step: the
  // one-barrier variant with per-thread redundant parameters, pair_evd(), was
  // measured 10 % slower at chi=512.)
  // max_in < 0: phase-timing probes only (-1: stop after the Gram/test, -2: after the EVD).
  if (max_in == -1) return;
  pair_evd_v1(S.G, S.R, S.sc, t, tol_in, floor2, max_in < 0 ? 1 : max_in);
  if (max_in == -2) return;

  // ---- 4. rotation on DMMA. Warp w computes row tiles {2(w%4), 2(w%4)+1} of
  // the chunk and complex column tiles {2(w/4), 2(w/4)+1}, i.e. the real column
  // tiles cj (Re) and 4+cj (Im) for both: 8 output tiles, R_ext slice for its 4
  // real column tiles held in registers (64 doubles), one A-fragment load per
  // 4 DMMAs. Each thread then owns Re and Im of the same complex outputs and
  // stores them straight to global (16-byte, 128-byte runs per 8 lanes).
  const int rbase = 2 * (warp % 4), cbase = 2 * (warp / 4);
  double bfrag[4][16];
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int cj = cbase + (ct & 1);                  // complex column tile
    const int jext = (ct < 2 ? 0 : kP) + 8 * cj + fr;  // Re tiles first, then Im tiles
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int cext = 4 * s + fk;  // B[k = c_ext][n = j_ext]
      const cplx r = S.R[(cext & (kP - 1)) * kPad + (jext & (kP - 1))];
      double v;
      if (cext < kP) v = jext < kP ? r.x : r.y;  // [[Re R, Im R],
      else v = jext < kP ? -r.y : r.x;           //  [-Im R, Re R]]
      bfrag[ct][s] = v;
    }
  }
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
    load_chunk(e0);
    __syncthreads();
    double o[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[a][c][0] = o[a][c][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const double av = xext(8 * (rbase + a) + fr, 4 * s + fk);  // A[m = e][k = c_ext]
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(o[a][c][0], o[a][c][1], av, bfrag[c][s]);
      }
    }
    // C fragment: row e = 8 rt + lane/4, column 2 (lane%4) + v of each tile.
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int e = 8 * (rbase + a) + fr;
          const int j = 8 * (cbase + c) + 2 * fk + v;  // complex column within the pair
          vec(j)[e0 + e] = make_double2(o[a][c][v], o[a][c + 2][v]);
        }
    __syncthreads();
  }
  if (t == 0) atomicAdd(rotated + gi, 1);  // rotated pair count of this gate, this sweep
}

size_t jacobi_dmma_smem_bytes() { return sizeof(JacobiDmmaSmem); }

void jacobi_dmma_init() {
  cudaFuncSetAttribute(jacobi_round_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(JacobiDmmaSmem));
}

void launch_jacobi_round_dmma(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                              int* d_rotated, int round, double tol, double tol_in, int max_in, const double* frob2,
                              double floor_rel2, const int* perm, long long perm_stride, double* maxoff,
                              cudaStream_t st) {
  jacobi_round_dmma_kernel<<<dim3(max_pairs, n_gates), 256, sizeof(JacobiDmmaSmem), st>>>(
      d_gates, ws, d_active, d_rotated, round, tol, tol_in, max_in, frob2, floor_rel2, perm, perm_stride, maxoff);
}

}  // namespace mpsim_gpu
