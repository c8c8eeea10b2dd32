// Batched theta contraction: merge the two sites of every gate in a layer and
// mix in the 4x4 gate, writing the Jacobi operand X (and its pristine copy X0).
//
// Reference: apply_2q_local, gate_apply.cpp:121-131 —
//   merged = contract(A_q, A_{q+1}, {{2,0}})          (tensor.hpp:269-331, GEMM)
//   applied = contract(merged, gate, {{1,2},{2,3}})   (4x4 mix)
//   ordered = permute(applied, {0,2,3,1})             -> theta[(l,p0'),(p1',r)]
// Here the three steps are one kernel: each CTA owns a 32(l) x 32(r) tile for
// all four (p0,p1) physical combinations, so the gate mix is a register-level
// epilogue of the merge GEMM and theta is never materialised in site order.
#include "common.cuh"

namespace mpsim_gpu {

constexpr int kTL = 32;  // l per tile
constexpr int kTR = 32;  // r per tile
constexpr int kTK = 8;   // contraction chunk

__global__ void __launch_bounds__(256) theta_kernel(const GateDesc* __restrict__ gates,
                                                    const cplx* __restrict__ sites,
                                                    long long site_stride, int chi,
                                                    cplx* __restrict__ ws,
                                                    double* __restrict__ frob2) {
  const GateDesc& g = gates[blockIdx.y];
  const int tiles_r = (g.dr + kTR - 1) / kTR;
  const int tiles_l = (g.dl + kTL - 1) / kTL;
  const int tl = blockIdx.x / tiles_r, tr = blockIdx.x % tiles_r;
  if (tl >= tiles_l) return;
  const int l0 = tl * kTL, r0 = tr * kTR;
  const int dl = g.dl, dm = g.dm, dr = g.dr;

  __shared__ cplx As[2 * kTL][kTK + 1];  // rows (l,p0)
  __shared__ cplx Bs[kTK][2 * kTR];      // cols (p1,r)
  __shared__ cplx U[16];

  const cplx* A = sites + (long long)g.q * site_stride;
  const cplx* B = sites + (long long)(g.q + 1) * site_stride;
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  if (t < 16) U[t] = g.u[t];

  cplx acc[2][2][2][2];  // [l-sub][r-sub][p0][p1]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int d = 0; d < 2; ++d) acc[a][b][c][d] = make_double2(0.0, 0.0);

  for (int m0 = 0; m0 < dm; m0 += kTK) {
    // A tile: 64 rows x 8 k; thread loads 2.
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int idx = t * 2 + s;
      const int i = idx / kTK, kk = idx % kTK;
      const int l = l0 + i / 2, m = m0 + kk;
      As[i][kk] = (l < dl && m < dm) ? A[(long long)(2 * l0 + i) * chi + m] : make_double2(0.0, 0.0);
    }
    // B tile: 8 k x 64 cols; thread loads 2.
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int idx = t * 2 + s;
      const int kk = idx / (2 * kTR), jj = idx % (2 * kTR);
      const int p1 = jj / kTR, r = r0 + jj % kTR, m = m0 + kk;
      Bs[kk][jj] = (m < dm && r < dr) ? B[(long long)(m * 2 + p1) * chi + r] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      cplx a[2][2], b[2][2];
#pragma unroll
      for (int ls = 0; ls < 2; ++ls)
#pragma unroll
        for (int p0 = 0; p0 < 2; ++p0) a[ls][p0] = As[2 * (ty + 16 * ls) + p0][kk];
#pragma unroll
      for (int rs = 0; rs < 2; ++rs)
#pragma unroll
        for (int p1 = 0; p1 < 2; ++p1) b[rs][p1] = Bs[kk][p1 * kTR + tx + 16 * rs];
#pragma unroll
      for (int ls = 0; ls < 2; ++ls)
#pragma unroll
        for (int rs = 0; rs < 2; ++rs)
#pragma unroll
          for (int p0 = 0; p0 < 2; ++p0)
#pragma unroll
            for (int p1 = 0; p1 < 2; ++p1) cfma(acc[ls][rs][p0][p1], a[ls][p0], b[rs][p1]);
    }
    __syncthreads();
  }

  // Jacobi operand X (or, preconditioned, the QR operand) in orientation
  // trans; X0 in the orientation of the factor formula f (common.cuh).
  cplx* X = ws + (g.pre ? g.qr_off : g.ws_off);
  const long long ldx = g.pre ? g.qr_m_pad : g.m_pad;
  cplx* X0 = ws + g.x0_off;
  double f2 = 0.0;  // this CTA's share of ||theta||_F^2 (Jacobi noise floor)
#pragma unroll
  for (int ls = 0; ls < 2; ++ls)
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
      const int l = l0 + ty + 16 * ls, r = r0 + tx + 16 * rs;
      if (l >= dl || r >= dr) continue;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        // theta'[p0',p1'] = sum_{p0,p1} u[2p0'+p1', 2p0+p1] T[p0][p1]  (gate_apply.cpp:127-128)
        cplx v = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 4; ++i) cfma(v, acc[ls][rs][i >> 1][i & 1], U[o * 4 + i]);
        const int p0o = o >> 1, p1o = o & 1;
        const long long row = l * 2 + p0o, col = p1o * dr + r;  // theta (2Dl x 2Dr)
        const cplx vc = make_double2(v.x, -v.y);
        if (g.trans == 0) X[col * ldx + row] = v;
        else X[row * ldx + col] = vc;
        if (g.f == 0) X0[col * g.x0_ld + row] = v;
        else X0[row * g.x0_ld + col] = vc;
        f2 += cabs2(v);
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, o);
  __shared__ double red[8];
  if (t % 32 == 0) red[t / 32] = f2;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[i];
    atomicAdd(frob2 + blockIdx.y, s);
  }
}

void launch_theta(const GateDesc* d_gates, int n_gates, int max_tiles, const cplx* sites,
                  long long site_stride, int chi, cplx* ws, double* frob2, cudaStream_t st) {
  if (n_gates == 0) return;
  theta_kernel<<<dim3(max_tiles, n_gates), 256, 0, st>>>(d_gates, sites, site_stride, chi, ws, frob2);
}

int theta_tiles(int dl, int dr) { return ((dl + kTL - 1) / kTL) * ((dr + kTR - 1) / kTR); }

}  // namespace mpsim_gpu
