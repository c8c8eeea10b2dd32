// Block one-sided Jacobi round split into three launches, each shaped for its
// own bound (the fused jacobi_dmma.cu kernel serialises them inside one CTA,
// so a CTA's latency-bound EVD stalls the FP64 tensor pipe):
//   A  jacobi_gram_kernel  — DMMA Gram of every block pair of the round, the
//                            relative convergence test, G -> global (16 KB/pair)
//   B  jacobi_evd_kernel   — one cyclic complex Jacobi sweep of each 32x32 G
//                            that needs it, R -> global; small footprint, so
//                            many CTAs per SM overlap its barrier-bound steps
//   C  jacobi_rot_kernel   — X_P <- X_P R on DMMA, R_ext slice in registers,
//                            results stored straight to global
// Algorithm, tolerances and numerics are those of jacobi_dmma.cu.
#include "common.cuh"
#include "evd.cuh"

namespace mpsim_gpu {

namespace {

constexpr int kPitchS = 36;  // conflict-free DMMA fragment pitch (== 4 mod 16)

__device__ __forceinline__ void dmma_s(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct PairCtx {
  cplx* X;
  const int* pm;
  long long mp;
  int ba, bb;
  __device__ __forceinline__ cplx* vec(int i) const {
    const int slot = i < kW ? ba * kW + i : bb * kW + (i - kW);
    return X + (long long)pm[slot] * mp;
  }
};

// Returns false if this CTA has no pair in this round.
__device__ __forceinline__ bool pair_ctx(const GateDesc& g, int gi, int round, const int* active, cplx* ws,
                                         const int* perm, long long perm_stride, PairCtx& c) {
  if (!active[gi]) return false;
  const int nb = g.nb;
  if (round >= nb - 1 || (int)blockIdx.x >= nb / 2) return false;
  rr_pair(round, blockIdx.x, nb - 1, c.ba, c.bb);
  c.X = ws + g.ws_off;
  c.pm = perm + gi * perm_stride;
  c.mp = g.m_pad;
  return true;
}

__device__ __forceinline__ void load_chunk_planes(const PairCtx& c, int e0, double* Tr, double* Ti, int t) {
#pragma unroll
  for (int s = 0; s < (kP * kE) / 256; ++s) {
    const int idx = t + 256 * s;
    const int vi = idx / kE, ee = idx % kE;
    const cplx v = c.vec(vi)[e0 + ee];
    Tr[ee * kPitchS + vi] = v.x;
    Ti[ee * kPitchS + vi] = v.y;
  }
}

struct GramSmem {
  union {
    struct {
      double Tr[kE * kPitchS];
      double Ti[kE * kPitchS];
    } t;
    double Gx[64 * 65];
  } u;
  cplx G[kP * kPad];
};

}  // namespace

__global__ void __launch_bounds__(256, 3) jacobi_gram_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                             const int* __restrict__ active, int round, double tol,
                                                             const double* __restrict__ frob2, double floor_rel2,
                                                             const int* __restrict__ perm, long long perm_stride,
                                                             double* __restrict__ maxoff, int* __restrict__ need,
                                                             cplx* __restrict__ gbuf, int max_pairs) {
  const int gi = blockIdx.y;
  const GateDesc& g = gates[gi];
  PairCtx c;
  if (!pair_ctx(g, gi, round, active, ws, perm, perm_stride, c)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  GramSmem& S = *reinterpret_cast<GramSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  double* Tr = S.u.t.Tr;
  double* Ti = S.u.t.Ti;
  auto xext = [&](int e, int col) -> double { return (col < kP ? Tr : Ti)[e * kPitchS + (col & (kP - 1))]; };
  const int fr = lane / 4, fk = lane % 4;
  // tiles of G_ext = [[A, B], [B^T, D]]: upper A and D, all of B (see jacobi_dmma.cu)
  int trow[5], tcol[5], nt;
  if (warp < 4) {
    nt = 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      trow[i] = warp;
      tcol[i] = 4 + i;
    }
    trow[4] = tcol[4] = 0;
  } else {
    const int r = warp - 4, na = 4 - r;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
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
    load_chunk_planes(c, e0, Tr, Ti, t);
    __syncthreads();
#pragma unroll 4
    for (int ks = 0; ks < kE / 4; ++ks) {
      const int e = 4 * ks + fk;
      const double a_first = xext(e, 8 * trow[0] + fr), a_last = xext(e, 8 * trow[4] + fr);
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if (i < nt) dmma_s(acc[i][0], acc[i][1], trow[i] == trow[0] ? a_first : a_last, xext(e, 8 * tcol[i] + fr));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (i < nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) S.u.Gx[(8 * trow[i] + fr) * 65 + 8 * tcol[i] + fk * 2 + v] = acc[i][v];
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
  const double tolg = tol * fmax(sqrt((double)g.m), (double)kP);
  const double floor2 = floor_rel2 * frob2[gi];
  const bool nd = pair_needs_rotation(S.G, t, tolg, floor2, maxoff + gi);
  const long long slot = (long long)gi * max_pairs + blockIdx.x;
  if (t == 0) need[slot] = nd ? 1 : 0;
  if (!nd) return;
  cplx* gout = gbuf + slot * (kP * kP);
  for (int idx = t; idx < kP * kP; idx += 256) gout[idx] = S.G[(idx / kP) * kPad + idx % kP];
}

struct EvdSmem {
  cplx G[kP * kPad];
  cplx R[kP * kPad];
  EvdScratch sc;
};

__global__ void __launch_bounds__(256, 6) jacobi_evd_kernel(const GateDesc* __restrict__ gates,
                                                            const int* __restrict__ active, int round, double tol_in,
                                                            const double* __restrict__ frob2, double floor_rel2,
                                                            const int* __restrict__ need, const cplx* __restrict__ gbuf,
                                                            cplx* __restrict__ rbuf, int max_pairs) {
  const int gi = blockIdx.y;
  if (!active[gi]) return;
  const GateDesc& g = gates[gi];
  if (round >= g.nb - 1 || (int)blockIdx.x >= g.nb / 2) return;
  const long long slot = (long long)gi * max_pairs + blockIdx.x;
  if (!need[slot]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EvdSmem& S = *reinterpret_cast<EvdSmem*>(smem_raw);
  const int t = threadIdx.x;
  const cplx* gin = gbuf + slot * (kP * kP);
  for (int idx = t; idx < kP * kP; idx += 256) S.G[(idx / kP) * kPad + idx % kP] = gin[idx];
  __syncthreads();
  pair_evd_v1(S.G, S.R, S.sc, t, tol_in, floor_rel2 * frob2[gi], 1);
  __syncthreads();
  cplx* rout = rbuf + slot * (kP * kP);
  for (int idx = t; idx < kP * kP; idx += 256) rout[idx] = S.R[(idx / kP) * kPad + idx % kP];
}

struct RotSmem {
  double Tr[kE * kPitchS];
  double Ti[kE * kPitchS];
};

__global__ void __launch_bounds__(256, 2) jacobi_rot_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                            const int* __restrict__ active, int* __restrict__ rotated,
                                                            int round, const int* __restrict__ perm,
                                                            long long perm_stride, const int* __restrict__ need,
                                                            const cplx* __restrict__ rbuf, int max_pairs) {
  const int gi = blockIdx.y;
  const GateDesc& g = gates[gi];
  PairCtx c;
  if (!pair_ctx(g, gi, round, active, ws, perm, perm_stride, c)) return;
  const long long slot = (long long)gi * max_pairs + blockIdx.x;
  if (!need[slot]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RotSmem& S = *reinterpret_cast<RotSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  const int fr = lane / 4, fk = lane % 4;
  const cplx* R = rbuf + slot * (kP * kP);
  // warp: row tiles {2(w%4), +1}, complex column tiles {2(w/4), +1} (Re and Im)
  const int rbase = 2 * (warp % 4), cbase = 2 * (warp / 4);
  double bfrag[4][16];
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int cj = cbase + (ct & 1);
    const int jext = (ct < 2 ? 0 : kP) + 8 * cj + fr;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int cext = 4 * s + fk;
      const cplx r = R[(cext & (kP - 1)) * kP + (jext & (kP - 1))];
      double v;
      if (cext < kP) v = jext < kP ? r.x : r.y;
      else v = jext < kP ? -r.y : r.x;
      bfrag[ct][s] = v;
    }
  }
  double* Tr = S.Tr;
  double* Ti = S.Ti;
  for (int e0 = 0; e0 < g.m_pad; e0 += kE) {
    load_chunk_planes(c, e0, Tr, Ti, t);
    __syncthreads();
    double o[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) o[a][q][0] = o[a][q][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int cext = 4 * s + fk;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int e = 8 * (rbase + a) + fr;
        const double av = (cext < kP ? Tr : Ti)[e * kPitchS + (cext & (kP - 1))];
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma_s(o[a][q][0], o[a][q][1], av, bfrag[q][s]);
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int e = 8 * (rbase + a) + fr;
          const int j = 8 * (cbase + q) + 2 * fk + v;
          c.vec(j)[e0 + e] = make_double2(o[a][q][v], o[a][q + 2][v]);
        }
    __syncthreads();
  }
  if (t == 0) atomicAdd(rotated + gi, 1);
}

void jacobi_split_init() {
  cudaFuncSetAttribute(jacobi_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GramSmem));
  cudaFuncSetAttribute(jacobi_evd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EvdSmem));
  cudaFuncSetAttribute(jacobi_rot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RotSmem));
}

void launch_jacobi_round_split(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                               int* d_rotated, int round, double tol, double tol_in, const double* frob2,
                               double floor_rel2, const int* perm, long long perm_stride, double* maxoff, int* need,
                               cplx* gbuf, cplx* rbuf, cudaStream_t st) {
  const dim3 grid(max_pairs, n_gates);
  jacobi_gram_kernel<<<grid, 256, sizeof(GramSmem), st>>>(d_gates, ws, d_active, round, tol, frob2, floor_rel2, perm,
                                                           perm_stride, maxoff, need, gbuf, max_pairs);
  jacobi_evd_kernel<<<grid, 256, sizeof(EvdSmem), st>>>(d_gates, d_active, round, tol_in, frob2, floor_rel2, need,
                                                         gbuf, rbuf, max_pairs);
  jacobi_rot_kernel<<<grid, 256, sizeof(RotSmem), st>>>(d_gates, ws, d_active, d_rotated, round, perm, perm_stride,
                                                         need, rbuf, max_pairs);
}

}  // namespace mpsim_gpu
