// Cross Gram of two sets of 32 complex vectors on the FP64 tensor path:
// W = P^H Q (32 x 32) over rows [r0, r1), in the real-extended form
//   [Pr | Pi]^T [Qr | Qi] = [[Pr^T Qr, Pr^T Qi], [Pi^T Qr, Pi^T Qi]]  (64 x 64)
//   Re W = Pr^T Qr + Pi^T Qi,  Im W = Pr^T Qi - Pi^T Qr
// with the chunk pipeline of the Jacobi pair kernel (jacobi_split.cu): 32-row
// chunks as vector-major split Re/Im planes of pitch 36 (conflict-free DMMA
// fragments), double-buffered with 16-byte cp.async. Used by the QR trailing update
// (V^H A, qr_pre.cu) and the split epilogue (U^H X0 / X0^H X, split.cu).
// 256-thread CTAs.
#pragma once

#include "common.cuh"

namespace mpsim_gpu {
namespace pg {

constexpr int kC = 32;                 // rows per chunk
constexpr int kPitch = 36;             // doubles per smem row (== 4 mod 16)
constexpr int kPlane = kC * kPitch;    // doubles per plane
constexpr int kBuf = 4 * kPlane;       // [Pr | Pi | Qr | Qi]

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Operands are split-plane vectors (common.cuh): Re in doubles [0, m),
// Im in [m, 2 m) of each vector's slot. Per chunk and thread eight 16-byte
// copies (two rows of one plane of one vector): in copy s, warp w moves
// vector w + 8 (s & 3) of P (s < 4) or Q, lanes 0-15 its Re rows and lanes
// 16-31 its Im rows, 256 contiguous bytes each; shared planes are vector-major
// [vector][row] with pitch 36 (conflict-free DMMA fragments).
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

struct Loader {
  const double* src[8];  // this thread's plane of its 8 vectors, at its row pair
  int soff;
  // pvec(v) / qvec(v): vector v (0..31) of P / Q (any valid vector for padding
  // vectors whose results are discarded); pm / qm: their plane offsets (m_pad)
  template <class PF, class QF>
  __device__ __forceinline__ void init(PF pvec, QF qvec, long long pm, long long qm, int t) {
    const int lane = t & 31, warp = t >> 5;
    const int rp = lane & 15, plane = lane >> 4;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      src[s] = reinterpret_cast<const double*>(pvec(warp + 8 * s)) + plane * pm + 2 * rp;
      src[4 + s] = reinterpret_cast<const double*>(qvec(warp + 8 * s)) + plane * qm + 2 * rp;
    }
    soff = plane * kPlane + warp * kPitch + 2 * rp;
  }
  __device__ __forceinline__ void issue(double* buf, long long r0) const {
#pragma unroll
    for (int s = 0; s < 8; ++s) cp_async16(buf + (s >> 2) * 2 * kPlane + soff + 8 * (s & 3) * kPitch, src[s] + r0);
    commit();
  }
};

// W (complex, row pitch wld) = P^H Q over rows [r0, r1) (multiples of kC).
// buf: 2 x kBuf doubles; Wx: 64 x 65 doubles (may alias buf). All 256
// threads; ends with a barrier (W complete).
__device__ __forceinline__ void cross_gram(const Loader& ld, double (*buf)[kBuf], double* Wx, cplx* W, int wld,
                                           long long r0, long long r1, int t) {
  const int lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  // warp w: quadrant (x = w / 4: P Re/Im, y = (w / 2) & 1: Q Re/Im), tile rows
  // 2 (w & 1) + {0, 1}, all four tile columns
  const int qx = warp >> 2, qy = (warp >> 1) & 1, tr0 = 2 * (warp & 1);
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
  const int nchunks = (int)((r1 - r0) / kC);
  if (nchunks > 0) ld.issue(buf[0], r0);
  for (int k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) {
      ld.issue(buf[(k + 1) & 1], r0 + (k + 1) * kC);
      wait<1>();
    } else {
      wait<0>();
    }
    __syncthreads();
    const double* Pv = buf[k & 1] + qx * kPlane;
    const double* Pa = buf[k & 1] + (2 + qy) * kPlane;
#pragma unroll
    for (int ks = 0; ks < kC / 4; ++ks) {
      const int row = 4 * ks + fk;
      double av[2], bv[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = Pv[(8 * (tr0 + a) + fr) * kPitch + row];  // A[m = p idx][k = e]
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Pa[(8 * c + fr) * kPitch + row];          // B[k = e][n = q idx]
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) dmma(acc[a][c][0], acc[a][c][1], av[a], bv[c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int v = 0; v < 2; ++v) Wx[(qx * 32 + 8 * (tr0 + a) + fr) * 65 + qy * 32 + 8 * c + 2 * fk + v] = acc[a][c][v];
  __syncthreads();
  for (int idx = t; idx < 32 * 32; idx += 256) {
    const int i = idx / 32, j = idx % 32;
    const double re = Wx[i * 65 + j] + Wx[(32 + i) * 65 + 32 + j];
    const double im = Wx[i * 65 + 32 + j] - Wx[(32 + i) * 65 + j];
    W[i * wld + j] = make_double2(re, im);
  }
  __syncthreads();
}

}  // namespace pg
}  // namespace mpsim_gpu
