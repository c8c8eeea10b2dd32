// Batched block one-sided Jacobi SVD (the truncated-SVD step of
// apply_2q_local, svd.hpp:93-108, replacing Eigen::BDCSVD): the pair visits
// live in jacobi_split.cu (DMMA Gram, pair EVD (evd.cuh), DMMA rotation);
// this file holds the per-sweep de Rijk ordering. Exactly-zero
// off-diagonals are never rotated, so exactly-zero columns stay exactly zero
// and their singular values are exact zeros — what the cutoff-0 trimming rule
// of svd.hpp:58 relies on (test_tensor.cpp:336-341).
#include "common.cuh"

namespace mpsim_gpu {

// de Rijk ordering: per sweep, the vectors of every gate sorted by descending
// norm (one CTA per gate: warp-per-vector norms, bitonic sort in shared
// memory) -> the slot permutation the tournament runs over.
__global__ void __launch_bounds__(1024) derijk_kernel(const GateDesc* __restrict__ gates,
                                                      const cplx* __restrict__ ws, const int* __restrict__ active,
                                                      int* __restrict__ perm, long long perm_stride) {
  const int gi = blockIdx.x;
  const GateDesc& g = gates[gi];
  if (!active[gi]) return;
  const int n2 = g.n_pad;  // multiple of 32; pad to a power of two below
  int p2 = 1;
  while (p2 < n2) p2 <<= 1;
  extern __shared__ double sort_smem[];  // p2 keys then p2 indices (launch: the batch's largest p2)
  double* key = sort_smem;
  int* idx = reinterpret_cast<int*>(sort_smem + p2);
  const cplx* X = ws + g.ws_off;
  // norms: one warp per vector
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int v = warp; v < p2; v += blockDim.x / 32) {
    double s = -1.0;
    if (v < g.n) {
      s = 0.0;
      const cplx* x = X + (long long)v * g.m_pad;
      for (int e = lane; e < g.m; e += 32) s += cabs2(xs_get(x, g.m_pad, e));
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

// Sort capacity: one CTA holds a gate's keys in shared memory (12 bytes per
// vector): up to kMaxSortN = 16384 vectors, i.e. bond dimensions up to 8192.
void launch_derijk(const GateDesc* d_gates, int n_gates, const cplx* ws, const int* d_active, int* perm,
                   long long perm_stride, int max_n_pad, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(derijk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSortN * 12);
    init = true;
  }
  int p2 = 1;
  while (p2 < max_n_pad) p2 <<= 1;
  derijk_kernel<<<n_gates, 1024, (size_t)p2 * 12, st>>>(d_gates, ws, d_active, perm, perm_stride);
}

}  // namespace mpsim_gpu
