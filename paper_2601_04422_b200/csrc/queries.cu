// Transfer-matrix query kernels: a general complex128 GEMM used for the
// environment recursions of norm / overlap / expectation values
// (mps.cpp:189-202, :223-239) and the statevector export (mps.cpp:241-256),
// plus a row-gathered GEMM step that advances the left environments of many
// bit strings at once (amplitude, mps.cpp:204-221, batched over strings).
#include <algorithm>

#include "common.cuh"

namespace mpsim_gpu {



constexpr int kGT = 64;  // tile
constexpr int kGK = 16;  // k chunk

// kSplit: blockIdx.z takes K range [z * kchunk, (z + 1) * kchunk) and writes
// its raw partial product to ws[z] (M x N, ld N); cgemm_splitk_reduce then
// sums the slices in z order (deterministic) and applies alpha / accumulate.
template <bool kSplit>
__global__ void __launch_bounds__(256) cgemm_kernel(GemmArgs a, cplx* __restrict__ ws, int kchunk) {
  __shared__ cplx As[kGK][kGT + 1];
  __shared__ cplx Bs[kGK][kGT + 1];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int i0 = blockIdx.y * kGT, j0 = blockIdx.x * kGT;
  cplx acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = make_double2(0.0, 0.0);
  const int kb = kSplit ? blockIdx.z * kchunk : 0;
  const int ke = kSplit ? min(a.K, kb + kchunk) : a.K;
  for (int k0 = kb; k0 < ke; k0 += kGK) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int idx = t + 256 * s;
      int i, k;
      if (a.opA == 0) {
        i = idx / kGK;
        k = idx % kGK;
      } else {
        k = idx / kGT;
        i = idx % kGT;
      }
      const int gi = i0 + i, gk = k0 + k;
      cplx v = make_double2(0.0, 0.0);
      if (gi < a.M && gk < ke) {
        if (a.opA == 0) {
          v = a.A[(long long)gi * a.lda + gk];
        } else {
          v = a.A[(long long)gk * a.lda + gi];
          v.y = -v.y;
        }
      }
      As[k][i] = v;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int idx = t + 256 * s;
      int j, k;
      if (a.opB == 0) {
        k = idx / kGT;
        j = idx % kGT;
      } else {
        j = idx / kGK;
        k = idx % kGK;
      }
      const int gj = j0 + j, gk = k0 + k;
      cplx v = make_double2(0.0, 0.0);
      if (gj < a.N && gk < ke) {
        if (a.opB == 0) {
          v = a.B[(long long)gk * a.ldb + gj];
        } else {
          v = a.B[(long long)gj * a.ldb + gk];
          v.y = -v.y;
        }
      }
      Bs[k][j] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kGK; ++k) {
      cplx av[4], bv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) av[x] = As[k][ty + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = Bs[k][tx + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) cfma(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int gi = i0 + ty + 16 * x, gj = j0 + tx + 16 * y;
      if (kSplit) {
        if (gi < a.M && gj < a.N) ws[((long long)blockIdx.z * a.M + gi) * a.N + gj] = acc[x][y];
      } else if (gi < a.M && gj < a.N) {
        cplx v = cmul(a.alpha, acc[x][y]);
        cplx* c = a.C + (long long)gi * a.ldc + gj;
        if (a.accumulate) v = cadd(v, *c);
        *c = v;
      }
    }
}

__global__ void cgemm_splitk_reduce(GemmArgs a, const cplx* __restrict__ ws, int slices) {
  const long long mn = (long long)a.M * a.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mn; e += (long long)gridDim.x * blockDim.x) {
    cplx sum = ws[e];
    for (int z = 1; z < slices; ++z) sum = cadd(sum, ws[z * mn + e]);
    const long long gi = e / a.N, gj = e % a.N;
    cplx v = cmul(a.alpha, sum);
    cplx* c = a.C + gi * a.ldc + gj;
    if (a.accumulate) v = cadd(v, *c);
    *c = v;
  }
}

void launch_cgemm(const GemmArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return;
  const dim3 g((a.N + kGT - 1) / kGT, (a.M + kGT - 1) / kGT);
  const int tiles = (int)(g.x * g.y);
  // Skinny products with a long K (the QR sweeps' V^H A2 / V^H Y panels,
  // 32 x n x m) fill a handful of SMs: split K so ~2 CTAs per SM run.
  int slices = 1;
  if (tiles < 74 && a.K >= 256) slices = std::min({a.K / 128, (2 * 148 + tiles - 1) / tiles, 16});
  if (slices <= 1) {
    cgemm_kernel<false><<<g, 256, 0, st>>>(a, nullptr, 0);
    return;
  }
  const int kchunk = ((a.K + slices - 1) / slices + kGK - 1) / kGK * kGK;
  slices = (a.K + kchunk - 1) / kchunk;
  cplx* ws = nullptr;
  const size_t bytes = sizeof(cplx) * (size_t)slices * a.M * a.N;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, st);
  if (e != cudaSuccess) {  // no workspace: the unsplit kernel
    (void)cudaGetLastError();
    cgemm_kernel<false><<<g, 256, 0, st>>>(a, nullptr, 0);
    return;
  }
  cgemm_kernel<true><<<dim3(g.x, g.y, slices), 256, 0, st>>>(a, ws, kchunk);
  const long long mn = (long long)a.M * a.N;
  cgemm_splitk_reduce<<<(unsigned)std::min<long long>((mn + 255) / 256, 4 * 148), 256, 0, st>>>(a, ws, slices);
  cudaFreeAsync(ws, st);
}

// env'[b][r] = sum_l env[b][l] * site[(l*2 + bit_b)*chi + r] for every string b.
__global__ void __launch_bounds__(256) amp_step_kernel(const cplx* __restrict__ env, long long ld_env,
                                                       cplx* __restrict__ out, long long ld_out,
                                                       const char* __restrict__ bits, int n_qubits, int site_idx,
                                                       int count, const cplx* __restrict__ site, int chi, int dl,
                                                       int dr) {
  __shared__ cplx Es[32][kGK + 1];
  __shared__ cplx S0[kGK][33], S1[kGK][33];
  __shared__ int bit[32];
  const int t = threadIdx.x, tx = t % 32, ty = t / 32;  // 8 rows of warps
  const int b0 = blockIdx.y * 32, r0 = blockIdx.x * 32;
  if (t < 32) bit[t] = (b0 + t < count) ? (bits[(long long)(b0 + t) * n_qubits + site_idx] == '1') : 0;
  cplx acc[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) acc[x] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int l0 = 0; l0 < dl; l0 += kGK) {
    for (int idx = t; idx < 32 * kGK; idx += 256) {
      const int b = idx / kGK, l = idx % kGK;
      Es[b][l] = (b0 + b < count && l0 + l < dl) ? env[(long long)(b0 + b) * ld_env + l0 + l] : make_double2(0.0, 0.0);
      const int l2 = idx / 32, r = idx % 32;
      const bool ok = (l0 + l2 < dl) && (r0 + r < dr);
      S0[l2][r] = ok ? site[(long long)((l0 + l2) * 2) * chi + r0 + r] : make_double2(0.0, 0.0);
      S1[l2][r] = ok ? site[(long long)((l0 + l2) * 2 + 1) * chi + r0 + r] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int l = 0; l < kGK; ++l) {
      const cplx s0 = S0[l][tx], s1 = S1[l][tx];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int b = ty + 8 * x;
        cfma(acc[x], Es[b][l], bit[b] ? s1 : s0);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int b = b0 + ty + 8 * x, r = r0 + tx;
    if (b < count && r < dr) out[(long long)b * ld_out + r] = acc[x];
  }
}

void launch_amp_step(const cplx* env, long long ld_env, cplx* out, long long ld_out, const char* bits,
                     int n_qubits, int site_idx, int count, const cplx* site, int chi, int dl, int dr,
                     cudaStream_t st) {
  amp_step_kernel<<<dim3((dr + 31) / 32, (count + 31) / 32), 256, 0, st>>>(
      env, ld_env, out, ld_out, bits, n_qubits, site_idx, count, site, chi, dl, dr);
}

__global__ void fill_kernel(cplx* p, long long n, cplx v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
void launch_fill(cplx* p, long long n, cplx v, cudaStream_t st) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, n, v);
}

}  // namespace mpsim_gpu
