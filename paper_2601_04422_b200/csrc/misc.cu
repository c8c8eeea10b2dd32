// Single-qubit gates and site-store maintenance kernels.
#include "common.cuh"

namespace mpsim_gpu {

// apply_1q (gate_apply.cpp:99-110): A'[l,p',r] = sum_p u[p',p] A[l,p,r],
// batched over every one-qubit gate of a layer. HBM-bound: each (l, r) reads
// and writes two complex values.
__global__ void __launch_bounds__(256) apply1q_kernel(const Gate1Desc* __restrict__ gates,
                                                      cplx* __restrict__ sites, long long site_stride,
                                                      int chi) {
  const Gate1Desc& g = gates[blockIdx.y];
  const long long total = (long long)g.dl * g.dr;
  cplx* s = sites + (long long)g.q * site_stride;
  const cplx u00 = g.u[0], u01 = g.u[1], u10 = g.u[2], u11 = g.u[3];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(i / g.dr), r = (int)(i % g.dr);
    cplx* a0p = s + (long long)(l * 2) * chi + r;
    cplx* a1p = a0p + chi;
    const cplx a0 = *a0p, a1 = *a1p;
    cplx n0 = cmul(u00, a0), n1 = cmul(u10, a0);
    cfma(n0, u01, a1);
    cfma(n1, u11, a1);
    *a0p = n0;
    *a1p = n1;
  }
}

void launch_apply1q(const Gate1Desc* d_gates, int n_gates, long long max_elems, cplx* sites,
                    long long site_stride, int chi, cudaStream_t st) {
  if (n_gates == 0) return;
  long long blocks = (max_elems + 255) / 256;
  if (blocks > 1184) blocks = 1184;  // 8 CTAs x 148 SMs, grid-stride beyond
  if (blocks < 1) blocks = 1;
  apply1q_kernel<<<dim3((unsigned)blocks, n_gates), 256, 0, st>>>(d_gates, sites, site_stride, chi);
}

// Copy the live (dl, 2, dr) block of every site from one store layout to
// another (capacity growth). dims: 2 ints per site.
__global__ void regrow_kernel(const cplx* __restrict__ src, long long src_stride, int src_chi,
                              cplx* __restrict__ dst, long long dst_stride, int dst_chi,
                              const int* __restrict__ dims) {
  const int site = blockIdx.y;
  const int dl = dims[2 * site], dr = dims[2 * site + 1];
  const long long total = (long long)dl * 2 * dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / dr), r = (int)(i % dr);
    dst[site * dst_stride + (long long)row * dst_chi + r] = src[site * src_stride + (long long)row * src_chi + r];
  }
}

void launch_regrow(const cplx* src, long long src_stride, int src_chi, cplx* dst, long long dst_stride,
                   int dst_chi, const int* d_dims, int n_sites, cudaStream_t st) {
  regrow_kernel<<<dim3(64, n_sites), 256, 0, st>>>(src, src_stride, src_chi, dst, dst_stride, dst_chi, d_dims);
}

// Pack / unpack one site between the padded store and a dense (dl,2,dr) buffer.
__global__ void pack_site_kernel(const cplx* __restrict__ site, int chi, int dl, int dr, cplx* __restrict__ out) {
  const long long total = (long long)dl * 2 * dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / dr), r = (int)(i % dr);
    out[i] = site[(long long)row * chi + r];
  }
}
__global__ void unpack_site_kernel(const cplx* __restrict__ in, int chi, int dl, int dr, cplx* __restrict__ site) {
  const long long total = (long long)dl * 2 * dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(i / dr), r = (int)(i % dr);
    site[(long long)row * chi + r] = in[i];
  }
}

void launch_pack_site(const cplx* site, int chi, int dl, int dr, cplx* out, cudaStream_t st) {
  pack_site_kernel<<<64, 256, 0, st>>>(site, chi, dl, dr, out);
}
void launch_unpack_site(const cplx* in, int chi, int dl, int dr, cplx* site, cudaStream_t st) {
  unpack_site_kernel<<<64, 256, 0, st>>>(in, chi, dl, dr, site);
}

}  // namespace mpsim_gpu
