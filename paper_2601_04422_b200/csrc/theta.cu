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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <string>

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
        // split planes (common.cuh): the Jacobi / QR operand and X0
        if (g.trans == 0) xs_set(X + col * ldx, ldx, row, v);
        else xs_set(X + row * ldx, ldx, col, vc);
        if (g.f == 0) xs_set(X0 + col * g.x0_ld, g.x0_ld, row, v);
        else xs_set(X0 + row * g.x0_ld, g.x0_ld, col, vc);
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

// ---- DMMA variant (default). Same tile (32 l x 32 r x all (p0, p1)) as a
// complex GEMM C (64 x 64) = A (64 x Dm) B (Dm x 64), rows (l, p0), cols
// (p1, r), on mma.sync.m8n8k4.f64 in real-extended form with the complex
// interleave as the K index: k = 2 m + c,
//   A_ext[row][2m + c] = (Re, Im)[c] A[row][m]        (the smem layout as loaded)
//   Re C: B_ext[2m + c][j] = (Re B, -Im B)[c],  Im C: B_ext[2m + c][j] = (Im B, Re B)[c]
// so one 16-byte B load feeds the Re and the Im tile. 16 m per stage, two
// stages in flight with cp.async (zero-filled outside the tensors).
namespace {
constexpr int kTM = 16;          // m per stage
constexpr int kPA = 2 * kTM + 4; // A row pitch (doubles): == 4 mod 16, conflict-free fragments
constexpr int kPB = 2 * 64 + 4;  // B row pitch (doubles)
struct ThetaSmem {
  union {
    struct {
      double A[2][64 * kPA];
      double B[2][kTM * kPB];
    } st;
    cplx C[64 * 65];  // epilogue staging
  } u;
  cplx U[16];
};
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void dmma_t(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
}  // namespace

__global__ void __launch_bounds__(256, 2) theta_dmma_kernel(const GateDesc* __restrict__ gates,
                                                            const cplx* __restrict__ sites, long long site_stride,
                                                            int chi, cplx* __restrict__ ws,
                                                            double* __restrict__ frob2) {
  const GateDesc& g = gates[blockIdx.y];
  const int tiles_r = (g.dr + kTR - 1) / kTR;
  const int tiles_l = (g.dl + kTL - 1) / kTL;
  const int tl = blockIdx.x / tiles_r, tr = blockIdx.x % tiles_r;
  if (tl >= tiles_l) return;
  const int l0 = tl * kTL, r0 = tr * kTR;
  const int dl = g.dl, dm = g.dm, dr = g.dr;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ThetaSmem& S = *reinterpret_cast<ThetaSmem*>(smem_raw);
  const cplx* A = sites + (long long)g.q * site_stride;
  const cplx* B = sites + (long long)(g.q + 1) * site_stride;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  if (t < 16) S.U[t] = g.u[t];

  auto issue = [&](int buf, int m0) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int idx = t + 256 * s;
      {  // A: row i = (l, p0), 16 m
        const int i = idx / kTM, mm = idx % kTM;
        const int l = l0 + i / 2, m = m0 + mm;
        const bool ok = l < dl && m < dm;
        cp_async16_zfill(&S.u.st.A[buf][i * kPA + 2 * mm], ok ? (const void*)(A + (long long)(2 * l0 + i) * chi + m)
                                                              : (const void*)A, ok);
      }
      {  // B: 16 m x 64 cols (p1, r)
        const int mm = idx / 64, j = idx % 64;
        const int p1 = j / kTR, r = r0 + j % kTR, m = m0 + mm;
        const bool ok = m < dm && r < dr;
        cp_async16_zfill(&S.u.st.B[buf][mm * kPB + 2 * j],
                         ok ? (const void*)(B + (long long)(m * 2 + p1) * chi + r) : (const void*)B, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  // warp w: row tiles 2 (w >> 1) + {0, 1}, complex column tiles 4 (w & 1) + {0..3}
  const int rt0 = 2 * (warp >> 1), ct0 = 4 * (warp & 1);
  double acc[2][4][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < 2; ++q) acc[a][c][q][0] = acc[a][c][q][1] = 0.0;
  const int nk = (dm + kTM - 1) / kTM;
  const bool im_lane = (fk & 1) != 0;  // c of this lane's k index
  issue(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      issue((kc + 1) & 1, (kc + 1) * kTM);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* As = S.u.st.A[kc & 1];
    const double* Bs = S.u.st.B[kc & 1];
#pragma unroll
    for (int ks = 0; ks < 2 * kTM / 4; ++ks) {
      const int kk = 4 * ks + fk;  // = 2 m + c
      double av[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = As[(8 * (rt0 + a) + fr) * kPA + kk];
      const int mm = kk >> 1;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 b = *reinterpret_cast<const double2*>(&Bs[mm * kPB + 2 * (8 * (ct0 + c) + fr)]);
        const double bre = im_lane ? -b.y : b.x;  // Re C tile
        const double bim = im_lane ? b.x : b.y;   // Im C tile
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          dmma_t(acc[a][c][0][0], acc[a][c][0][1], av[a], bre);
          dmma_t(acc[a][c][1][0], acc[a][c][1][1], av[a], bim);
        }
      }
    }
    __syncthreads();
  }
  // stage C (rows (l, p0), cols (p1, r)) for the gate-mix epilogue
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        S.u.C[(8 * (rt0 + a) + fr) * 65 + 8 * (ct0 + c) + 2 * fk + v] = make_double2(acc[a][c][0][v], acc[a][c][1][v]);
  __syncthreads();

  cplx* X = ws + (g.pre ? g.qr_off : g.ws_off);
  const long long ldx = g.pre ? g.qr_m_pad : g.m_pad;
  cplx* X0 = ws + g.x0_off;
  const int tx = t % 16, ty = t / 16;
  double f2 = 0.0;
#pragma unroll
  for (int ls = 0; ls < 2; ++ls)
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
      const int li = ty + 16 * ls, ri = tx + 16 * rs;
      const int l = l0 + li, r = r0 + ri;
      if (l >= dl || r >= dr) continue;
      cplx T[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) T[i] = S.u.C[(2 * li + (i >> 1)) * 65 + (i & 1) * kTR + ri];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        // theta'[p0',p1'] = sum_{p0,p1} u[2p0'+p1', 2p0+p1] T[p0][p1]  (gate_apply.cpp:127-128)
        cplx v = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 4; ++i) cfma(v, T[i], S.U[o * 4 + i]);
        const int p0o = o >> 1, p1o = o & 1;
        const long long row = l * 2 + p0o, col = p1o * dr + r;  // theta (2Dl x 2Dr)
        const cplx vc = make_double2(v.x, -v.y);
        // split planes (common.cuh): the Jacobi / QR operand and X0
        if (g.trans == 0) xs_set(X + col * ldx, ldx, row, v);
        else xs_set(X + row * ldx, ldx, col, vc);
        if (g.f == 0) xs_set(X0 + col * g.x0_ld, g.x0_ld, row, v);
        else xs_set(X0 + row * g.x0_ld, g.x0_ld, col, vc);
        f2 += cabs2(v);
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, o);
  __shared__ double red[8];
  if (lane == 0) red[warp] = f2;
  __syncthreads();
  if (t == 0) {
    double sum = 0.0;
    for (int i = 0; i < 8; ++i) sum += red[i];
    atomicAdd(frob2 + blockIdx.y, sum);
  }
}

// ---- TMA variant: the same 64 x 64 DMMA tile with its A / B stages moved by
// the tensor-memory accelerator (cp.async.bulk.tensor, mbarrier-completed)
// from per-gate tensor maps over the site store. The maps carry the gate's
// real extents, so out-of-range rows / columns arrive as zeros (no predicated
// loads), and 128-byte swizzling keeps the DMMA fragment reads conflict-free
// on the dense tiles:
//   A (site q as (2 Dl) x (Dm complex)): boxes of 64 rows x 8 complex (128 B),
//     two per 16-m stage;
//   B (site q+1 as [m][p1][r]): boxes of 16 m x 2 p1 x 8 complex r, four per
//     stage (32 r).
// Byte offset of double c in row R of a 128-B-swizzled box: R * 128 +
// ((c >> 1) ^ (R & 7)) * 16 + (c & 1) * 8.
namespace {
struct alignas(1024) ThetaTmaSmem {
  union {
    struct {
      double A[2][2][64 * 16];      // [stage][box][row * 16 + double]
      double B[2][4][16 * 2 * 16];  // [stage][box][(m * 2 + p1) * 16 + double]
    } st;
    cplx C[64 * 65];
  } u;
  unsigned long long bar[2];
  cplx U[16];
};
constexpr unsigned kThetaStageBytes = 2 * 64 * 16 * 8 + 4 * 16 * 2 * 16 * 8;  // 32 KB

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const void* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const void* map, int c0, int c1, int c2, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ int swz(int row, int c) { return row * 16 + ((((c >> 1) ^ (row & 7))) << 1) + (c & 1); }
}  // namespace

// maps: per gate two 128-byte CUtensorMaps (A, then B), 64-byte aligned.
__global__ void __launch_bounds__(256, 2) theta_tma_kernel(const GateDesc* __restrict__ gates,
                                                           const CUtensorMap* __restrict__ maps,
                                                           cplx* __restrict__ ws, double* __restrict__ frob2) {
  const GateDesc& g = gates[blockIdx.y];
  const int tiles_r = (g.dr + kTR - 1) / kTR;
  const int tiles_l = (g.dl + kTL - 1) / kTL;
  const int tl = blockIdx.x / tiles_r, tr = blockIdx.x % tiles_r;
  if (tl >= tiles_l) return;
  const int l0 = tl * kTL, r0 = tr * kTR;
  const int dl = g.dl, dm = g.dm, dr = g.dr;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 128-byte swizzling needs 1024-byte aligned boxes: align the dynamic base
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  ThetaTmaSmem& S = *reinterpret_cast<ThetaTmaSmem*>(base);
  const CUtensorMap* mapA = maps + 2 * blockIdx.y;
  const CUtensorMap* mapB = mapA + 1;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  if (t < 16) S.U[t] = g.u[t];
  if (t == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(mapB) : "memory");
  }
  __syncthreads();
  auto issue = [&](int buf, int m0) {  // one thread: arm the stage's barrier, start six boxes
    mbar_expect_tx(&S.bar[buf], kThetaStageBytes);
    for (int b = 0; b < 2; ++b) tma_2d(S.u.st.A[buf][b], mapA, 2 * m0 + 16 * b, 2 * l0, &S.bar[buf]);
    for (int b = 0; b < 4; ++b) tma_3d(S.u.st.B[buf][b], mapB, 2 * (r0 + 8 * b), 0, m0, &S.bar[buf]);
  };
  const int rt0 = 2 * (warp >> 1), ct0 = 4 * (warp & 1);
  double acc[2][4][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < 2; ++q) acc[a][c][q][0] = acc[a][c][q][1] = 0.0;
  const int nk = (dm + kTM - 1) / kTM;
  const bool im_lane = (fk & 1) != 0;
  if (t == 0) issue(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (t == 0 && kc + 1 < nk) issue(buf ^ 1, (kc + 1) * kTM);
    mbar_wait(&S.bar[buf], (kc >> 1) & 1);
#pragma unroll
    for (int ks = 0; ks < 2 * kTM / 4; ++ks) {
      const int kk = 4 * ks + fk;  // = 2 m + c over the stage's 16 m
      const double* Ab = S.u.st.A[buf][kk >> 4];
      const int cA = kk & 15;
      double av[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = Ab[swz(8 * (rt0 + a) + fr, cA)];
      const int mm = kk >> 1;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = 8 * (ct0 + c);  // complex column tile start: p1 = j / 32, box (j % 32) / 8
        const double* Bb = S.u.st.B[buf][(j & 31) >> 3];
        const int row = mm * 2 + (j >> 5);
        const double2 b = *reinterpret_cast<const double2*>(&Bb[swz(row, 2 * fr)]);
        const double bre = im_lane ? -b.y : b.x;
        const double bim = im_lane ? b.x : b.y;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          dmma_t(acc[a][c][0][0], acc[a][c][0][1], av[a], bre);
          dmma_t(acc[a][c][1][0], acc[a][c][1][1], av[a], bim);
        }
      }
    }
    __syncthreads();  // every warp is done with this stage before TMA refills it
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        S.u.C[(8 * (rt0 + a) + fr) * 65 + 8 * (ct0 + c) + 2 * fk + v] = make_double2(acc[a][c][0][v], acc[a][c][1][v]);
  __syncthreads();

  cplx* X = ws + (g.pre ? g.qr_off : g.ws_off);
  const long long ldx = g.pre ? g.qr_m_pad : g.m_pad;
  cplx* X0 = ws + g.x0_off;
  const int tx = t % 16, ty = t / 16;
  double f2 = 0.0;
#pragma unroll
  for (int ls = 0; ls < 2; ++ls)
#pragma unroll
    for (int rs = 0; rs < 2; ++rs) {
      const int li = ty + 16 * ls, ri = tx + 16 * rs;
      const int l = l0 + li, r = r0 + ri;
      if (l >= dl || r >= dr) continue;
      cplx T[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) T[i] = S.u.C[(2 * li + (i >> 1)) * 65 + (i & 1) * kTR + ri];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        cplx v = make_double2(0.0, 0.0);  // gate mix, gate_apply.cpp:127-128
#pragma unroll
        for (int i = 0; i < 4; ++i) cfma(v, T[i], S.U[o * 4 + i]);
        const int p0o = o >> 1, p1o = o & 1;
        const long long row = l * 2 + p0o, col = p1o * dr + r;
        const cplx vc = make_double2(v.x, -v.y);
        if (g.trans == 0) xs_set(X + col * ldx, ldx, row, v);
        else xs_set(X + row * ldx, ldx, col, vc);
        if (g.f == 0) xs_set(X0 + col * g.x0_ld, g.x0_ld, row, v);
        else xs_set(X0 + row * g.x0_ld, g.x0_ld, col, vc);
        f2 += cabs2(v);
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f2 += __shfl_xor_sync(0xffffffffu, f2, o);
  __shared__ double red[8];
  if (lane == 0) red[warp] = f2;
  __syncthreads();
  if (t == 0) {
    double sum = 0.0;
    for (int i = 0; i < 8; ++i) sum += red[i];
    atomicAdd(frob2 + blockIdx.y, sum);
  }
}

void theta_init() {
  cudaFuncSetAttribute(theta_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ThetaSmem));
  cudaFuncSetAttribute(theta_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(ThetaTmaSmem) + 1024);
}

// Theta staging: TMA (default; tensor maps per gate) or 16-byte cp.async
// (MPSIM_THETA=cpasync) or the SIMT DFMA kernel (MPSIM_THETA=simt), A/B only.
static int theta_variant() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_THETA");
    if (e != nullptr && std::string(e) == "simt") return 2;
    if (e != nullptr && std::string(e) == "cpasync") return 1;
    return 0;
  }();
  return v;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Per-gate maps: A = site q as rows (l, p0) x 2 Dm doubles, B = site q+1 as
// [m][p1][2 Dr doubles]; row strides are the padded slot's (chi complex).
bool encode_maps(const GateDesc& g, const cplx* sites, long long site_stride, int chi, CUtensorMap* out) {
  auto enc = encode_fn();
  if (!enc) return false;
  const cplx* A = sites + (long long)g.q * site_stride;
  const cplx* B = sites + (long long)(g.q + 1) * site_stride;
  const cuuint32_t es[3] = {1, 1, 1};
  {
    const cuuint64_t dim[2] = {(cuuint64_t)2 * g.dm, (cuuint64_t)2 * g.dl};
    const cuuint64_t str[1] = {(cuuint64_t)chi * sizeof(cplx)};
    const cuuint32_t box[2] = {16, 64};
    if (enc(&out[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  {
    const cuuint64_t dim[3] = {(cuuint64_t)2 * g.dr, 2, (cuuint64_t)g.dm};
    const cuuint64_t str[2] = {(cuuint64_t)chi * sizeof(cplx), (cuuint64_t)2 * chi * sizeof(cplx)};
    const cuuint32_t box[3] = {16, 2, 16};
    if (enc(&out[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)B, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}
}  // namespace

// Returns the kernel launched (0 TMA, 1 cp.async, 2 SIMT). maps_h / maps_d:
// room for 2 * n_gates CUtensorMaps (pinned host / device, 64-byte aligned).
int launch_theta(const GateDesc* d_gates, const GateDesc* h_gates, int n_gates, int max_tiles, const cplx* sites,
                 long long site_stride, int chi, cplx* ws, double* frob2, CUtensorMap* maps_h, CUtensorMap* maps_d,
                 cudaStream_t st) {
  if (n_gates == 0) return 0;
  int v = theta_variant();
  if (v == 0) {
    for (int i = 0; i < n_gates && v == 0; ++i)
      if (!encode_maps(h_gates[i], sites, site_stride, chi, maps_h + 2 * i)) v = 1;
  }
  if (v == 0) {
    cudaMemcpyAsync(maps_d, maps_h, sizeof(CUtensorMap) * 2 * n_gates, cudaMemcpyHostToDevice, st);
    theta_tma_kernel<<<dim3(max_tiles, n_gates), 256, sizeof(ThetaTmaSmem) + 1024, st>>>(d_gates, maps_d, ws, frob2);
  } else if (v == 2) {
    theta_kernel<<<dim3(max_tiles, n_gates), 256, 0, st>>>(d_gates, sites, site_stride, chi, ws, frob2);
  } else {
    theta_dmma_kernel<<<dim3(max_tiles, n_gates), 256, sizeof(ThetaSmem), st>>>(d_gates, sites, site_stride, chi,
                                                                                 ws, frob2);
  }
  return v;
}

int theta_tiles(int dl, int dr) { return ((dl + kTL - 1) / kTL) * ((dr + kTR - 1) / kTR); }

}  // namespace mpsim_gpu
