// Block one-sided Jacobi on the FP64 tensor path: the visit of one block pair
// (2W = 32 vectors) of a tournament round —
//   1. Gram G = X_P^H X_P on DMMA (36 tiles of the real-extended 64 x 64 Gram,
//      or the 16 cross-block tiles when the in-block Grams are reused),
//   2. the relative convergence test,
//   3. one cyclic complex Jacobi sweep of the 32 x 32 G (evd.cuh) -> R,
//   4. X_P <- X_P R on DMMA —
// as one persistent launch per sweep (jacobi_sweep_kernel, default), one
// launch per round (jacobi_gram_kernel<2>), or split into Gram+EVD / rotation
// or Gram / EVD / rotation launches (A/B). The Jacobi operand X lives in
// global memory as split planes per vector (Re[0, m_pad) then Im[0, m_pad),
// common.cuh), so 32-row chunks stream into vector-major shared planes with
// 16-byte cp.async.
#include "common.cuh"
#include "evd.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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
  // vector i of the pair as split planes: Re at [0, mp), Im at [mp, 2 mp)
  __device__ __forceinline__ double* vec(int i) const {
    const int slot = i < kW ? ba * kW + i : bb * kW + (i - kW);
    return reinterpret_cast<double*>(X + (long long)pm[slot] * mp);
  }
};

// Returns false if this CTA has no pair in this round.
__device__ __forceinline__ bool pair_ctx(const GateDesc& g, int gi, int round, const int* active, cplx* ws,
                                         const int* perm, long long perm_stride, PairCtx& c, int k) {
  if (!active[gi]) return false;
  const int nb = g.nb;
  if (round >= nb - 1 || k >= nb / 2) return false;
  rr_pair(round, k, nb - 1, c.ba, c.bb);
  c.X = ws + g.ws_off;
  c.pm = perm + gi * perm_stride;
  c.mp = g.m_pad;
  return true;
}

// Chunks of kC rows x 32 vectors stream through shared memory as split Re/Im
// planes [vector][row] (pitch 36), double-buffered with cp.async so the next
// chunk's loads are in flight while the DMMAs consume the current one.
constexpr int kC = 32;
constexpr int kChunkPlane = kP * kPitchS;  // doubles per plane

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
// 16-byte copy with an L2 eviction-priority hint (createpolicy below)
__device__ __forceinline__ void cp_async16_hint(double* smem, const double* gmem, unsigned long long pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "l"(pol));
}
// L2 policies: 0 normal, 1 evict_first, 2 evict_last
__device__ __forceinline__ unsigned long long l2_policy(int kind) {
  unsigned long long p;
  if (kind == 1)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* gmem, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(gmem), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Per chunk and thread four 16-byte copies (two rows of one plane of one
// vector): in copy s, warp w moves vector w + 8 s, lanes 0-15 its Re rows and
// lanes 16-31 its Im rows, 256 contiguous bytes each (full lines from global,
// conflict-free in shared memory).
struct ChunkLoader {
  const double* src[4];  // this thread's plane of vectors w + 8 s, at its row pair
  int soff;              // shared offset of vector w, plane, row pair
  __device__ __forceinline__ void init(const PairCtx& c, int t) {
    const int lane = t & 31, warp = t >> 5;
    const int rp = lane & 15, plane = lane >> 4;
#pragma unroll
    for (int s = 0; s < 4; ++s) src[s] = c.vec(warp + 8 * s) + plane * c.mp + 2 * rp;
    soff = plane * kChunkPlane + warp * kPitchS + 2 * rp;
  }
  unsigned long long pol;  // L2 policy of the copies (set per pass)
  // rows e0 .. e0 + kC of the pair -> buffer (Re plane at buf, Im at buf + kChunkPlane)
  __device__ __forceinline__ void issue(double* buf, int e0) const {
#pragma unroll
    for (int s = 0; s < 4; ++s) cp_async16_hint(buf + soff + 8 * s * kPitchS, src[s] + e0, pol);
    cp_async_commit();
  }
};

constexpr int kPitchR = 34;  // complex R row pitch (== 2 mod 8: conflict-free 16-byte B fragments)

// Gram (+ pair EVD (+ rotation)) of one block pair in one CTA. R aliases the
// chunk buffers / Gx, dead once G is built; the rotation's copy of R aliases G,
// dead once the in-block Grams are stored: 55 KB per CTA.
struct PairSmem {
  union {
    double buf[2][2 * kChunkPlane];
    double Gx[64 * 65];  // real 64x64 Gram (after the chunk loop)
  } u;
  union {
    cplx G[kP * kPad];
    cplx Rs[kP * kPitchR];           // R for the rotation
    double buf3[2 * kChunkPlane];    // third Gram-pass stage (G / Rs are dead then)
  } v;
  EvdScratch sc;
};
static_assert(sizeof(cplx) * kP * kPad <= sizeof(PairSmem::u), "R must fit in the chunk buffers");

// X_P <- X_P R over all chunks, on DMMA with the three-real-product complex
// multiply: one 16-byte load of R[c][j] gives the B fragments of Re R, Im R
// and Re R + Im R for a k-step. Warp w computes row tiles {2(w&1), +1} of a
// chunk and complex column tile w/2: per k-step four A loads (Re and Im planes)
// and one B load feed six DMMAs, and each thread ends up with Re and Im of
// the same complex outputs.
__device__ __forceinline__ void rotate_pair(const PairCtx& c, const ChunkLoader& ld, double (*buf)[2 * kChunkPlane],
                                            const cplx* Rs, int c0, int nchunks, int t, int b0 = 0,
                                            unsigned long long spol = 0, bool shint = false) {
  const int lane = t % 32, warp = t / 32;
  const int fr = lane / 4, fk = lane % 4;
  const int rbase = 2 * (warp & 1), cj = warp >> 1;
  const int jb = 8 * cj + fr;
  // this thread's two output vectors (the permutation lookups stay out of the loop)
  double* const xo[2] = {c.vec(8 * cj + 2 * fk), c.vec(8 * cj + 2 * fk + 1)};
  // chunks [c0, c0 + nchunks) last to first: the rows the Gram pass read last
  // are the likeliest still in L2 (the caller issues chunk c0 + nchunks - 1
  // into buffer b0)
  for (int k = 0; k < nchunks; ++k) {
    // one barrier per chunk: it publishes chunk k and certifies that every
    // warp is done with chunk k - 1, whose buffer the next load then reuses
    cp_async_wait<0>();
    __syncthreads();
    if (k + 1 < nchunks) ld.issue(buf[(k + 1 + b0) & 1], (c0 + nchunks - 2 - k) * kC);
    const double* B = buf[(k + b0) & 1];
    // complex product in three real products (Gauss): T1 = Xr Rr, T2 = Xi Ri,
    // T3 = (Xr + Xi)(Rr + Ri); Re = T1 - T2, Im = T3 - T1 - T2. 48 DMMAs per
    // warp and chunk instead of 64; each output column's error stays bounded
    // by eps * sum_q |x_q| |R_qp| (columnwise, as the Jacobi needs)
    double t1[2][2], t2[2][2], t3[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a) t1[a][0] = t1[a][1] = t2[a][0] = t2[a][1] = t3[a][0] = t3[a][1] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int cc = 4 * s + fk;
      const double* pr = B + cc * kPitchS;
      const double* pim = pr + kChunkPlane;
      const double ar0 = pr[8 * rbase + fr], ar1 = pr[8 * (rbase + 1) + fr];
      const double ai0 = pim[8 * rbase + fr], ai1 = pim[8 * (rbase + 1) + fr];
      const cplx r = Rs[cc * kPitchR + jb];
      const double rs = r.x + r.y;
      dmma_s(t1[0][0], t1[0][1], ar0, r.x);
      dmma_s(t1[1][0], t1[1][1], ar1, r.x);
      dmma_s(t2[0][0], t2[0][1], ai0, r.y);
      dmma_s(t2[1][0], t2[1][1], ai1, r.y);
      dmma_s(t3[0][0], t3[0][1], ar0 + ai0, rs);
      dmma_s(t3[1][0], t3[1][1], ar1 + ai1, rs);
    }
    double o[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        o[a][0][v] = t1[a][v] - t2[a][v];
        o[a][1][v] = t3[a][v] - t1[a][v] - t2[a][v];
      }
    const int e0 = (c0 + nchunks - 1 - k) * kC;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = 8 * (rbase + a) + fr;
        double* xj = xo[v];
        if (shint) {
          st_hint(xj + e0 + e, o[a][0][v], spol);
          st_hint(xj + c.mp + e0 + e, o[a][1][v], spol);
        } else {
          xj[e0 + e] = o[a][0][v];
          xj[c.mp + e0 + e] = o[a][1][v];
        }
      }
  }
}

// R (complex, pitch rpitch) -> Rs (pitch kPitchR)
__device__ __forceinline__ void copy_rotation(const cplx* R, long long rpitch, cplx* Rs, int t) {
  for (int idx = t; idx < kP * kP; idx += 256) {
    const int i = idx / kP, j = idx % kP;
    Rs[i * kPitchR + j] = R[i * rpitch + j];
  }
}

}  // namespace

// Gram pass over chunks [c0, c0 + nchunks) of the pair into S.u.Gx: the 16
// cross tiles (cross_only) or the 36 tiles of the upper real-extended Gram.
// nchunks may be 0 (the tiles are then zero). Ends with a block barrier.
__device__ __forceinline__ void gram_pass(PairSmem& S, const ChunkLoader& ld, int c0, int nchunks, bool cross_only,
                                          int t) {
  const int lane = t % 32, warp = t / 32;
  const int fr = lane / 4, fk = lane % 4;
  // column offsets (plane + index) of this thread's fragments
  auto coff = [&](int col) { return (col < kP ? 0 : kChunkPlane) + (col & (kP - 1)) * kPitchS; };
  // Gram pass: a three-stage cp.async ring (two chunk buffers + the G / R
  // union, free until the Gram is assembled): the pass does only 16-36 tiles
  // of DMMA per 32-row chunk, too little to hide a load issued one chunk ahead
  auto stage = [&](int k) -> double* {
    const int s3 = k % 3;
    return s3 == 2 ? S.v.buf3 : S.u.buf[s3];
  };
  // One barrier per chunk: after it, chunk k is visible to every warp and every
  // warp is done with chunk k - 1, whose stage the load of chunk k + 2 reuses.
  auto next_chunk = [&](int k) {  // chunk k's data ready in shared memory
    if (k + 1 < nchunks) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    if (k + 2 < nchunks) ld.issue(stage(k + 2), (c0 + k + 2) * kC);
  };
  if (nchunks > 0) ld.issue(stage(0), c0 * kC);
  if (nchunks > 1) ld.issue(stage(1), (c0 + 1) * kC);
  if (cross_only) {
    // the 16 cross tiles (rows Re_a / Im_a = tiles 0,1 / 4,5; cols Re_b / Im_b =
    // 2,3 / 6,7) as four 2x2 blocks, warp & 3 picks the block and warp >> 2
    // the half of each chunk's k-steps: two A and two B loads feed four DMMAs
    const int q = warp & 3, kh = warp >> 2;
    const int tr0 = (q >> 1) ? 4 : 0, tc0 = (q & 1) ? 6 : 2;
    const int oa0 = coff(8 * tr0 + fr), oa1 = coff(8 * (tr0 + 1) + fr);
    const int ob0 = coff(8 * tc0 + fr), ob1 = coff(8 * (tc0 + 1) + fr);
    double acc[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int k = 0; k < nchunks; ++k) {
      next_chunk(k);
      const double* B = stage(k);
#pragma unroll
      for (int ks = 0; ks < kC / 8; ++ks) {
        const int row = 4 * (ks + (kC / 8) * kh) + fk;
        const double a0 = B[row + oa0], a1 = B[row + oa1], b0 = B[row + ob0], b1 = B[row + ob1];
        dmma_s(acc[0][0][0], acc[0][0][1], a0, b0);
        dmma_s(acc[0][1][0], acc[0][1][1], a0, b1);
        dmma_s(acc[1][0][0], acc[1][0][1], a1, b0);
        dmma_s(acc[1][1][0], acc[1][1][1], a1, b1);
      }
    }
    __syncthreads();  // the last stage is read; Gx aliases the chunk buffers
    for (int h = 0; h < 2; ++h) {  // the two k-halves into Gx
      if (kh == h)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              double& gx = S.u.Gx[(8 * (tr0 + a) + fr) * 65 + 8 * (tc0 + b) + fk * 2 + v];
              gx = h == 0 ? acc[a][b][v] : gx + acc[a][b][v];
            }
      __syncthreads();
    }
  } else {
    // tiles of G_ext = [[A, B], [B^T, D]]: upper A and D, all of B (Re G = A + D,
    // Im G = B - B^T); warps 0-3: tile row w of B (4 tiles), warps 4-7: tile row
    // r of A and 3 - r of D (5 tiles)
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
    const int oa0 = coff(8 * trow[0] + fr), oa4 = coff(8 * trow[4] + fr);
    int ob[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) ob[i] = coff(8 * tcol[i] + fr);
    double acc[5][2];
#pragma unroll
    for (int i = 0; i < 5; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int k = 0; k < nchunks; ++k) {
      next_chunk(k);
      const double* B = stage(k);
#pragma unroll
      for (int ks = 0; ks < kC / 4; ++ks) {
        const int row = 4 * ks + fk;
        const double a_first = B[row + oa0], a_last = B[row + oa4];
#pragma unroll
        for (int i = 0; i < 5; ++i)
          if (i < nt) dmma_s(acc[i][0], acc[i][1], trow[i] == trow[0] ? a_first : a_last, B[row + ob[i]]);
      }
    }
    __syncthreads();  // the last stage is read; Gx aliases the chunk buffers
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if (i < nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) S.u.Gx[(8 * trow[i] + fr) * 65 + 8 * tcol[i] + fk * 2 + v] = acc[i][v];
    __syncthreads();
  }
}

#ifdef MPSIM_AB_KNOBS
// A/B builds: per-phase SM clock totals of the persistent sweep (thread 0 of
// every CTA): 0 visits, 1 wait for blocks, 2 Gram pass, 3 assembly + test,
// 4 EVD, 5 rotation, 6 visit count, 7 EVD count.
__device__ unsigned long long g_phase_clk[8];
#define PHASE_MARK(var) long long var = clock64()
#define PHASE_ADD(i, v) \
  if (threadIdx.x == 0) atomicAdd(&g_phase_clk[i], (unsigned long long)(v))
#else
#define PHASE_MARK(var)
#define PHASE_ADD(i, v)
#endif

// Cross-block-only pair EVD: every round of a pre-asymptotic sweep (active
// bit 2), else the rounds off a period of 2 (bit 16) or 3 (bits 16 | 32):
// the remaining rounds still rotate the in-block pairs, which keeps the
// outer sweep count (tools/emu_jacobi.py).
__device__ __forceinline__ bool cross_only_evd(int active, int round) {
  if (active & 2) return true;
  if (!(active & 16)) return false;
  return round % ((active & 32) ? 3 : 2) != 0;
}

// kMode 0: Gram only (G -> gbuf); 1: Gram + pair EVD (R -> rbuf); 2: the whole
// pair visit, Gram + EVD + rotation, in one CTA.
// Pre-asymptotic (in-block-cached) visits decide on rotation and report maxoff
// from the cross entries alone.
constexpr int kCrossTest = 1;
struct RoundArgs {
  const GateDesc* gates;
  cplx* ws;
  const int* active;
  double tol;
  const double* frob2;
  double floor_rel2;
  const int* perm;
  long long perm_stride;
  double* maxoff;
  int* need;
  cplx* gbuf;
  int max_pairs;
  double* offsum;
  cplx* rbuf;
  double tol_in;
  cplx* gblk;
  int* rotated;
  int probe;
  int* blkok;  // per block: gblk holds its exact in-block Gram (persistent sweeps; nullable)
  int l2hint;  // L2 priorities: 0 none; 1 rotation loads / stores evict_first; 2 and Gram loads evict_last
  int ns_iters = 2;  // Newton-Schulz steps of the FP32 pair EVD's polar factor (A/B)
  int xtest = kCrossTest;  // pre-asymptotic visits: rotation test on the cross entries only (A/B: MPSIM_XTEST)
};

// One pair visit (block pair k of gate gi in tournament round `round`).
template <int kMode>
__device__ __forceinline__ void pair_visit(const RoundArgs& A, int gi, int round, int k, PairSmem& S) {
  constexpr bool kFuseEvd = kMode >= 1;
  const GateDesc* __restrict__ gates = A.gates;
  cplx* __restrict__ ws = A.ws;
  const int* __restrict__ active = A.active;
  const double tol = A.tol, floor_rel2 = A.floor_rel2, tol_in = A.tol_in;
  const double* __restrict__ frob2 = A.frob2;
  const int* __restrict__ perm = A.perm;
  const long long perm_stride = A.perm_stride;
  double* __restrict__ maxoff = A.maxoff;
  int* __restrict__ need = A.need;
  cplx* __restrict__ gbuf = A.gbuf;
  const int max_pairs = A.max_pairs;
  double* __restrict__ offsum = A.offsum;
  cplx* __restrict__ rbuf = A.rbuf;
  cplx* __restrict__ gblk = A.gblk;
  int* __restrict__ rotated = A.rotated;
  const int probe = A.probe;
  const GateDesc& g = gates[gi];
  PairCtx c;
  if (!pair_ctx(g, gi, round, active, ws, perm, perm_stride, c, k)) return;
  cplx* const SG = S.v.G;
  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  ChunkLoader ld;
  ld.init(c, t);
  ld.pol = l2_policy(A.l2hint >= 2 ? 2 : 0);
  // Stored in-block Grams (active bit 4, rounds > 0 of a pre-asymptotic
  // sweep): the in-block 16 x 16 Grams of both blocks are those the pair EVD
  // left at the blocks' previous visit this sweep (R^H G R, exact up to
  // rounding: the blocks have not changed since), so only the cross block
  // X_a^H X_b is computed: 16 of the 36 DMMA tiles.
  const bool approx = kFuseEvd && (active[gi] & 4) && round > 0;
  // Exact cache (active bit 8, closing sweeps): a visit that computed all 36
  // tiles and did not rotate leaves the blocks' in-block Grams in gblk and
  // flags them; a later visit of two flagged (hence unchanged) blocks this
  // sweep needs only the cross tiles — the in-block values are exactly what
  // recomputing them would give. A rotation clears the flags.
  int* const ok_a = A.blkok ? A.blkok + (long long)gi * 2 * max_pairs + c.ba : nullptr;
  int* const ok_b = A.blkok ? A.blkok + (long long)gi * 2 * max_pairs + c.bb : nullptr;
  const bool cached = kFuseEvd && !approx && ok_a && (active[gi] & 8) && round > 0 && *ok_a && *ok_b;
  const bool cross_only = approx || cached;
  cplx* const gblk_a = gblk + ((long long)gi * 2 * max_pairs + c.ba) * (kW * kW);
  cplx* const gblk_b = gblk + ((long long)gi * 2 * max_pairs + c.bb) * (kW * kW);
  const int nchunks = g.m_pad / kC;
  PHASE_MARK(c_g0);
  gram_pass(S, ld, 0, nchunks, cross_only, t);
  PHASE_MARK(c_g1);
  PHASE_ADD(2, c_g1 - c_g0);
  if (cross_only) {
    const double* Gx = S.u.Gx;
    const int i = t >> 4, j = kW + (t & 15);
    const double re = Gx[i * 65 + j] + Gx[(kP + i) * 65 + kP + j];
    const double im = Gx[i * 65 + kP + j] - Gx[(kP + i) * 65 + j];
    SG[i * kPad + j] = make_double2(re, im);
    SG[j * kPad + i] = make_double2(re, -im);
    const int r = t >> 4, q = t & 15;
    SG[r * kPad + q] = gblk_a[t];
    SG[(kW + r) * kPad + kW + q] = gblk_b[t];
  } else {
    for (int idx = t; idx < kP * kP; idx += 256) {
      const int i = idx / kP, j = idx % kP;
      if (i > j) continue;
      const double* Gx = S.u.Gx;
      const double re = Gx[i * 65 + j] + Gx[(kP + i) * 65 + kP + j];
      const double im = Gx[i * 65 + kP + j] - Gx[j * 65 + kP + i];
      SG[i * kPad + j] = make_double2(re, i == j ? 0.0 : im);
      if (i != j) SG[j * kPad + i] = make_double2(re, -im);
    }
  }
  __syncthreads();
  const double tolg = tol * fmax(sqrt((double)g.m), (double)kP);
  const double floor2 = floor_rel2 * frob2[gi];
  double rx;  // this thread's squared relative cross off-diagonal
  {
    // sum of squared relative off-diagonals between the two blocks: the host
    // turns it into the sweep's rms off-norm (cross-only EVD policy)
    const int i = t >> 4, j = kW + (t & 15);
    const double gii = SG[i * kPad + i].x, gjj = SG[j * kPad + j].x;
    // (policy input only: the squared ratio in FP32 when in range)
    const double c2 = cabs2(SG[i * kPad + j]), d = gii * gjj;
    double r = 0.0;
    if (fmin(gii, gjj) > floor2)
      r = (d < 1e30 && d > 1e-12) ? (double)__fdividef((float)c2, (float)d) : c2 / d;
    rx = r;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0 && r > 0.0) atomicAdd(offsum + gi, r);
  }
  bool nd;
  if (approx && A.xtest) {
    // pre-asymptotic visit: the in-block Grams are the cached EVD output, so
    // the test and maxoff use the cross entries (the ratios above) only; the
    // closing sweeps test every pair on exact Grams
    double mx = rx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(maxoff + gi),
                (unsigned long long)__double_as_longlong(sqrt(mx)));
    nd = __syncthreads_or(rx > tolg * tolg);
  } else {
    nd = pair_needs_rotation(SG, t, tolg, floor2, maxoff + gi);
  }
  PHASE_MARK(c_a1);
  PHASE_ADD(3, c_a1 - c_g1);
  const long long slot = (long long)gi * max_pairs + k;
  if (t == 0) need[slot] = nd ? 1 : 0;
  auto store_inblock = [&]() {  // the in-block Grams for this sweep's later visits
    const int r = t >> 4, q = t & 15;
    gblk_a[t] = SG[r * kPad + q];
    gblk_b[t] = SG[(kW + r) * kPad + kW + q];
  };
  if (!nd) {
    if (kFuseEvd && !cross_only) {
      store_inblock();
      if (ok_a && t == 0) *ok_a = *ok_b = 1;
    }
    return;
  }
  if (ok_a && t == 0) *ok_a = *ok_b = 0;
  if (probe == 1) return;  // profiling (MPSIM_PHASE_PROBE): Gram only
  if constexpr (kFuseEvd) {
    cplx* R = reinterpret_cast<cplx*>(S.u.buf);
    bool evd32 = false;
    static_assert(sizeof(cplx) * kP * kPad <= sizeof(double) * 2 * kChunkPlane, "R must fit in buffer 0");
    const unsigned long long rpol = l2_policy(A.l2hint >= 1 ? 1 : 0);
    ld.pol = rpol;
    if (probe == 4) {  // profiling: the visit without its EVD (R = I)
      for (int idx = t; idx < kP * kP; idx += 256)
        R[(idx / kP) * kPad + idx % kP] = make_double2(idx / kP == idx % kP ? 1.0 : 0.0, 0.0);
      __syncthreads();
    } else if (active[gi] & 64) {
      // pre-asymptotic sweep: FP32 inner sweep + FP64 polar factor (evd.cuh);
      // W = buffer 1 (R holds buffer 0), G is scratch after the sweep
      static_assert(sizeof(cplx) * kP * kPad <= sizeof(double) * 2 * kChunkPlane, "W must fit in buffer 1");
      pair_evd_f32(SG, reinterpret_cast<cplx*>(S.u.buf[1]), R, S.sc, t, floor2, cross_only_evd(active[gi], round),
                   [&](const float2* G32) {
                     const int r = t >> 4, q = t & 15;
                     const float2 ga = G32[r * kPad + q], gb = G32[(kW + r) * kPad + kW + q];
                     gblk_a[t] = make_double2(ga.x, ga.y);
                     gblk_b[t] = make_double2(gb.x, gb.y);
                   },
                   probe == 5 ? 0 : A.ns_iters);
      evd32 = true;
    } else {
      pair_evd_v1(SG, R, S.sc, t, tol_in, floor2, 1, cross_only_evd(active[gi], round));
    }
    if (probe == 2) return;  // Gram + EVD
    __syncthreads();
    PHASE_MARK(c_e1);
    PHASE_ADD(4, c_e1 - c_a1);
    PHASE_ADD(7, 1);
    if (!evd32) store_inblock();
    if constexpr (kMode == 1) {
      cplx* rout = rbuf + slot * (kP * kP);
      for (int idx = t; idx < kP * kP; idx += 256) rout[idx] = R[(idx / kP) * kPad + idx % kP];
    } else {
      __syncthreads();  // G (aliased by R_ext) has been stored
      copy_rotation(R, kPad, S.v.Rs, t);
      __syncthreads();  // R (aliased by the chunk buffers) has been read
      ld.issue(S.u.buf[0], (nchunks - 1) * kC);
      rotate_pair(c, ld, S.u.buf, S.v.Rs, 0, nchunks, t, 0, rpol, A.l2hint >= 1);
      PHASE_MARK(c_r1);
      PHASE_ADD(5, c_r1 - c_e1);
      if (t == 0) atomicAdd(rotated + gi, 1);
    }
  } else {
    cplx* gout = gbuf + slot * (kP * kP);
    for (int idx = t; idx < kP * kP; idx += 256) gout[idx] = SG[(idx / kP) * kPad + idx % kP];
  }
}

template <int kMode>
__global__ void __launch_bounds__(256, 3) jacobi_gram_kernel(RoundArgs A, int round) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pair_visit<kMode>(A, blockIdx.y, round, blockIdx.x, *reinterpret_cast<PairSmem*>(smem_raw));
}

// A whole sweep in one persistent launch: CTAs claim pair visits in
// (round, gate, pair) order from a global counter and start a visit as soon
// as both of its blocks have finished the previous round (per-block round
// counters, release/acquire at gpu scope) instead of waiting for the whole
// round: no per-round launch and tail, and CTAs drift out of phase, so one
// CTA's pair EVD overlaps the DMMA phases of its neighbours. Deadlock-free:
// a visit only waits on visits claimed before it, all of which are held by
// running CTAs.
#ifndef MPSIM_SWEEP_MINB
#define MPSIM_SWEEP_MINB 4
#endif
__global__ void __launch_bounds__(256, MPSIM_SWEEP_MINB) jacobi_sweep_kernel(RoundArgs A, int n_gates, int max_rounds,
                                                              int* __restrict__ ctl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(smem_raw);
  __shared__ int s_item;
  int* counter = ctl;
  int* ready = ctl + 1;  // [gate][block]: rounds completed this sweep
  const int per_round = n_gates * A.max_pairs;
  const long long total = (long long)per_round * max_rounds;
  const int t = threadIdx.x;
  for (;;) {
    __syncthreads();  // shared memory of the previous visit is free
    if (t == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    const int round = item / per_round, rem = item % per_round;
    const int gi = rem / A.max_pairs, k = rem % A.max_pairs;
    const GateDesc& g = A.gates[gi];
    const int nb = g.nb;
    if (!A.active[gi] || round >= nb - 1 || k >= nb / 2) continue;
    int ba, bb;
    rr_pair(round, k, nb - 1, ba, bb);
    int* ra = ready + gi * 2 * A.max_pairs + ba;
    int* rb = ready + gi * 2 * A.max_pairs + bb;
    PHASE_MARK(c_w0);
    if (t == 0) {
      int v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ra) : "memory");
        if (v >= round) break;
        __nanosleep(64);
      }
      for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(rb) : "memory");
        if (v >= round) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
    PHASE_MARK(c_w1);
    PHASE_ADD(1, c_w1 - c_w0);
    pair_visit<2>(A, gi, round, k, S);
    __syncthreads();  // every thread's writes of this visit are issued
    PHASE_MARK(c_v1);
    PHASE_ADD(0, c_v1 - c_w0);
    PHASE_ADD(6, 1);
    if (t == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ra), "r"(round + 1) : "memory");
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(rb), "r"(round + 1) : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// Cluster pair visits. One visit is split by rows over a cluster of kCl CTAs
// (CTA r streams chunks [r nch / kCl, (r + 1) nch / kCl)): each computes the
// partial Gram of its rows; rank 0 sums the kCl partials in rank order through
// distributed shared memory, runs the convergence test and the pair EVD, and
// writes R into every CTA's shared memory; each CTA rotates its own rows.
// A quarter of the CTAs are in visits at any time compared with one CTA per
// visit, and visits are claimed gate group by gate group (`group` gates of
// the active list, all rounds, then the next group), so the blocks a round
// writes are read by the next round while still in L2: the sweep's working
// set is group x 16 MB (chi = 512) instead of the whole layer.
namespace {
constexpr int kCl = 4;

__device__ __forceinline__ bool decode_item(const RoundArgs& A, const int* glist, int n_list, int group,
                                            int max_rounds, long long item, int& gi, int& round, int& k) {
  const long long per_round_g = (long long)group * A.max_pairs;
  const long long per_group = per_round_g * max_rounds;
  const long long grp = item / per_group;
  long long rem = item - grp * per_group;
  round = (int)(rem / per_round_g);
  rem -= (long long)round * per_round_g;
  const int j = (int)(rem / A.max_pairs);
  k = (int)(rem - (long long)j * A.max_pairs);
  const long long idx = grp * group + j;
  if (idx >= n_list) return false;
  gi = glist[idx];
  const int nb = A.gates[gi].nb;
  return A.active[gi] && round < nb - 1 && k < nb / 2;
}

__device__ __forceinline__ void wait_round(const int* p, int round) {
  int v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= round) break;
    __nanosleep(64);
  }
}

// One pair visit by the whole cluster (every CTA calls it with the same item).
__device__ __forceinline__ void pair_visit_cl(const RoundArgs& A, int gi, int round, int k, PairSmem& S, int* s_nd,
                                              unsigned rank, cg::cluster_group& cl) {
  const GateDesc& g = A.gates[gi];
  PairCtx c;
  rr_pair(round, k, g.nb - 1, c.ba, c.bb);
  c.X = A.ws + g.ws_off;
  c.pm = A.perm + gi * A.perm_stride;
  c.mp = g.m_pad;
  const int t = threadIdx.x;
  ChunkLoader ld;
  ld.init(c, t);
  ld.pol = l2_policy(0);
  const int act = A.active[gi];
  // (see pair_visit: stored in-block Grams / exact cache)
  const bool approx = (act & 4) && round > 0;
  int* const ok_a = A.blkok ? A.blkok + (long long)gi * 2 * A.max_pairs + c.ba : nullptr;
  int* const ok_b = A.blkok ? A.blkok + (long long)gi * 2 * A.max_pairs + c.bb : nullptr;
  const bool cached = !approx && ok_a && (act & 8) && round > 0 && __ldcg(ok_a) && __ldcg(ok_b);
  const bool cross_only = approx || cached;
  const int nch = g.m_pad / kC;
  const int c0 = (int)((rank * nch) / kCl), c1 = (int)(((rank + 1) * nch) / kCl);
  gram_pass(S, ld, c0, c1 - c0, cross_only, t);
  cl.sync();  // every partial Gram is in its CTA's shared memory
  if (rank == 0) {
    cplx* const SG = S.v.G;
    cplx* const gblk_a = A.gblk + ((long long)gi * 2 * A.max_pairs + c.ba) * (kW * kW);
    cplx* const gblk_b = A.gblk + ((long long)gi * 2 * A.max_pairs + c.bb) * (kW * kW);
    const double* gx[kCl];
#pragma unroll
    for (int r = 0; r < kCl; ++r) gx[r] = cl.map_shared_rank(S.u.Gx, r);
    auto sum = [&](int off) {
      double v = gx[0][off];
#pragma unroll
      for (int r = 1; r < kCl; ++r) v += gx[r][off];
      return v;
    };
    if (cross_only) {
      const int i = t >> 4, j = kW + (t & 15);
      const double re = sum(i * 65 + j) + sum((kP + i) * 65 + kP + j);
      const double im = sum(i * 65 + kP + j) - sum((kP + i) * 65 + j);
      SG[i * kPad + j] = make_double2(re, im);
      SG[j * kPad + i] = make_double2(re, -im);
      const int r = t >> 4, q = t & 15;
      SG[r * kPad + q] = gblk_a[t];
      SG[(kW + r) * kPad + kW + q] = gblk_b[t];
    } else {
      for (int idx = t; idx < kP * kP; idx += 256) {
        const int i = idx / kP, j = idx % kP;
        if (i > j) continue;
        const double re = sum(i * 65 + j) + sum((kP + i) * 65 + kP + j);
        const double im = sum(i * 65 + kP + j) - sum(j * 65 + kP + i);
        SG[i * kPad + j] = make_double2(re, i == j ? 0.0 : im);
        if (i != j) SG[j * kPad + i] = make_double2(re, -im);
      }
    }
    __syncthreads();
    const double tolg = A.tol * fmax(sqrt((double)g.m), (double)kP);
    const double floor2 = A.floor_rel2 * A.frob2[gi];
    {
      const int i = t >> 4, j = kW + (t & 15), lane = t & 31;
      const double gii = SG[i * kPad + i].x, gjj = SG[j * kPad + j].x;
      double r = (fmin(gii, gjj) > floor2) ? cabs2(SG[i * kPad + j]) / (gii * gjj) : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
      if (lane == 0 && r > 0.0) atomicAdd(A.offsum + gi, r);
    }
    const bool nd = pair_needs_rotation(SG, t, tolg, floor2, A.maxoff + gi);
    const long long slot = (long long)gi * A.max_pairs + k;
    if (t == 0) A.need[slot] = nd ? 1 : 0;
    auto store_inblock = [&]() {
      const int r = t >> 4, q = t & 15;
      gblk_a[t] = SG[r * kPad + q];
      gblk_b[t] = SG[(kW + r) * kPad + kW + q];
    };
    if (!nd) {
      if (!cross_only) {
        store_inblock();
        if (ok_a && t == 0) *ok_a = *ok_b = 1;
      }
    } else {
      if (ok_a && t == 0) *ok_a = *ok_b = 0;
      cplx* R = reinterpret_cast<cplx*>(S.u.buf);  // this CTA's partial Gram is summed: free
      pair_evd_v1(SG, R, S.sc, t, A.tol_in, floor2, 1, cross_only_evd(act, round));
      __syncthreads();
      store_inblock();
      __syncthreads();  // G (aliased by Rs) has been stored
#pragma unroll
      for (int r = 0; r < kCl; ++r) copy_rotation(R, kPad, cl.map_shared_rank(S.v.Rs, r), t);
      if (t == 0) atomicAdd(A.rotated + gi, 1);
    }
    if (t < kCl) *cl.map_shared_rank(s_nd, t) = nd ? 1 : 0;
  }
  cl.sync();  // R and the rotate flag are in every CTA
  if (!*s_nd) return;
  if (c1 > c0) {
    ld.issue(S.u.buf[0], (c1 - 1) * kC);
    rotate_pair(c, ld, S.u.buf, S.v.Rs, c0, c1 - c0, t);
  }
}
}  // namespace

// A whole sweep as a persistent launch of kCl-CTA clusters (one pair visit per
// cluster at a time, claimed in gate-group order; dataflow start as in
// jacobi_sweep_kernel: rank 0 waits until both blocks finished the previous
// round, and releases them when every CTA's rotated rows are written).
__global__ void __launch_bounds__(256, 4) jacobi_sweep_cl_kernel(RoundArgs A, const int* __restrict__ glist,
                                                                 int n_list, int group, int max_rounds,
                                                                 int* __restrict__ ctl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PairSmem& S = *reinterpret_cast<PairSmem*>(smem_raw);
  __shared__ long long s_item;
  __shared__ int s_nd;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  int* counter = ctl;
  int* ready = ctl + 1;  // [gate][block]: rounds completed this sweep
  const long long total =
      (long long)((n_list + group - 1) / group) * group * A.max_pairs * max_rounds;
  const int t = threadIdx.x;
  for (;;) {
    if (rank == 0 && t == 0) {
      long long item;
      int gi = 0, round = 0, k = 0;
      for (;;) {
        item = atomicAdd(counter, 1);
        if (item >= total || decode_item(A, glist, n_list, group, max_rounds, item, gi, round, k)) break;
      }
      if (item < total) {
        int ba, bb;
        rr_pair(round, k, A.gates[gi].nb - 1, ba, bb);
        wait_round(ready + gi * 2 * A.max_pairs + ba, round);
        wait_round(ready + gi * 2 * A.max_pairs + bb, round);
      }
#pragma unroll
      for (int r = 0; r < kCl; ++r) *cl.map_shared_rank(&s_item, r) = item;
    }
    cl.sync();  // the item (and, through rank 0's acquire, its blocks) for every CTA
    const long long item = s_item;
    if (item >= total) break;
    int gi, round, k;
    decode_item(A, glist, n_list, group, max_rounds, item, gi, round, k);
    pair_visit_cl(A, gi, round, k, S, &s_nd, rank, cl);
    __syncthreads();
    if (t == 0) __threadfence();
    cl.sync();  // every CTA's rows are written; shared memory is free
    if (rank == 0 && t == 0) {
      int ba, bb;
      rr_pair(round, k, A.gates[gi].nb - 1, ba, bb);
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + gi * 2 * A.max_pairs + ba), "r"(round + 1)
                   : "memory");
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + gi * 2 * A.max_pairs + bb), "r"(round + 1)
                   : "memory");
    }
  }
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
  pair_evd_v1(S.G, S.R, S.sc, t, tol_in, floor_rel2 * frob2[gi], 1, cross_only_evd(active[gi], round));
  __syncthreads();
  cplx* rout = rbuf + slot * (kP * kP);
  for (int idx = t; idx < kP * kP; idx += 256) rout[idx] = S.R[(idx / kP) * kPad + idx % kP];
}

struct RotSmem {
  double buf[2][2 * kChunkPlane];
  cplx Rs[kP * kPitchR];
};

// 3 CTAs x 72 KB per SM.
__global__ void __launch_bounds__(256, 3) jacobi_rot_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                            const int* __restrict__ active, int* __restrict__ rotated,
                                                            int round, const int* __restrict__ perm,
                                                            long long perm_stride, const int* __restrict__ need,
                                                            const cplx* __restrict__ rbuf, int max_pairs) {
  const int gi = blockIdx.y;
  const GateDesc& g = gates[gi];
  PairCtx c;
  if (!pair_ctx(g, gi, round, active, ws, perm, perm_stride, c, blockIdx.x)) return;
  const long long slot = (long long)gi * max_pairs + blockIdx.x;
  if (!need[slot]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RotSmem& S = *reinterpret_cast<RotSmem*>(smem_raw);
  const int t = threadIdx.x;
  ChunkLoader ld;
  ld.init(c, t);
  ld.pol = l2_policy(0);
  const int nchunks = g.m_pad / kC;
  ld.issue(S.buf[0], (nchunks - 1) * kC);
  copy_rotation(rbuf + slot * (kP * kP), kP, S.Rs, t);
  rotate_pair(c, ld, S.buf, S.Rs, 0, nchunks, t);
  if (t == 0) atomicAdd(rotated + gi, 1);
}

#ifdef MPSIM_AB_KNOBS
void jacobi_phase_clocks(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z));
  }
}
#endif

void jacobi_split_init() {
  cudaFuncSetAttribute(jacobi_gram_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PairSmem));
  cudaFuncSetAttribute(jacobi_gram_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PairSmem));
  cudaFuncSetAttribute(jacobi_gram_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PairSmem));
  cudaFuncSetAttribute(jacobi_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PairSmem));
  cudaFuncSetAttribute(jacobi_sweep_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PairSmem));
  cudaFuncSetAttribute(jacobi_evd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EvdSmem));
  cudaFuncSetAttribute(jacobi_rot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RotSmem));
}

static RoundArgs make_args(const GateDesc* d_gates, cplx* ws, const int* d_active, int* d_rotated, double tol,
                           double tol_in, const double* frob2, double floor_rel2, const int* perm,
                           long long perm_stride, double* maxoff, int* need, cplx* gbuf, cplx* rbuf, double* offsum,
                           int max_pairs, cplx* gblk, int probe, int* blkok = nullptr, int l2hint = 0) {
  RoundArgs a;
  a.gates = d_gates;
  a.ws = ws;
  a.active = d_active;
  a.tol = tol;
  a.frob2 = frob2;
  a.floor_rel2 = floor_rel2;
  a.perm = perm;
  a.perm_stride = perm_stride;
  a.maxoff = maxoff;
  a.need = need;
  a.gbuf = gbuf;
  a.max_pairs = max_pairs;
  a.offsum = offsum;
  a.rbuf = rbuf;
  a.tol_in = tol_in;
  a.gblk = gblk;
  a.rotated = d_rotated;
  a.probe = probe;
  a.blkok = blkok;
  a.l2hint = l2hint;
  {
    const char* e = ab_knob("MPSIM_NS_ITERS");
    a.ns_iters = e ? std::atoi(e) : 2;
    const char* x = ab_knob("MPSIM_XTEST");
    a.xtest = x ? std::atoi(x) : kCrossTest;
  }
  return a;
}

// fuse: 0 = three launches, 1 = Gram+EVD / rotation, 2 = one launch per round.
void launch_jacobi_round_split(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                               int* d_rotated, int round, double tol, double tol_in, const double* frob2,
                               double floor_rel2, const int* perm, long long perm_stride, double* maxoff, int* need,
                               cplx* gbuf, cplx* rbuf, double* offsum, int fuse, cplx* gblk, int probe,
                               cudaStream_t st) {
  const dim3 grid(max_pairs, n_gates);
  const size_t sm = sizeof(PairSmem);
  const RoundArgs a = make_args(d_gates, ws, d_active, d_rotated, tol, tol_in, frob2, floor_rel2, perm, perm_stride,
                                maxoff, need, gbuf, rbuf, offsum, max_pairs, gblk, probe);
  if (fuse == 2) {
    jacobi_gram_kernel<2><<<grid, 256, sm, st>>>(a, round);
    return;
  }
  if (fuse == 1) {
    jacobi_gram_kernel<1><<<grid, 256, sm, st>>>(a, round);
  } else {
    jacobi_gram_kernel<0><<<grid, 256, sm, st>>>(a, round);
    jacobi_evd_kernel<<<grid, 256, sizeof(EvdSmem), st>>>(d_gates, d_active, round, tol_in, frob2, floor_rel2, need,
                                                           gbuf, rbuf, max_pairs);
  }
  jacobi_rot_kernel<<<grid, 256, sizeof(RotSmem), st>>>(d_gates, ws, d_active, d_rotated, round, perm, perm_stride,
                                                         need, rbuf, max_pairs);
}

// One whole sweep (all rounds) as a persistent dataflow launch. ctl: 1 +
// n_gates * 2 * max_pairs ints, zeroed here.
void launch_jacobi_sweep(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                         int* d_rotated, double tol, double tol_in, const double* frob2, double floor_rel2,
                         const int* perm, long long perm_stride, double* maxoff, int* need, cplx* gbuf, cplx* rbuf,
                         double* offsum, cplx* gblk, int* ctl, int probe, int l2hint, cudaStream_t st) {
  static int ctas = 0;
  if (ctas == 0) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_sweep_kernel, 256, sizeof(PairSmem));
    ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  // ctl: [item counter | per-block round counters | per-block exact-Gram flags]
  const size_t nblk = (size_t)n_gates * 2 * max_pairs;
  cudaMemsetAsync(ctl, 0, sizeof(int) * (1 + 2 * nblk), st);
  const RoundArgs a = make_args(d_gates, ws, d_active, d_rotated, tol, tol_in, frob2, floor_rel2, perm, perm_stride,
                                maxoff, need, gbuf, rbuf, offsum, max_pairs, gblk, probe, ctl + 1 + nblk, l2hint);
  jacobi_sweep_kernel<<<ctas, 256, sizeof(PairSmem), st>>>(a, n_gates, 2 * max_pairs - 1, ctl);
}

// One whole sweep as a persistent launch of 4-CTA clusters over the gates in
// d_glist (n_list active gates), claimed `group` gates at a time. ctl as for
// launch_jacobi_sweep.
void launch_jacobi_sweep_cl(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                            const int* d_glist, int n_list, int group, int* d_rotated, double tol, double tol_in,
                            const double* frob2, double floor_rel2, const int* perm, long long perm_stride,
                            double* maxoff, int* need, double* offsum, cplx* gblk, int* ctl, cudaStream_t st) {
  static int clusters = 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = sizeof(PairSmem);
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (clusters == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(kCl * sms);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, jacobi_sweep_cl_kernel, &cfg) != cudaSuccess || n < 1) n = sms / kCl;
    clusters = n;
  }
  const size_t nblk = (size_t)n_gates * 2 * max_pairs;
  cudaMemsetAsync(ctl, 0, sizeof(int) * (1 + 2 * nblk), st);
  const RoundArgs a = make_args(d_gates, ws, d_active, d_rotated, tol, tol_in, frob2, floor_rel2, perm, perm_stride,
                                maxoff, need, nullptr, nullptr, offsum, max_pairs, gblk, 0, ctl + 1 + nblk);
  cfg.gridDim = dim3(kCl * clusters);
  cudaLaunchKernelEx(&cfg, jacobi_sweep_cl_kernel, a, d_glist, n_list, group, 2 * max_pairs - 1, ctl);
}

}  // namespace mpsim_gpu
