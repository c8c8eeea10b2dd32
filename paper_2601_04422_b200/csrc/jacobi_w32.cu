// Block one-sided Jacobi with 32-vector blocks (pair visits of 64 vectors):
// the same visit as jacobi_split.cu (DMMA Gram, relative convergence test,
// one cyclic complex Jacobi sweep of the pair Gram, X_P <- X_P R on DMMA) with
// twice the block width, run by one 512-thread CTA per SM as a persistent
// dataflow launch per sweep.
//
// Why: a sweep over n vectors makes (n / W)^2 / 2 pair visits, each streaming
// its 2W vectors through shared memory twice (Gram, rotation) and writing
// them once, so the sweep's HBM traffic is 1.5 (n / W) x the operand. At
// W = 16 that traffic (3 GB per 1024 x 1024 operand per sweep) and the DMMA
// work are of the same size (the kernel sits on the FP64 ridge, about 65 % of
// both); W = 32 halves the traffic at the same DMMA work per sweep, so the
// sweep becomes DMMA-bound. The price is shared memory (the 64 x 64 Gram and
// R: one CTA per SM), so the pair EVD no longer overlaps other CTAs' visits;
// it is a sixth of a visit.
//
// Operand layout as in jacobi_split.cu: vector-major split Re / Im planes of
// m_pad doubles; chunks of 32 rows x 64 vectors stream into vector-major
// shared planes (pitch 36 doubles) with 16-byte cp.async.
#include "common.cuh"
#include "evd.cuh"

namespace mpsim_gpu {

namespace {

constexpr int kW2 = 32;         // vectors per block
constexpr int kP2 = 2 * kW2;    // vectors per pair
constexpr int kT2 = 512;        // threads per CTA
constexpr int kC2 = 32;         // rows per chunk
constexpr int kPitch2 = 36;     // doubles per vector in a chunk plane (== 4 mod 32: conflict-free fragments)
constexpr int kPlane2 = kP2 * kPitch2;     // doubles per chunk plane
constexpr int kStage2 = 2 * kPlane2;       // doubles per chunk stage (Re, Im planes)
constexpr int kLdG = kP2 + 1;              // complex row pitch of G and of the EVD's R
constexpr int kLdR = kP2 + 2;              // complex row pitch of R for the rotation (== 2 mod 8)
constexpr int kGx = 2 * kP2;               // real-extended Gram order (128)
constexpr int kLdGx = kGx + 1;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait_groups() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct Pair2 {
  cplx* X;
  const int* pm;
  long long mp;
  int ba, bb;
  __device__ __forceinline__ double* vec(int i) const {
    const int slot = i < kW2 ? ba * kW2 + i : bb * kW2 + (i - kW2);
    return reinterpret_cast<double*>(X + (long long)pm[slot] * mp);
  }
};

// Per chunk and thread four 16-byte copies: in copy s warp w moves vector
// w + 16 s, lanes 0-15 two rows each of its Re plane, lanes 16-31 of its Im plane.
struct Loader2 {
  const double* src[4];
  int soff;
  __device__ __forceinline__ void init(const Pair2& c, int t) {
    const int lane = t & 31, warp = t >> 5;
    const int rp = lane & 15, plane = lane >> 4;
#pragma unroll
    for (int s = 0; s < 4; ++s) src[s] = c.vec(warp + 16 * s) + plane * c.mp + 2 * rp;
    soff = plane * kPlane2 + warp * kPitch2 + 2 * rp;
  }
  __device__ __forceinline__ void issue(double* buf, int e0) const {
#pragma unroll
    for (int s = 0; s < 4; ++s) cp16(buf + soff + 16 * s * kPitch2, src[s] + e0);
    commit();
  }
};

struct Smem2 {
  union {
    double stage[3][kStage2];  // chunk ring (Gram pass: 3 stages; rotation: stages 2, 0)
    double Gx[kGx * kLdGx];    // real-extended Gram after the pass
    cplx R[kP2 * kLdG];        // the EVD's rotation (Gx is consumed by then)
  } u;
  union {
    cplx G[kP2 * kLdG];
    cplx Rs[kP2 * kLdR];
  } v;
  EvdScratchT<kP2> sc;
  int s_item;
};
static_assert(sizeof(cplx) * kP2 * kLdG <= sizeof(double) * 2 * kStage2, "R must leave stage 2 free");

// column offset (plane + vector) of real-extended column `col` in a chunk stage
// Cross-only Gram passes in three real products: at chi = 1024 +1.5 % (the
// pass is DMMA-bound here, one CTA per SM at the full clock), all parity
// green (profiles/sweep_ab_r02.txt). -DMPSIM_W32_GAUSS=0 restores four.
#ifndef MPSIM_W32_GAUSS
#define MPSIM_W32_GAUSS 1
#endif
constexpr bool kGauss2 = MPSIM_W32_GAUSS;
__device__ __forceinline__ int coff2(int col) { return (col < kP2 ? 0 : kPlane2) + (col & (kP2 - 1)) * kPitch2; }

// Gram pass over all chunks into S.u.Gx: the 64 cross tiles (cross_only) or
// the 136 tiles of the upper real-extended Gram (A and D upper, B full).
__device__ __forceinline__ void gram_pass2(Smem2& S, const Loader2& ld, int nchunks, bool cross_only, int t) {
  const int lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  auto next_chunk = [&](int k) {
    if (k + 1 < nchunks) wait_groups<1>();
    else wait_groups<0>();
    __syncthreads();
    if (k + 2 < nchunks) ld.issue(S.u.stage[(k + 2) % 3], (k + 2) * kC2);
  };
  ld.issue(S.u.stage[0], 0);
  if (nchunks > 1) ld.issue(S.u.stage[1], kC2);
  if (cross_only && kGauss2) {
    // the complex cross block X_a^H X_b in three real products (Gauss):
    // T1 = Ar^T Br, T2 = Ai^T Bi, T3 = (Ar + Ai)^T (Br - Bi); Re = T1 + T2,
    // Im = T1 - T2 - T3: 48 tiles instead of 64. Warp w owns tile position
    // (w >> 2, w & 3) of the 32 x 32 block: four loads and two adds feed three
    // DMMAs per k-step. Re lands in Gx's (Re_a, Re_b) tiles, Im in (Re_a, Im_b).
    const int tr = warp >> 2, tc = warp & 3;
    const int oar = coff2(8 * tr + fr), oai = coff2(kP2 + 8 * tr + fr);
    const int obr = coff2(kW2 + 8 * tc + fr), obi = coff2(kP2 + kW2 + 8 * tc + fr);
    double t1[2] = {0.0, 0.0}, t2[2] = {0.0, 0.0}, t3[2] = {0.0, 0.0};
    for (int k = 0; k < nchunks; ++k) {
      next_chunk(k);
      const double* B = S.u.stage[k % 3];
#pragma unroll
      for (int ks = 0; ks < kC2 / 4; ++ks) {
        const int row = 4 * ks + fk;
        const double ar = B[row + oar], ai = B[row + oai], br = B[row + obr], bi = B[row + obi];
        dmma(t1[0], t1[1], ar, br);
        dmma(t2[0], t2[1], ai, bi);
        dmma(t3[0], t3[1], ar + ai, br - bi);
      }
    }
    __syncthreads();  // the last stage is read; Gx aliases the stages
    double* const row = S.u.Gx + (8 * tr + fr) * kLdGx;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      row[kW2 + 8 * tc + 2 * fk + v] = t1[v] + t2[v];
      row[kP2 + kW2 + 8 * tc + 2 * fk + v] = t1[v] - t2[v] - t3[v];
    }
    __syncthreads();
  } else if (cross_only) {
    // block q of the cross Gram: rows Re_a (tiles 0-3) / Im_a (8-11), columns
    // Re_b (4-7) / Im_b (12-15); warp >> 2 picks the tile row: one A and four
    // B loads feed four DMMAs per k-step
    const int q = warp & 3;
    const int tr = ((q >> 1) ? 8 : 0) + (warp >> 2), tc0 = (q & 1) ? 12 : 4;
    const int oa = coff2(8 * tr + fr);
    int ob[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) ob[i] = coff2(8 * (tc0 + i) + fr);
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int k = 0; k < nchunks; ++k) {
      next_chunk(k);
      const double* B = S.u.stage[k % 3];
#pragma unroll
      for (int ks = 0; ks < kC2 / 4; ++ks) {
        const int row = 4 * ks + fk;
        const double a = B[row + oa];
#pragma unroll
        for (int i = 0; i < 4; ++i) dmma(acc[i][0], acc[i][1], a, B[row + ob[i]]);
      }
    }
    __syncthreads();  // the last stage is read; Gx aliases the stages
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int v = 0; v < 2; ++v) S.u.Gx[(8 * tr + fr) * kLdGx + 8 * (tc0 + i) + 2 * fk + v] = acc[i][v];
    __syncthreads();
  } else {
    // warps 0-7: tile row w of B (tiles (w, 8..15)); warps 8-15: tile row r of
    // A (tiles (r, r..7)) and tile row 15 - r of D (tiles (15 - r, 15 - r..15))
    int trow[9], tcol[9], nt;
    if (warp < 8) {
      nt = 8;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        trow[i] = warp;
        tcol[i] = 8 + (i & 7);
      }
    } else {
      const int r = warp - 8, na = 8 - r;
      nt = 9;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        if (i < na) {
          trow[i] = r;
          tcol[i] = r + i;
        } else {
          trow[i] = 15 - r;
          tcol[i] = 15 - r + (i - na);
        }
      }
    }
    const int oa0 = coff2(8 * trow[0] + fr), oa8 = coff2(8 * trow[8] + fr);
    int ob[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) ob[i] = coff2(8 * tcol[i] + fr);
    double acc[9][2];
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int k = 0; k < nchunks; ++k) {
      next_chunk(k);
      const double* B = S.u.stage[k % 3];
#pragma unroll
      for (int ks = 0; ks < kC2 / 4; ++ks) {
        const int row = 4 * ks + fk;
        const double a_first = B[row + oa0], a_last = B[row + oa8];
#pragma unroll
        for (int i = 0; i < 9; ++i)
          if (i < nt) dmma(acc[i][0], acc[i][1], trow[i] == trow[0] ? a_first : a_last, B[row + ob[i]]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 9; ++i)
      if (i < nt)
#pragma unroll
        for (int v = 0; v < 2; ++v) S.u.Gx[(8 * trow[i] + fr) * kLdGx + 8 * tcol[i] + 2 * fk + v] = acc[i][v];
    __syncthreads();
  }
}

// X_P <- X_P R over all chunks (last to first), three-real-product complex
// multiply on DMMA. Warp w: complex column tile w / 2, row tiles 2 (w & 1) + {0, 1}.
// Chunk k streams through stage 2 (k even; the caller prefetches the first
// there during the EVD) or stage 0 (k odd).
__device__ __forceinline__ void rotate_pair2(const Pair2& c, const Loader2& ld, Smem2& S, int nchunks, int t) {
  const int lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int rbase = 2 * (warp & 1), cj = warp >> 1;
  const int jb = 8 * cj + fr;
  double* const xo[2] = {c.vec(8 * cj + 2 * fk), c.vec(8 * cj + 2 * fk + 1)};
  const cplx* Rs = S.v.Rs;
  for (int k = 0; k < nchunks; ++k) {
    wait_groups<0>();
    __syncthreads();
    if (k + 1 < nchunks) ld.issue(S.u.stage[(k + 1) & 1 ? 0 : 2], (nchunks - 2 - k) * kC2);
    const double* B = S.u.stage[k & 1 ? 0 : 2];
    double t1[2][2], t2[2][2], t3[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a) t1[a][0] = t1[a][1] = t2[a][0] = t2[a][1] = t3[a][0] = t3[a][1] = 0.0;
#pragma unroll
    for (int s = 0; s < kP2 / 4; ++s) {
      const int cc = 4 * s + fk;
      const double* pr = B + cc * kPitch2;
      const double* pim = pr + kPlane2;
      const double ar0 = pr[8 * rbase + fr], ar1 = pr[8 * (rbase + 1) + fr];
      const double ai0 = pim[8 * rbase + fr], ai1 = pim[8 * (rbase + 1) + fr];
      const cplx r = Rs[cc * kLdR + jb];
      const double rs = r.x + r.y;
      dmma(t1[0][0], t1[0][1], ar0, r.x);
      dmma(t1[1][0], t1[1][1], ar1, r.x);
      dmma(t2[0][0], t2[0][1], ai0, r.y);
      dmma(t2[1][0], t2[1][1], ai1, r.y);
      dmma(t3[0][0], t3[0][1], ar0 + ai0, rs);
      dmma(t3[1][0], t3[1][1], ar1 + ai1, rs);
    }
    const int e0 = (nchunks - 1 - k) * kC2;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = 8 * (rbase + a) + fr;
        double* xj = xo[v];
        xj[e0 + e] = t1[a][v] - t2[a][v];
        xj[c.mp + e0 + e] = t3[a][v] - t1[a][v] - t2[a][v];
      }
  }
}

}  // namespace

#ifdef MPSIM_AB_KNOBS
__device__ unsigned long long g_phase_clk2[8];  // as jacobi_split.cu g_phase_clk
#define PHASE_MARK2(var) long long var = clock64()
#define PHASE_ADD2(i, v) \
  if (threadIdx.x == 0) atomicAdd(&g_phase_clk2[i], (unsigned long long)(v))
void jacobi_w32_phase_clocks(unsigned long long* out, bool reset) {
  cudaMemcpyFromSymbol(out, g_phase_clk2, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase_clk2, z, sizeof(z));
  }
}
#else
#define PHASE_MARK2(var)
#define PHASE_ADD2(i, v)
#endif

struct SweepArgs2 {
  const GateDesc* gates;
  cplx* ws;
  const int* active;
  int* rotated;
  double tol, tol_in;
  const double* frob2;
  double floor_rel2;
  const int* perm;
  long long perm_stride;
  double* maxoff;
  double* offsum;
  cplx* gblk;   // [gate][block] 32 x 32 in-block Grams
  int* blkok;   // [gate][block] exact-cache flags
  int max_pairs;
};

__device__ __forceinline__ bool cross_only_evd2(int active, int round) {
  if (active & 2) return true;
  if (!(active & 16)) return false;
  return round % ((active & 32) ? 3 : 2) != 0;
}

// One pair visit (block pair k of gate gi in tournament round `round`).
__device__ __forceinline__ void pair_visit2(const SweepArgs2& A, int gi, int round, int k, Smem2& S) {
  const GateDesc& g = A.gates[gi];
  const int nb = g.n_pad / kW2;
  Pair2 c;
  rr_pair(round, k, nb - 1, c.ba, c.bb);
  c.X = A.ws + g.ws_off;
  c.pm = A.perm + gi * A.perm_stride;
  c.mp = g.m_pad;
  const int t = threadIdx.x;
  Loader2 ld;
  ld.init(c, t);
  const int act = A.active[gi];
  // stored in-block Grams (bit 4, rounds > 0 of a pre-asymptotic sweep) or the
  // exact cache (bit 8): see jacobi_split.cu pair_visit
  const bool approx = (act & 4) && round > 0;
  int* const ok_a = A.blkok + (long long)gi * 2 * A.max_pairs + c.ba;
  int* const ok_b = A.blkok + (long long)gi * 2 * A.max_pairs + c.bb;
  const bool cached = !approx && (act & 8) && round > 0 && *ok_a && *ok_b;
  const bool cross_only = approx || cached;
  cplx* const gblk_a = A.gblk + ((long long)gi * 2 * A.max_pairs + c.ba) * (kW2 * kW2);
  cplx* const gblk_b = A.gblk + ((long long)gi * 2 * A.max_pairs + c.bb) * (kW2 * kW2);
  const int nchunks = g.m_pad / kC2;
  PHASE_MARK2(c_g0);
  gram_pass2(S, ld, nchunks, cross_only, t);
  PHASE_MARK2(c_g1);
  PHASE_ADD2(2, c_g1 - c_g0);
  cplx* const SG = S.v.G;
  const double* Gx = S.u.Gx;
  if (cross_only) {
    for (int idx = t; idx < kW2 * kW2; idx += kT2) {
      const int i = idx / kW2, j = kW2 + idx % kW2;
      const double re = kGauss2 ? Gx[i * kLdGx + j] : Gx[i * kLdGx + j] + Gx[(kP2 + i) * kLdGx + kP2 + j];
      const double im = kGauss2 ? Gx[i * kLdGx + kP2 + j] : Gx[i * kLdGx + kP2 + j] - Gx[(kP2 + i) * kLdGx + j];
      SG[i * kLdG + j] = make_double2(re, im);
      SG[j * kLdG + i] = make_double2(re, -im);
      const int r = idx / kW2, q = idx % kW2;
      SG[r * kLdG + q] = gblk_a[idx];
      SG[(kW2 + r) * kLdG + kW2 + q] = gblk_b[idx];
    }
  } else {
    for (int idx = t; idx < kP2 * kP2; idx += kT2) {
      const int i = idx / kP2, j = idx % kP2;
      if (i > j) continue;
      const double re = Gx[i * kLdGx + j] + Gx[(kP2 + i) * kLdGx + kP2 + j];
      const double im = Gx[i * kLdGx + kP2 + j] - Gx[j * kLdGx + kP2 + i];
      SG[i * kLdG + j] = make_double2(re, i == j ? 0.0 : im);
      if (i != j) SG[j * kLdG + i] = make_double2(re, -im);
    }
  }
  __syncthreads();
  const double tolg = A.tol * fmax(sqrt((double)g.m), (double)kP);  // the W = 16 test's threshold
  const double floor2 = A.floor_rel2 * A.frob2[gi];
  double rx = 0.0;   // this thread's largest squared relative cross off-diagonal
  bool xneed = false;  // ... above the rotation threshold
  {
    // sum of squared relative off-diagonals between the two blocks (rms policy)
    double r = 0.0;
    const double tolg2 = tolg * tolg;
    for (int idx = t; idx < kW2 * kW2; idx += kT2) {
      const int i = idx / kW2, j = kW2 + idx % kW2;
      const double gii = SG[i * kLdG + i].x, gjj = SG[j * kLdG + j].x;
      if (fmin(gii, gjj) > floor2) {
        const double c2 = cabs2(SG[i * kLdG + j]), d = gii * gjj;
        const double q = (d < 1e30 && d > 1e-12) ? (double)__fdividef((float)c2, (float)d) : c2 / d;
        r += q;
        rx = fmax(rx, q);
        xneed |= c2 > tolg2 * d;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if ((t & 31) == 0 && r > 0.0) atomicAdd(A.offsum + gi, r);
  }
  bool nd;
  if (approx) {
    // pre-asymptotic visit: the in-block Grams are the cached EVD output, so
    // the test and maxoff use the cross entries only (as jacobi_split.cu)
    double mx = rx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0 && mx > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(A.maxoff + gi),
                (unsigned long long)__double_as_longlong(sqrt(mx)));
    nd = __syncthreads_or(xneed);
  } else {
    nd = pair_needs_rotation_t<kP2, kLdG, kT2>(SG, t, tolg, floor2, A.maxoff + gi);
  }
  PHASE_MARK2(c_a1);
  PHASE_ADD2(3, c_a1 - c_g1);
  auto store_inblock = [&]() {
    for (int idx = t; idx < kW2 * kW2; idx += kT2) {
      const int r = idx / kW2, q = idx % kW2;
      gblk_a[idx] = SG[r * kLdG + q];
      gblk_b[idx] = SG[(kW2 + r) * kLdG + kW2 + q];
    }
  };
  if (!nd) {
    if (!cross_only) {
      store_inblock();
      if (t == 0) *ok_a = *ok_b = 1;
    }
    return;
  }
  if (t == 0) *ok_a = *ok_b = 0;
  // the rotation's first chunk (the pass's last) loads into stage 2 during the EVD
  ld.issue(S.u.stage[2], (nchunks - 1) * kC2);
  pair_evd_t<kP2, kLdG, kT2, 1>(SG, S.u.R, S.sc, t, A.tol_in, floor2, 1, cross_only_evd2(act, round));
  __syncthreads();
  PHASE_MARK2(c_e1);
  PHASE_ADD2(4, c_e1 - c_a1);
  PHASE_ADD2(7, 1);
  store_inblock();
  __syncthreads();  // G (aliased by Rs) has been stored
  for (int idx = t; idx < kP2 * kP2; idx += kT2) {
    const int i = idx / kP2, j = idx % kP2;
    S.v.Rs[i * kLdR + j] = S.u.R[i * kLdG + j];
  }
  __syncthreads();  // R (aliased by stage 0) has been read
  rotate_pair2(c, ld, S, nchunks, t);
  PHASE_MARK2(c_r1);
  PHASE_ADD2(5, c_r1 - c_e1);
  if (t == 0) atomicAdd(A.rotated + gi, 1);
}

// A whole sweep in one persistent launch (one CTA per SM): CTAs claim pair
// visits in (round, gate, pair) order and start one when both of its blocks
// have finished the previous round (see jacobi_split.cu jacobi_sweep_kernel).
__global__ void __launch_bounds__(kT2, 1) jacobi_sweep_w32_kernel(SweepArgs2 A, int n_gates, int max_rounds,
                                                                   int* __restrict__ ctl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem2& S = *reinterpret_cast<Smem2*>(smem_raw);
  int* counter = ctl;
  int* ready = ctl + 1;  // [gate][block]: rounds completed this sweep
  const int per_round = n_gates * A.max_pairs;
  const long long total = (long long)per_round * max_rounds;
  const int t = threadIdx.x;
  for (;;) {
    __syncthreads();  // shared memory of the previous visit is free
    if (t == 0) S.s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int item = S.s_item;
    if (item >= total) break;
    const int round = item / per_round, rem = item % per_round;
    const int gi = rem / A.max_pairs, k = rem % A.max_pairs;
    const GateDesc& g = A.gates[gi];
    const int nb = g.n_pad / kW2;
    if (!A.active[gi] || round >= nb - 1 || k >= nb / 2) continue;
    int ba, bb;
    rr_pair(round, k, nb - 1, ba, bb);
    int* ra = ready + gi * 2 * A.max_pairs + ba;
    int* rb = ready + gi * 2 * A.max_pairs + bb;
    PHASE_MARK2(c_w0);
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
    PHASE_MARK2(c_w1);
    PHASE_ADD2(1, c_w1 - c_w0);
    pair_visit2(A, gi, round, k, S);
    __syncthreads();  // every thread's writes of this visit are issued
    PHASE_MARK2(c_v1);
    PHASE_ADD2(0, c_v1 - c_w0);
    PHASE_ADD2(6, 1);
    if (t == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ra), "r"(round + 1) : "memory");
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(rb), "r"(round + 1) : "memory");
    }
  }
}

// One sweep of the W = 32 Jacobi over the gates (every n_pad a multiple of
// 64): max_pairs = max(n_pad) / 64; ctl: 1 + 2 * n_gates * 2 * max_pairs ints
// (zeroed here); gblk: n_gates * 2 * max_pairs * 32 * 32 complex.
void launch_jacobi_sweep_w32(const GateDesc* d_gates, int n_gates, int max_pairs, cplx* ws, const int* d_active,
                             int* d_rotated, double tol, double tol_in, const double* frob2, double floor_rel2,
                             const int* perm, long long perm_stride, double* maxoff, double* offsum, cplx* gblk,
                             int* ctl, cudaStream_t st) {
  static int ctas = 0;
  if (ctas == 0) {
    cudaFuncSetAttribute(jacobi_sweep_w32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem2));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_sweep_w32_kernel, kT2, sizeof(Smem2));
    ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  const size_t nblk = (size_t)n_gates * 2 * max_pairs;
  cudaMemsetAsync(ctl, 0, sizeof(int) * (1 + 2 * nblk), st);
  SweepArgs2 a;
  a.gates = d_gates;
  a.ws = ws;
  a.active = d_active;
  a.rotated = d_rotated;
  a.tol = tol;
  a.tol_in = tol_in;
  a.frob2 = frob2;
  a.floor_rel2 = floor_rel2;
  a.perm = perm;
  a.perm_stride = perm_stride;
  a.maxoff = maxoff;
  a.offsum = offsum;
  a.gblk = gblk;
  a.blkok = ctl + 1 + nblk;
  a.max_pairs = max_pairs;
  jacobi_sweep_w32_kernel<<<ctas, kT2, sizeof(Smem2), st>>>(a, n_gates, 2 * max_pairs - 1, ctl);
}

size_t jacobi_w32_smem() { return sizeof(Smem2); }

}  // namespace mpsim_gpu
