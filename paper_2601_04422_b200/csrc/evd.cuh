// Shared pieces of the block-Jacobi pair step: the relative convergence test
// on a 2W x 2W complex Gram block and one cyclic complex Jacobi EVD of it
// (see jacobi.cu for the algorithm notes). 256-thread CTAs, kP = 32.
//
// Per step of the parallel (round-robin) ordering the 16 disjoint rotations
// J_k = [[cs, sn], [-ph sn, ph cs]] are applied in ONE pass: thread (a, b)
// owns the 2x2 block of G at (pair a rows, pair b cols) and computes
// J_a^H G_ab J_b, plus rows (p_a, q_a) x cols (p_b, q_b) of R <- R J. Blocks
// are disjoint, so a step costs two barriers.
//
// The rotation angle t is computed in FP32 (fast SFU ops); cs = 1/sqrt(1+t^2),
// sn = cs t and the phase ph = conj(g)/|g| are formed in FP64, so every J is
// unitary to FP64 rounding whatever the angle's accuracy. An angle accurate to
// ~1e-7 only means a rotated off-diagonal is reduced by ~1e-7 instead of to
// zero; the outer sweeps keep rotating a pair until the FP64 test passes.
#pragma once

#include "common.cuh"

// Pair-EVD G update of the 256-thread (16-vector block) sweeps: 0 = every
// (row pair, column pair) block, 2 = Hermitian-folded (pair_evd_t kSym)
#ifndef MPSIM_EVD_FOLD
#define MPSIM_EVD_FOLD 0
#endif

namespace mpsim_gpu {

template <int kPP>
struct EvdScratchT {
  double cs[kPP / 2], sn[kPP / 2];
  cplx ph[kPP / 2];
  float csf[kPP / 2], snf[kPP / 2];
  float2 phf[kPP / 2];
  int pp[kPP / 2], pq[kPP / 2];
  int any;
};
using EvdScratch = EvdScratchT<kP>;

__device__ __forceinline__ void rr_pair(int step, int k, int M, int& a, int& b) {
  // Round-robin tournament over M+1 players (M odd); player M is fixed.
  if (k == 0) {
    a = step;
    b = M;
  } else {
    a = (step + k) % M;
    b = (step - k + M) % M;
  }
}

// True if any off-diagonal |G_ij| > tolg sqrt(G_ii G_jj) among columns above
// the noise floor. All 256 threads must call it. If maxoff != nullptr the
// largest relative off-diagonal of the block is folded into *maxoff
// (atomicMax on the bit pattern: non-negative doubles order as integers).
// (kPP x kPP Gram with row pitch kLd, kT threads; kPP^2 / 4 must be a multiple of kT)
template <int kPP, int kLd, int kT>
__device__ __forceinline__ bool pair_needs_rotation_t(const cplx* G, int t, double tolg, double floor2,
                                                      double* maxoff = nullptr) {
  // |G_ij|^2 > tolg^2 G_ii G_jj in FP64 without square roots or divisions
  // (the FP64 units are shared with the other CTAs' DMMA); the squared ratio
  // for maxoff, which only steers sweep policy, in FP32 when in range
  bool need = false;
  float mx2 = 0.0f;
  double mx2d = 0.0;
  const double tolg2 = tolg * tolg;
#pragma unroll
  for (int h = 0; h < (kPP * kPP / 4) / kT; ++h) {
    const int blk = t + h * kT;
    const int ip = blk / (kPP / 2), jp = blk % (kPP / 2);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = 2 * ip + a, j = 2 * jp + b;
        if (i < j) {
          const double g2 = cabs2(G[i * kLd + j]);
          const double gii = G[i * kLd + i].x, gjj = G[j * kLd + j].x;
          if (g2 > 0.0 && fmin(gii, gjj) > floor2) {
            const double d = gii * gjj;
            if (g2 > tolg2 * d) need = true;
            if (maxoff != nullptr) {
              // FP32 when d is in (1e-12, 1e30): g2 <= d, and a g2 below
              // FP32's normal range then means a squared ratio < 1e-26, under
              // every threshold the host applies (the smallest: 1e-24)
              if (d < 1e30 && d > 1e-12)
                mx2 = fmaxf(mx2, __fdividef((float)g2, (float)d));
              else
                mx2d = fmax(mx2d, g2 / d);
            }
          }
        }
      }
  }
  if (maxoff != nullptr) {
    double mx = sqrt(fmax((double)mx2, mx2d));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0 && mx > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(maxoff), (unsigned long long)__double_as_longlong(mx));
  }
  return __syncthreads_or(need);
}
__device__ __forceinline__ bool pair_needs_rotation(const cplx* G, int t, double tolg, double floor2,
                                                    double* maxoff = nullptr) {
  return pair_needs_rotation_t<kP, kPad, 256>(G, t, tolg, floor2, maxoff);
}

// Two barriers per step: 16 threads form the parameters, then all 256 update.
// cross = true: one pass over the 256 pairs (i < W <= j) that straddle the two
// blocks only, 16 steps of pairs (i, W + (i + step) % W) instead of 31 steps
// over all 496 pairs. Used in the pre-asymptotic outer sweeps (engine.cu),
// where the in-block pairs are near-orthogonal from their previous visits.
// kPP x kPP Hermitian G and R (row pitch kLd), kT threads; each thread owns
// (kPP / 2)^2 / kT (row pair, column pair) blocks per step.
// kSym: only the (row pair, column pair) blocks with ba <= bb of G are formed
// and mirrored (fewer FP64 instructions; measured +0.8 % for the 512-thread
// 64 x 64 EVD of jacobi_w32.cu, where the update is FP64-throughput-bound; the
// 256-thread 32 x 32 EVD keeps the full update: the split loops spill there).
template <int kPP, int kLd, int kT, int kSym = 0>
__device__ __forceinline__ void pair_evd_t(cplx* G, cplx* R, EvdScratchT<kPP>& S, int t, double tol_in,
                                           double floor2, int max_in, bool cross = false) {
  constexpr int kH = kPP / 2;
  constexpr int kBlk = kH * kH / kT;
  static_assert(kH * kH % kT == 0, "blocks per thread");
  for (int idx = t; idx < kPP * kPP; idx += kT) {
    const int i = idx / kPP, j = idx % kPP;
    R[i * kLd + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  }
  if (t < kPP) G[t * kLd + t].y = 0.0;
  const double tol2 = tol_in * tol_in;
  __syncthreads();
  for (int sweep = 0; sweep < max_in; ++sweep) {
    if (t == 0) S.any = 0;
    __syncthreads();
    const int nsteps = cross ? kH : kPP - 1;
    for (int step = 0; step < nsteps; ++step) {
      if (t < kH) {
        int p, q;
        if (cross) {
          p = t;
          q = kH + (t + step) % kH;
        } else {
          rr_pair(step, t, kPP - 1, p, q);
        }
        const double a = G[p * kLd + p].x, b = G[q * kLd + q].x;
        const cplx g = G[p * kLd + q];
        const double c2 = cabs2(g);
        double cs = 1.0, sn = 0.0;
        cplx ph = make_double2(1.0, 0.0);
        if (c2 > 0.0 && c2 > tol2 * fabs(a * b) && fmin(a, b) > floor2) {
          const double inv_c = rsqrt(c2);
          ph = make_double2(g.x * inv_c, -g.y * inv_c);  // e^{-i phi}, |ph| = 1 to rounding
          const float zf = (float)((b - a) * 0.5 * inv_c);
          const float az = fabsf(zf);
          const float tf = copysignf(1.0f, zf) / (az > 1e18f ? 2.0f * az : az + sqrtf(1.0f + zf * zf));
          const double tt = (double)tf;
          cs = rsqrt(1.0 + tt * tt);
          sn = cs * tt;
          S.any = 1;
        }
        S.cs[t] = cs;
        S.sn[t] = sn;
        S.ph[t] = ph;
        S.pp[t] = p;
        S.pq[t] = q;
      }
      __syncthreads();
      if constexpr (kSym == 2) {
        // one (row pair, column pair) block per thread, G kept exactly
        // Hermitian: threads [0, kNU) take the blocks ba <= bb (folded as in
        // kSym == 1) and update G (+ its mirror) and R; the others take the
        // blocks ba > bb and update R only, so whole warps skip the G update
        static_assert(kBlk == 1 && kH % 2 == 0, "one block per thread");
        constexpr int kNU = kH * (kH + 1) / 2;
        int ba, bb;
        const bool doG = t < kNU;
        if (doG) {
          const int fi = t / (kH + 1), fj = t % (kH + 1);
          ba = fj < kH - fi ? fi : kH - 1 - fi;
          bb = fj < kH - fi ? fi + fj : kH - 1 - fi + (fj - (kH - fi));
        } else {  // strictly upper (a < b) folded: rows a and kH - 2 - a share a row of kH
          const int u = t - kNU, fi = u / kH, fj = u % kH;
          int a, b;
          if (fj < kH - 1 - fi) {
            a = fi;
            b = fi + 1 + fj;
          } else {
            a = kH - 2 - fi;
            b = kH - 1 - fi + (fj - (kH - 1 - fi));
          }
          ba = b;
          bb = a;
        }
        const double csa = S.cs[ba], sna = S.sn[ba], csb = S.cs[bb], snb = S.sn[bb];
        int pa, qa, pb, qb;
        if (cross) {
          pa = ba;
          qa = kH + (ba + step) % kH;
          pb = bb;
          qb = kH + (bb + step) % kH;
        } else {
          rr_pair(step, ba, kPP - 1, pa, qa);
          rr_pair(step, bb, kPP - 1, pb, qb);
        }
        const cplx phb = S.ph[bb];
        const cplx jb_qp = make_double2(-phb.x * snb, -phb.y * snb), jb_qq = make_double2(phb.x * csb, phb.y * csb);
        if (doG && (sna != 0.0 || snb != 0.0)) {
          const cplx pha = S.ph[ba];
          const cplx ca_qp = make_double2(-pha.x * sna, pha.y * sna), ca_qq = make_double2(pha.x * csa, -pha.y * csa);
          const cplx b00 = G[pa * kLd + pb], b01 = G[pa * kLd + qb], b10 = G[qa * kLd + pb], b11 = G[qa * kLd + qb];
          cplx m00 = make_double2(csa * b00.x, csa * b00.y), m01 = make_double2(csa * b01.x, csa * b01.y);
          cplx m10 = make_double2(sna * b00.x, sna * b00.y), m11 = make_double2(sna * b01.x, sna * b01.y);
          cfma(m00, ca_qp, b10);
          cfma(m01, ca_qp, b11);
          cfma(m10, ca_qq, b10);
          cfma(m11, ca_qq, b11);
          cplx n00 = make_double2(csb * m00.x, csb * m00.y), n01 = make_double2(snb * m00.x, snb * m00.y);
          cplx n10 = make_double2(csb * m10.x, csb * m10.y), n11 = make_double2(snb * m10.x, snb * m10.y);
          cfma(n00, m01, jb_qp);
          cfma(n01, m01, jb_qq);
          cfma(n10, m11, jb_qp);
          cfma(n11, m11, jb_qq);
          if (ba == bb) {
            n00.y = 0.0;
            n11.y = 0.0;
            n01 = make_double2(0.0, 0.0);
            n10 = make_double2(0.0, 0.0);
          }
          G[pa * kLd + pb] = n00;
          G[pa * kLd + qb] = n01;
          G[qa * kLd + pb] = n10;
          G[qa * kLd + qb] = n11;
          if (ba != bb) {
            G[pb * kLd + pa] = make_double2(n00.x, -n00.y);
            G[qb * kLd + pa] = make_double2(n01.x, -n01.y);
            G[pb * kLd + qa] = make_double2(n10.x, -n10.y);
            G[qb * kLd + qa] = make_double2(n11.x, -n11.y);
          }
        }
        if (snb != 0.0) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int row = r == 0 ? pa : qa;
            const cplx x0 = R[row * kLd + pb], x1 = R[row * kLd + qb];
            cplx y0 = make_double2(csb * x0.x, csb * x0.y), y1 = make_double2(snb * x0.x, snb * x0.y);
            cfma(y0, x1, jb_qp);
            cfma(y1, x1, jb_qq);
            R[row * kLd + pb] = y0;
            R[row * kLd + qb] = y1;
          }
        }
      } else if constexpr (kSym == 1) {
      // G stays exactly Hermitian: only the (row pair, column pair) blocks with
      // ba <= bb are formed — kH (kH + 1) / 2 of them, folded into kH / 2 rows
      // of kH + 1 so whole warps drop out — and each off-diagonal block is
      // stored with its conjugate transpose
      constexpr int kNU = kH * (kH + 1) / 2;
#pragma unroll
      for (int hb = 0; hb < (kNU + kT - 1) / kT; ++hb) {
        const int u = t + hb * kT;
        if (u < kNU) {
          const int fi = u / (kH + 1), fj = u % (kH + 1);
          const int ba = fj < kH - fi ? fi : kH - 1 - fi;
          const int bb = fj < kH - fi ? fi + fj : kH - 1 - fi + (fj - (kH - fi));
          const double csa = S.cs[ba], sna = S.sn[ba], csb = S.cs[bb], snb = S.sn[bb];
          if (sna != 0.0 || snb != 0.0) {
            int pa, qa, pb, qb;
            if (cross) {
              pa = ba;
              qa = kH + (ba + step) % kH;
              pb = bb;
              qb = kH + (bb + step) % kH;
            } else {
              rr_pair(step, ba, kPP - 1, pa, qa);
              rr_pair(step, bb, kPP - 1, pb, qb);
            }
            const cplx pha = S.ph[ba], phb = S.ph[bb];
            const cplx jb_qp = make_double2(-phb.x * snb, -phb.y * snb), jb_qq = make_double2(phb.x * csb, phb.y * csb);
            const cplx ca_qp = make_double2(-pha.x * sna, pha.y * sna), ca_qq = make_double2(pha.x * csa, -pha.y * csa);
            const cplx b00 = G[pa * kLd + pb], b01 = G[pa * kLd + qb], b10 = G[qa * kLd + pb], b11 = G[qa * kLd + qb];
            cplx m00 = make_double2(csa * b00.x, csa * b00.y), m01 = make_double2(csa * b01.x, csa * b01.y);
            cplx m10 = make_double2(sna * b00.x, sna * b00.y), m11 = make_double2(sna * b01.x, sna * b01.y);
            cfma(m00, ca_qp, b10);
            cfma(m01, ca_qp, b11);
            cfma(m10, ca_qq, b10);
            cfma(m11, ca_qq, b11);
            cplx n00 = make_double2(csb * m00.x, csb * m00.y), n01 = make_double2(snb * m00.x, snb * m00.y);
            cplx n10 = make_double2(csb * m10.x, csb * m10.y), n11 = make_double2(snb * m10.x, snb * m10.y);
            cfma(n00, m01, jb_qp);
            cfma(n01, m01, jb_qq);
            cfma(n10, m11, jb_qp);
            cfma(n11, m11, jb_qq);
            if (ba == bb) {
              n00.y = 0.0;
              n11.y = 0.0;
              n01 = make_double2(0.0, 0.0);
              n10 = make_double2(0.0, 0.0);
            }
            G[pa * kLd + pb] = n00;
            G[pa * kLd + qb] = n01;
            G[qa * kLd + pb] = n10;
            G[qa * kLd + qb] = n11;
            if (ba != bb) {
              G[pb * kLd + pa] = make_double2(n00.x, -n00.y);
              G[qb * kLd + pa] = make_double2(n01.x, -n01.y);
              G[pb * kLd + qa] = make_double2(n10.x, -n10.y);
              G[qb * kLd + qa] = make_double2(n11.x, -n11.y);
            }
          }
        }
      }
      // R <- R J_b on rows (pa, qa), columns (pb, qb): every block
#pragma unroll
      for (int hb = 0; hb < kBlk; ++hb) {
        const int ba = (t + hb * kT) / kH, bb = (t + hb * kT) % kH;
        const double csb = S.cs[bb], snb = S.sn[bb];
        if (snb != 0.0) {
          int pa, qa, pb, qb;
          if (cross) {
            pa = ba;
            qa = kH + (ba + step) % kH;
            pb = bb;
            qb = kH + (bb + step) % kH;
          } else {
            rr_pair(step, ba, kPP - 1, pa, qa);
            rr_pair(step, bb, kPP - 1, pb, qb);
          }
          const cplx phb = S.ph[bb];
          const cplx jb_qp = make_double2(-phb.x * snb, -phb.y * snb), jb_qq = make_double2(phb.x * csb, phb.y * csb);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int row = r == 0 ? pa : qa;
            const cplx x0 = R[row * kLd + pb], x1 = R[row * kLd + qb];
            cplx y0 = make_double2(csb * x0.x, csb * x0.y), y1 = make_double2(snb * x0.x, snb * x0.y);
            cfma(y0, x1, jb_qp);
            cfma(y1, x1, jb_qq);
            R[row * kLd + pb] = y0;
            R[row * kLd + qb] = y1;
          }
        }
      }
      } else {
#pragma unroll
      for (int hb = 0; hb < kBlk; ++hb) {
      const int ba = (t + hb * kT) / kH, bb = (t + hb * kT) % kH;  // this thread's (row pair, column pair)
      const double csa = S.cs[ba], sna = S.sn[ba], csb = S.cs[bb], snb = S.sn[bb];
      if (sna != 0.0 || snb != 0.0) {
        // the step's pairs ba and bb, recomputed (no shared-memory round trip
        // in front of the Gram loads)
        int pa, qa, pb, qb;
        if (cross) {
          pa = ba;
          qa = kH + (ba + step) % kH;
          pb = bb;
          qb = kH + (bb + step) % kH;
        } else {
          rr_pair(step, ba, kPP - 1, pa, qa);
          rr_pair(step, bb, kPP - 1, pb, qb);
        }
        const cplx pha = S.ph[ba], phb = S.ph[bb];
        // J entries: Jpp = cs, Jpq = sn, Jqp = -ph sn, Jqq = ph cs
        const cplx jb_qp = make_double2(-phb.x * snb, -phb.y * snb), jb_qq = make_double2(phb.x * csb, phb.y * csb);
        // conj(J_a) entries used on the left: conj(Jpp)=cs, conj(Jqp)=-conj(ph) sn, conj(Jpq)=sn, conj(Jqq)=conj(ph) cs
        const cplx ca_qp = make_double2(-pha.x * sna, pha.y * sna), ca_qq = make_double2(pha.x * csa, -pha.y * csa);
        const cplx b00 = G[pa * kLd + pb], b01 = G[pa * kLd + qb], b10 = G[qa * kLd + pb], b11 = G[qa * kLd + qb];
        // M = J_a^H B
        cplx m00 = make_double2(csa * b00.x, csa * b00.y), m01 = make_double2(csa * b01.x, csa * b01.y);
        cplx m10 = make_double2(sna * b00.x, sna * b00.y), m11 = make_double2(sna * b01.x, sna * b01.y);
        cfma(m00, ca_qp, b10);
        cfma(m01, ca_qp, b11);
        cfma(m10, ca_qq, b10);
        cfma(m11, ca_qq, b11);
        // N = M J_b
        cplx n00 = make_double2(csb * m00.x, csb * m00.y), n01 = make_double2(snb * m00.x, snb * m00.y);
        cplx n10 = make_double2(csb * m10.x, csb * m10.y), n11 = make_double2(snb * m10.x, snb * m10.y);
        cfma(n00, m01, jb_qp);
        cfma(n01, m01, jb_qq);
        cfma(n10, m11, jb_qp);
        cfma(n11, m11, jb_qq);
        if (ba == bb) {  // the rotated pair itself: exact zeros off the diagonal, real diagonal
          n00.y = 0.0;
          n11.y = 0.0;
          n01 = make_double2(0.0, 0.0);
          n10 = make_double2(0.0, 0.0);
        }
        G[pa * kLd + pb] = n00;
        G[pa * kLd + qb] = n01;
        G[qa * kLd + pb] = n10;
        G[qa * kLd + qb] = n11;
        if (snb != 0.0) {  // R <- R J_b on rows (pa, qa), columns (pb, qb)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int row = r == 0 ? pa : qa;
            const cplx x0 = R[row * kLd + pb], x1 = R[row * kLd + qb];
            cplx y0 = make_double2(csb * x0.x, csb * x0.y), y1 = make_double2(snb * x0.x, snb * x0.y);
            cfma(y0, x1, jb_qp);
            cfma(y1, x1, jb_qq);
            R[row * kLd + pb] = y0;
            R[row * kLd + qb] = y1;
          }
        }
      }
      }
      }
      __syncthreads();
    }
    const int any = S.any;
    __syncthreads();
    if (!any) break;
  }
}
// Pre-asymptotic inner sweep, FP32 throughout, then an exactly unitary R.
//
// Measured (A/B build, SM clocks per visit at chi=512): the FP64 inner sweep
// takes ~38 % of a visit (135-180k cycles) although it is ~2 % of the visit's
// FP64 work: DMMA executes on the FP64 units (37.1 vs 33.9 TF/s peaks), so
// while the other CTAs of the SM rotate, every dependent FP64 instruction of
// the EVD queues behind their DMMAs. Here the sweep's dependent chain is FP32
// only (its own, idle pipe): G32 and R32 in FP32, the angles in FP32. R32 is
// unitary to ~1e-7; R is its polar factor, two Newton-Schulz steps in FP64
// on DMMA (R <- R (3 I - R^H R) / 2: 1e-7 -> 1e-14 -> 1e-28), i.e. unitary
// to FP64 rounding like the FP64 sweep's R. The rotation R applies differs
// from the exact inner-sweep rotation by ~1e-7 — irrelevant while the pair's
// relative off-diagonals are >> 1e-7 (the host runs this only in sweeps whose
// predecessor measured a largest relative off-diagonal above 1e-2).
// Exact zeros survive: a zero vector's Gram row is zero, it is never rotated,
// so its rows and columns of R32, R^H R and R stay those of the identity.
//
// Buffers (256 threads): G (FP64, kP x kPad, holds the pair Gram on entry; used
// as scratch for R^H R afterwards), W (FP64, kP x kPad: G32 and R32 as float2
// on entry to the polar step, then one NS iterate), R (FP64 output, kP x kPad).
// store_inblock(G32) runs while G32 is alive (FP32-accurate in-block Grams).

// C = op(A) B for 32 x 32 complex matrices in shared memory (pitch kPad),
// op = conjugate transpose if ah; on DMMA with the three-real-product complex
// multiply (T1 = Ar Br, T2 = Ai Bi, T3 = (Ar + Ai)(Br + Bi)); warp w computes
// output tiles (w >> 1, 2 (w & 1) + {0, 1}); herm: only tiles on or above the
// diagonal (C Hermitian; the caller mirrors). C must not alias A or B.
__device__ __forceinline__ void gemm32c(const cplx* A, const cplx* B, cplx* C, bool ah, bool herm, int t) {
  const int lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int tr = warp >> 1, tc0 = 2 * (warp & 1);
  if (herm && tr > tc0 + 1) return;
  double t1[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, t2[2][2] = {{0.0, 0.0}, {0.0, 0.0}},
         t3[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < kP / 4; ++kk) {
    const int k = 4 * kk + fk, i = 8 * tr + fr;
    cplx a = ah ? A[k * kPad + i] : A[i * kPad + k];
    if (ah) a.y = -a.y;
    const double as = a.x + a.y;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const cplx b = B[k * kPad + 8 * (tc0 + c) + fr];
      const double bs = b.x + b.y;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(t1[c][0]), "+d"(t1[c][1]) : "d"(a.x), "d"(b.x));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(t2[c][0]), "+d"(t2[c][1]) : "d"(a.y), "d"(b.y));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(t3[c][0]), "+d"(t3[c][1]) : "d"(as), "d"(bs));
    }
  }
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int v = 0; v < 2; ++v)
      C[(8 * tr + fr) * kPad + 8 * (tc0 + c) + 2 * fk + v] =
          make_double2(t1[c][v] - t2[c][v], t3[c][v] - t1[c][v] - t2[c][v]);
}

template <typename StoreInblock>
__device__ __forceinline__ void pair_evd_f32(cplx* G, cplx* W, cplx* R, EvdScratch& S, int t, double floor2,
                                             bool cross, StoreInblock store_inblock, int ns_iters = 2) {
  float2* const G32 = reinterpret_cast<float2*>(W);
  float2* const R32 = G32 + kP * kPad;
  static_assert(2 * sizeof(float2) <= sizeof(cplx), "G32 and R32 share W");
  for (int idx = t; idx < kP * kP; idx += 256) {
    const int i = idx / kP, j = idx % kP;
    const cplx g = G[i * kPad + j];
    G32[i * kPad + j] = make_float2((float)g.x, i == j ? 0.0f : (float)g.y);
    R32[i * kPad + j] = make_float2(i == j ? 1.0f : 0.0f, 0.0f);
  }
  const float floor2f = (float)floor2;
  const int ba = t / (kP / 2), bb = t % (kP / 2);
  __syncthreads();
  const int nsteps = cross ? kP / 2 : kP - 1;
  for (int step = 0; step < nsteps; ++step) {
    if (t < kP / 2) {
      int p, q;
      if (cross) {
        p = t;
        q = kP / 2 + (t + step) % (kP / 2);
      } else {
        rr_pair(step, t, kP - 1, p, q);
      }
      const float a = G32[p * kPad + p].x, b = G32[q * kPad + q].x;
      const float2 g = G32[p * kPad + q];
      const float c2 = g.x * g.x + g.y * g.y;
      float cs = 1.0f, sn = 0.0f;
      float2 ph = make_float2(1.0f, 0.0f);
      if (c2 > 1e-14f * fabsf(a * b) && c2 > 0.0f && fminf(a, b) > floor2f) {
        const float inv_c = rsqrtf(c2);
        ph = make_float2(g.x * inv_c, -g.y * inv_c);
        const float z = (b - a) * 0.5f * inv_c, az = fabsf(z);
        const float tt = copysignf(1.0f, z) / (az > 1e18f ? 2.0f * az : az + sqrtf(1.0f + z * z));
        cs = rsqrtf(1.0f + tt * tt);
        sn = cs * tt;
      }
      S.csf[t] = cs;
      S.snf[t] = sn;
      S.phf[t] = ph;
    }
    __syncthreads();
    const float csa = S.csf[ba], sna = S.snf[ba], csb = S.csf[bb], snb = S.snf[bb];
    if (sna != 0.0f || snb != 0.0f) {
      int pa, qa, pb, qb;
      if (cross) {
        pa = ba;
        qa = kP / 2 + (ba + step) % (kP / 2);
        pb = bb;
        qb = kP / 2 + (bb + step) % (kP / 2);
      } else {
        rr_pair(step, ba, kP - 1, pa, qa);
        rr_pair(step, bb, kP - 1, pb, qb);
      }
      const float2 pha = S.phf[ba], phb = S.phf[bb];
      const float2 jb_qp = make_float2(-phb.x * snb, -phb.y * snb), jb_qq = make_float2(phb.x * csb, phb.y * csb);
      const float2 ca_qp = make_float2(-pha.x * sna, pha.y * sna), ca_qq = make_float2(pha.x * csa, -pha.y * csa);
      auto fma2 = [](float2& acc, float2 x, float2 y) {  // acc += x y
        acc.x = fmaf(x.x, y.x, acc.x);
        acc.x = fmaf(-x.y, y.y, acc.x);
        acc.y = fmaf(x.x, y.y, acc.y);
        acc.y = fmaf(x.y, y.x, acc.y);
      };
      const float2 b00 = G32[pa * kPad + pb], b01 = G32[pa * kPad + qb], b10 = G32[qa * kPad + pb],
                   b11 = G32[qa * kPad + qb];
      float2 m00 = make_float2(csa * b00.x, csa * b00.y), m01 = make_float2(csa * b01.x, csa * b01.y);
      float2 m10 = make_float2(sna * b00.x, sna * b00.y), m11 = make_float2(sna * b01.x, sna * b01.y);
      fma2(m00, ca_qp, b10);
      fma2(m01, ca_qp, b11);
      fma2(m10, ca_qq, b10);
      fma2(m11, ca_qq, b11);
      float2 n00 = make_float2(csb * m00.x, csb * m00.y), n01 = make_float2(snb * m00.x, snb * m00.y);
      float2 n10 = make_float2(csb * m10.x, csb * m10.y), n11 = make_float2(snb * m10.x, snb * m10.y);
      fma2(n00, m01, jb_qp);
      fma2(n01, m01, jb_qq);
      fma2(n10, m11, jb_qp);
      fma2(n11, m11, jb_qq);
      if (ba == bb) {
        n00.y = 0.0f;
        n11.y = 0.0f;
        n01 = make_float2(0.0f, 0.0f);
        n10 = make_float2(0.0f, 0.0f);
      }
      G32[pa * kPad + pb] = n00;
      G32[pa * kPad + qb] = n01;
      G32[qa * kPad + pb] = n10;
      G32[qa * kPad + qb] = n11;
      if (snb != 0.0f) {  // R32 <- R32 J_b on rows (pa, qa), columns (pb, qb)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int row = r == 0 ? pa : qa;
          const float2 x0 = R32[row * kPad + pb], x1 = R32[row * kPad + qb];
          float2 y0 = make_float2(csb * x0.x, csb * x0.y), y1 = make_float2(snb * x0.x, snb * x0.y);
          fma2(y0, x1, jb_qp);
          fma2(y1, x1, jb_qq);
          R32[row * kPad + pb] = y0;
          R32[row * kPad + qb] = y1;
        }
      }
    }
    __syncthreads();
  }
  store_inblock(G32);  // (FP32-accurate in-block Grams for the stored-Gram policy)
  for (int idx = t; idx < kP * kP; idx += 256) {
    const int i = idx / kP, j = idx % kP;
    const float2 r = R32[i * kPad + j];
    R[i * kPad + j] = make_double2(r.x, r.y);
  }
  __syncthreads();
  // polar factor, two Newton-Schulz steps R <- R - R E / 2, E = R^H R - I:
  // step 1 in FP64 on DMMA (E ~ 1e-7: R E must be exact to 1e-16), step 2
  // with E ~ 1e-14 (from an FP64 R^H R) and R E in FP32 (its error, ~1e-21,
  // is below FP64 rounding of R). R -> W -> R.
  if (ns_iters > 0) {
    gemm32c(R, R, G, true, true, t);  // G <- R^H R (upper tiles)
    __syncthreads();
    for (int idx = t; idx < kP * kP; idx += 256) {  // G <- 3/2 I - G / 2 (mirrored)
      const int i = idx / kP, j = idx % kP;
      if (i > j) continue;
      const cplx s = G[i * kPad + j];
      const cplx v = make_double2((i == j ? 1.5 : 0.0) - 0.5 * s.x, i == j ? 0.0 : -0.5 * s.y);
      G[i * kPad + j] = v;
      G[j * kPad + i] = make_double2(v.x, -v.y);
    }
    __syncthreads();
    gemm32c(R, G, W, false, false, t);  // W <- R (3 I - R^H R) / 2
    __syncthreads();
    if (ns_iters == 1) {  // (A/B: one step only, R unitary to ~1e-14)
      for (int idx = t; idx < kP * kP; idx += 256) {
        const int i = idx / kP, j = idx % kP;
        R[i * kPad + j] = W[i * kPad + j];
      }
      __syncthreads();
      return;
    }
    gemm32c(W, W, G, true, true, t);  // G <- W^H W (upper tiles)
    __syncthreads();
    float2* const E32 = reinterpret_cast<float2*>(R);  // R (step-1 input) is dead
    float2* const W32 = E32 + kP * kPad;
    for (int idx = t; idx < kP * kP; idx += 256) {
      const int i = idx / kP, j = idx % kP;
      const cplx w = W[i * kPad + j];
      W32[i * kPad + j] = make_float2((float)w.x, (float)w.y);
      if (i > j) continue;
      const cplx s = G[i * kPad + j];
      const float2 e = make_float2((float)(s.x - (i == j ? 1.0 : 0.0)), i == j ? 0.0f : (float)s.y);
      E32[i * kPad + j] = e;
      E32[j * kPad + i] = make_float2(e.x, -e.y);
    }
    __syncthreads();
    float2 pe[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {  // (W E)[i][j], FP32
      const int idx = t + 256 * h, i = idx / kP, j = idx % kP;
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll 8
      for (int k = 0; k < kP; ++k) {
        const float2 w = W32[i * kPad + k], e = E32[k * kPad + j];
        acc.x = fmaf(w.x, e.x, fmaf(-w.y, e.y, acc.x));
        acc.y = fmaf(w.x, e.y, fmaf(w.y, e.x, acc.y));
      }
      pe[h] = acc;
    }
    __syncthreads();  // E32 / W32 (aliasing R) are read
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int idx = t + 256 * h, i = idx / kP, j = idx % kP;
      const cplx w = W[i * kPad + j];
      R[i * kPad + j] = make_double2(w.x - 0.5 * (double)pe[h].x, w.y - 0.5 * (double)pe[h].y);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void pair_evd_v1(cplx* G, cplx* R, EvdScratch& S, int t, double tol_in, double floor2,
                                            int max_in, bool cross = false) {
  pair_evd_t<kP, kPad, 256, MPSIM_EVD_FOLD>(G, R, S, t, tol_in, floor2, max_in, cross);
}

}  // namespace mpsim_gpu
