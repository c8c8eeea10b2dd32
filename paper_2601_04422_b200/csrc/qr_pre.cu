// QR preconditioning of the batched Jacobi SVD (Drmac-Veselic): theta = Q R by
// blocked Householder QR, then the one-sided Jacobi runs on R^H, whose columns
// are far closer to orthogonal in the sense the sweeps need: at chi = 512 the
// 1024 x 1024 theta of a random circuit converges in 11 sweeps instead of 14
// (tools/emu_jacobi.py). Q is never formed: R^H = U' Sigma W^H gives the right
// singular vectors of theta directly (S V^dag = X^H), and U = theta X / sigma^2
// from the pristine theta (split.cu, f = 1; the transposed case likewise).
//
// Two-step variant (pre = 2): R^H = Q2 R2 again and the Jacobi runs on R2^H
// (9 instead of 11 sweeps at chi = 512); R2^H = U'' S W^H gives theta =
// Q1 U'' S (Q2 W)^H, so the converged X is mapped back through the stored
// block reflectors of the first QR, Z = Q1 [X; 0] (qrp_update_kernel<true>,
// kept columns only, after the truncation), and the epilogue writes the
// factors as without preconditioning (f = trans).
//
// Per 32-column panel p of every gate's QR operand A (vectors = columns,
// stride qr_m_pad, rows [0, qr_m)):
//   qrp_panel_kernel    one 1024-thread CTA per gate: 32 Householder
//                       reflectors (zlarfg convention, H = I - tau v v^H),
//                       R written on and above the diagonal, explicit V
//                       (unit diagonal, zeros above) and the compact-WY T
//                       (zlarft, Q_p = I - V T V^H) to scratch
//   qrp_update_kernel   A_b <- Q_p^H A_b = A_b - V T^H (V^H A_b) for each
//                       32-column block b right of the panel, both GEMMs on
//                       DMMA with the pair-chunk pipeline of jacobi_split.cu
// and finally qrp_form_rh_kernel writes X = R^H (n vectors of length n).
#include <cooperative_groups.h>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "pair_gemm.cuh"

namespace mpsim_gpu {

namespace {

constexpr int kQ = 32;                  // panel width
constexpr int kQC = pg::kC;             // rows per streamed chunk
constexpr int kQPitch = pg::kPitch;     // conflict-free DMMA fragment pitch (== 4 mod 16)
constexpr int kQPlane = pg::kPlane;
constexpr int kQPitchW = 34;  // complex W2 pitch (== 2 mod 8: conflict-free 16-byte B fragments)

__device__ __forceinline__ double block_sum_1024(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int t = threadIdx.x;
  __syncthreads();  // red is reused across calls
  if ((t & 31) == 0) red[t >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll 8
  for (int w = 0; w < 32; ++w) s += red[w];
  return s;
}

}  // namespace

// vbuf: per gate and panel kQ vectors of stride vld (>= qr_m_pad); tbuf: per
// gate and panel kQ x kQ; npan panel slots per gate (all kept for Q1 [X; 0]).
// The current reflector is also staged in shared memory (dynamic, qr_m_pad
// complex) and the per-warp column loops keep 8 independent loads in flight:
// the panel is latency-bound (32 dependent reflectors), not bandwidth-bound.
__global__ void __launch_bounds__(1024) qrp_panel_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                         int p, cplx* __restrict__ vbuf, long long vld,
                                                         cplx* __restrict__ tbuf, int npan) {
  const GateDesc& g = gates[blockIdx.x];
  if (!g.pre) return;
  const int n = g.n, m = g.qr_m;
  const long long ld = g.qr_m_pad;
  const int c0 = kQ * p;
  if (c0 >= n) return;
  const int jb = min(kQ, n - c0);
  cplx* A = ws + g.qr_off;
  cplx* V = vbuf + ((long long)blockIdx.x * npan + p) * kQ * vld;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  __shared__ double red[32];
  __shared__ cplx taus[kQ];
  __shared__ cplx Gv[kQ][kQ + 1];
  __shared__ cplx T[kQ][kQ + 1];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* vs = reinterpret_cast<cplx*>(smem_raw);  // current reflector, rows [0, qr_m_pad)

  for (int j = 0; j < jb; ++j) {
    const int row0 = c0 + j;
    cplx* col = A + (long long)(c0 + j) * ld;
    double s = 0.0;
    for (int r = row0 + 1 + t; r < m; r += 1024) s += cabs2(xs_get(col, ld, r));
    const double xn2 = block_sum_1024(s, red);
    const cplx alpha = row0 < m ? xs_get(col, ld, row0) : make_double2(0.0, 0.0);
    // zlarfg: H^H x = beta e_1, beta real, v = [1; x(2:)/(alpha - beta)]
    cplx tau = make_double2(0.0, 0.0), inv = make_double2(0.0, 0.0);
    double beta = alpha.x;
    if (!(xn2 == 0.0 && alpha.y == 0.0)) {
      beta = -copysign(sqrt(cabs2(alpha) + xn2), alpha.x);
      tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
      const cplx d = make_double2(alpha.x - beta, alpha.y);
      const double dd = cabs2(d);
      inv = make_double2(d.x / dd, -d.y / dd);
    }
    const bool refl = tau.x != 0.0 || tau.y != 0.0;
    cplx* vj = V + (long long)j * vld;
    for (long long r = t; r < vld; r += 1024) {
      cplx v = make_double2(0.0, 0.0);
      if (r == row0) v = make_double2(1.0, 0.0);
      else if (r > row0 && r < m && refl) v = cmul(xs_get(col, ld, r), inv);
      xs_set(vj, vld, r, v);
      if (r < ld) vs[r] = v;
    }
    if (t == 0) {
      if (row0 < m) xs_set(col, ld, row0, make_double2(refl ? beta : alpha.x, refl ? 0.0 : alpha.y));
      taus[j] = tau;
    }
    __syncthreads();
    // warps [jb-1-j, jb-1): Gv[i][j] = v_i^H v_j, i < j (for zlarft), while
    // warps [0, jb-1-j) apply H^H = I - conj(tau) v v^H to panel columns
    // j+1 .. jb-1, one column each
    if (warp >= jb - 1 - j && warp < jb - 1) {
      const int i = warp - (jb - 1 - j);
      const cplx* vi = V + (long long)i * vld;
      constexpr int kU = 4;
      cplx w[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) w[u] = make_double2(0.0, 0.0);
      for (int rb = row0; rb < m; rb += 32 * kU) {
        cplx xv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          xv[u] = r < m ? xs_get(vi, vld, r) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          if (r < m) cfmac(w[u], xv[u], vs[r]);
        }
      }
#pragma unroll
      for (int u = 1; u < kU; ++u) {
        w[0].x += w[u].x;
        w[0].y += w[u].y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w[0].x += __shfl_xor_sync(0xffffffffu, w[0].x, o);
        w[0].y += __shfl_xor_sync(0xffffffffu, w[0].y, o);
      }
      if (lane == 0) Gv[i][j] = w[0];
    }
    if (refl && warp < jb - 1 - j) {
      cplx* a = A + (long long)(c0 + j + 1 + warp) * ld;
      constexpr int kU = 4;
      cplx w[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) w[u] = make_double2(0.0, 0.0);
      for (int rb = row0; rb < m; rb += 32 * kU) {
        cplx av[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          av[u] = r < m ? xs_get(a, ld, r) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          if (r < m) cfmac(w[u], vs[r], av[u]);
        }
      }
#pragma unroll
      for (int u = 1; u < kU; ++u) {
        w[0].x += w[u].x;
        w[0].y += w[u].y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w[0].x += __shfl_xor_sync(0xffffffffu, w[0].x, o);
        w[0].y += __shfl_xor_sync(0xffffffffu, w[0].y, o);
      }
      const cplx coef = cmul(make_double2(tau.x, -tau.y), w[0]);
      for (int rb = row0; rb < m; rb += 32 * kU) {
        cplx av[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          av[u] = r < m ? xs_get(a, ld, r) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int r = rb + 32 * u + lane;
          if (r < m) {
            const cplx vr = vs[r];
            av[u].x -= vr.x * coef.x - vr.y * coef.y;
            av[u].y -= vr.x * coef.y + vr.y * coef.x;
            xs_set(a, ld, r, av[u]);
          }
        }
      }
    }
    __syncthreads();
  }
  // unused reflector slots of a short last panel: v = 0, tau = 0
  for (int j = jb; j < kQ; ++j) {
    cplx* vj = V + (long long)j * vld;
    for (long long r = t; r < vld; r += 1024) xs_set(vj, vld, r, make_double2(0.0, 0.0));
    if (t == 0) taus[j] = make_double2(0.0, 0.0);
  }
  for (int idx = t; idx < kQ * (kQ + 1); idx += 1024) T[idx / (kQ + 1)][idx % (kQ + 1)] = make_double2(0.0, 0.0);
  __syncthreads();
  // zlarft (forward, columnwise): T[j][j] = tau_j, T[0:j, j] = -tau_j T[0:j,0:j] Gv[0:j, j]
  for (int j = 0; j < jb; ++j) {
    if (t < j) {
      cplx z = make_double2(0.0, 0.0);
      for (int k = t; k < j; ++k) cfma(z, T[t][k], Gv[k][j]);
      const cplx tj = taus[j];
      T[t][j] = make_double2(-(tj.x * z.x - tj.y * z.y), -(tj.x * z.y + tj.y * z.x));
    } else if (t == j) {
      T[j][j] = taus[j];
    }
    __syncthreads();
  }
  cplx* To = tbuf + ((long long)blockIdx.x * npan + p) * kQ * kQ;
  for (int idx = t; idx < kQ * kQ; idx += 1024) To[idx] = T[idx / kQ][idx % kQ];
}

// ---- Cluster-resident panel (default for qr_m_pad <= 256 * 8): the 32
// panel columns live in registers, spread over a cluster of cs = qr_m_pad /
// 256 CTAs of 32 warps: warp w of CTA k holds rows [256 k, 256 k + 256) of
// panel column w, 8 rows per lane. A reflector costs two cluster barriers:
// (1) partial norms -> every CTA forms beta / tau redundantly; (2) partial
// v^H a_c (and v_i^H v_j for zlarft) -> every CTA updates its rows. The
// previous kernel (qrp_panel_kernel) streamed the columns through L2 on every
// reflector and spent 10 us per reflector waiting on those loads.
namespace cgp = cooperative_groups;
constexpr int kPR = 256;  // panel rows per CTA
constexpr int kPL = kPR / 32;

struct PanelSmem {
  cplx vs[kQ][kPR];       // this CTA's rows of every reflector
  double pn[2];           // partial ||x(2:)||^2 (double-buffered by reflector parity)
  cplx pal[2];            // alpha, written by the CTA owning the diagonal row
  cplx pw[2][kQ];         // partial v_j^H a_c (c > j) and v_i^H v_j (i < j)
  cplx taus[kQ];
  cplx Gv[kQ][kQ + 1];
  cplx T[kQ][kQ + 1];
  cplx tau, inv, alpha;  // this reflector's zlarfg results (thread 0 forms them)
  double beta;
};

__global__ void __launch_bounds__(1024, 1) qrp_panel_cluster_kernel(const GateDesc* __restrict__ gates,
                                                                    cplx* __restrict__ ws, int p,
                                                                    cplx* __restrict__ vbuf, long long vld,
                                                                    cplx* __restrict__ tbuf, int npan) {
  cgp::cluster_group cl = cgp::this_cluster();
  const int rank = (int)cl.block_rank(), cs = (int)cl.num_blocks();
  const GateDesc& g = gates[blockIdx.y];
  // whole clusters skip together (no barrier is ever left waiting)
  if (!g.pre) return;
  const int n = g.n, m = g.qr_m;
  const long long ld = g.qr_m_pad;
  const int c0 = kQ * p;
  if (c0 >= n) return;
  const int jb = min(kQ, n - c0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PanelSmem& S = *reinterpret_cast<PanelSmem*>(smem_raw);
  cplx* A = ws + g.qr_off;
  cplx* V = vbuf + ((long long)blockIdx.y * npan + p) * kQ * vld;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rbase = kPR * rank;
  // this warp's column slice: rows rbase + lane + 32 s
  cplx a[kPL];
  cplx* acol = A + (long long)(c0 + warp) * ld;
#pragma unroll
  for (int s2 = 0; s2 < kPL; ++s2) {
    const int r = rbase + lane + 32 * s2;
    a[s2] = (warp < jb && r < m) ? xs_get(acol, ld, r) : make_double2(0.0, 0.0);
  }
  for (int j = 0; j < jb; ++j) {
    const int row0 = c0 + j, buf = j & 1;
    // (1) partial norm of column j below the diagonal, and alpha
    if (warp == j) {
      double sn = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < kPL; ++s2) {
        const int r = rbase + lane + 32 * s2;
        if (r > row0 && r < m) sn += cabs2(a[s2]);
        if (r == row0) S.pal[buf] = a[s2];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sn += __shfl_xor_sync(0xffffffffu, sn, o);
      if (lane == 0) S.pn[buf] = sn;
    }
    cl.sync();
    if (t == 0) {  // one thread per CTA gathers the partials and forms zlarfg
      double xn2 = 0.0;
      for (int k = 0; k < cs; ++k) xn2 += *cl.map_shared_rank(&S.pn[buf], k);
      const int owner = row0 / kPR;
      const cplx al = row0 < m ? *cl.map_shared_rank(&S.pal[buf], owner) : make_double2(0.0, 0.0);
      // zlarfg: H^H x = beta e_1, beta real, v = [1; x(2:)/(alpha - beta)]
      cplx ta = make_double2(0.0, 0.0), iv = make_double2(0.0, 0.0);
      double be = al.x;
      if (!(xn2 == 0.0 && al.y == 0.0)) {
        be = -copysign(sqrt(cabs2(al) + xn2), al.x);
        ta = make_double2((be - al.x) / be, -al.y / be);
        const cplx d = make_double2(al.x - be, al.y);
        const double dd = cabs2(d);
        iv = make_double2(d.x / dd, -d.y / dd);
      }
      S.tau = ta;
      S.inv = iv;
      S.alpha = al;
      S.beta = be;
    }
    __syncthreads();
    const cplx tau = S.tau, inv = S.inv, alpha = S.alpha;
    const double beta = S.beta;
    const bool refl = tau.x != 0.0 || tau.y != 0.0;
    if (warp == j) {
#pragma unroll
      for (int s2 = 0; s2 < kPL; ++s2) {
        const int r = rbase + lane + 32 * s2;
        cplx v = make_double2(0.0, 0.0);
        if (r == row0) {
          v = make_double2(1.0, 0.0);
          a[s2] = make_double2(refl ? beta : alpha.x, refl ? 0.0 : alpha.y);  // R diagonal
        } else if (r > row0 && r < m && refl) {
          v = cmul(a[s2], inv);
        }
        S.vs[j][lane + 32 * s2] = v;
      }
      if (t == 32 * j) S.taus[j] = tau;
    }
    __syncthreads();
    // (2) partial v^H a_c for the columns right of j, v_i^H v_j for i < j
    cplx w = make_double2(0.0, 0.0);
    if (warp != j) {
#pragma unroll
      for (int s2 = 0; s2 < kPL; ++s2) {
        const cplx v = S.vs[j][lane + 32 * s2];
        if (warp > j) cfmac(w, v, a[s2]);
        else cfmac(w, S.vs[warp][lane + 32 * s2], v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w.x += __shfl_xor_sync(0xffffffffu, w.x, o);
        w.y += __shfl_xor_sync(0xffffffffu, w.y, o);
      }
      if (lane == 0) S.pw[buf][warp] = w;
    }
    cl.sync();
    if (warp != j && warp < jb) {
      cplx x = make_double2(0.0, 0.0);
      if (lane < cs) x = *cl.map_shared_rank(&S.pw[buf][warp], lane);  // one remote read per lane
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        x.x += __shfl_xor_sync(0xffffffffu, x.x, o);
        x.y += __shfl_xor_sync(0xffffffffu, x.y, o);
      }
      const cplx tot = make_double2(__shfl_sync(0xffffffffu, x.x, 0), __shfl_sync(0xffffffffu, x.y, 0));
      if (warp > j) {
        if (refl) {
          const cplx coef = cmul(make_double2(tau.x, -tau.y), tot);
#pragma unroll
          for (int s2 = 0; s2 < kPL; ++s2) {
            const int r = rbase + lane + 32 * s2;
            if (r >= row0 && r < m) {
              const cplx v = S.vs[j][lane + 32 * s2];
              a[s2].x -= v.x * coef.x - v.y * coef.y;
              a[s2].y -= v.x * coef.y + v.y * coef.x;
            }
          }
        }
      } else if (lane == 0) {
        S.Gv[warp][j] = tot;
      }
    }
  }
  // write back R (and whatever lies below the diagonal) and the reflectors
#pragma unroll
  for (int s2 = 0; s2 < kPL; ++s2) {
    const int r = rbase + lane + 32 * s2;
    if (warp < jb && r < ld) xs_set(acol, ld, r, a[s2]);
  }
  for (int idx = t; idx < kQ * kPR; idx += 1024) {
    const int jj = idx / kPR, rr = idx % kPR, r = rbase + rr;
    if (r < vld) xs_set(V + (long long)jj * vld, vld, r, jj < jb ? S.vs[jj][rr] : make_double2(0.0, 0.0));
  }
  if (rank == 0) {
    // zlarft (forward, columnwise): T[j][j] = tau_j, T[0:j, j] = -tau_j T[0:j,0:j] Gv[0:j, j]
    for (int idx = t; idx < kQ * (kQ + 1); idx += 1024) S.T[idx / (kQ + 1)][idx % (kQ + 1)] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int j = 0; j < jb; ++j) {
      if (t < j) {
        cplx z = make_double2(0.0, 0.0);
        for (int k = t; k < j; ++k) cfma(z, S.T[t][k], S.Gv[k][j]);
        const cplx tj = S.taus[j];
        S.T[t][j] = make_double2(-(tj.x * z.x - tj.y * z.y), -(tj.x * z.y + tj.y * z.x));
      } else if (t == j) {
        S.T[j][j] = S.taus[j];
      }
      __syncthreads();
    }
    cplx* To = tbuf + ((long long)blockIdx.y * npan + p) * kQ * kQ;
    for (int idx = t; idx < kQ * kQ; idx += 1024) To[idx] = S.T[idx / kQ][idx % kQ];
  }
  cl.sync();  // no CTA leaves while its shared memory may still be read remotely
}

namespace {

struct QrUpdSmem {
  union {
    double buf[2][pg::kBuf];
    struct {                     // after pass 1 (the chunk buffers are dead)
      double Wx[64 * 65];        // real 64 x 64 V_ext^T A_ext
      cplx W[kQ * (kQ + 1)];     // V^H A_b
      cplx T[kQ * (kQ + 1)];
    } w;
  } u;
  cplx W2[kQ * kQPitchW];        // -(T^H W) (or -(T W)), complex, pitch 34
};

}  // namespace

// kApply = false: A_b <- Q_p^H A_b = A_b - V T^H (V^H A_b) for the 32-column
// block b at c0 + 32 (b + 1) (trailing update of the factorisation);
// kApply = true:  A_b <- Q_p A_b = A_b - V T (V^H A_b) for block b at 32 b
// (Z = Q1 [X; 0], panels applied last to first). Rows [c0, qr_m_pad).
// Grid (blocks, gates), 256 threads.
template <bool kApply>
__global__ void __launch_bounds__(256, 2) qrp_update_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                            int p, const cplx* __restrict__ vbuf, long long vld,
                                                            const cplx* __restrict__ tbuf, int npan,
                                                            const GateOut* __restrict__ out) {
  const GateDesc& g = gates[blockIdx.y];
  if (!g.pre) return;
  const int c0 = kQ * p;
  if (kApply && c0 >= g.n) return;
  const int cb = kApply ? kQ * blockIdx.x : c0 + kQ * (blockIdx.x + 1);
  if (cb >= g.n_pad) return;
  if (kApply && cb >= out[blockIdx.y].k) return;  // only the kept columns are mapped back
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QrUpdSmem& S = *reinterpret_cast<QrUpdSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const long long ald = g.qr_m_pad;
  cplx* A = ws + g.qr_off + (long long)cb * ald;
  const cplx* V = vbuf + ((long long)blockIdx.y * npan + p) * kQ * vld;
  pg::Loader ld;
  ld.init([&](int v) { return V + (long long)v * vld; }, [&](int v) { return A + (long long)v * ald; }, vld, ald, t);
  const int nchunks = (int)((ald - c0) / kQC);

  // ---- pass 1: W = V^H A_b (pair_gemm.cuh), then T
  pg::cross_gram(ld, S.u.buf, S.u.w.Wx, S.u.w.W, kQ + 1, c0, ald, t);
  const cplx* Tg = tbuf + ((long long)blockIdx.y * npan + p) * kQ * kQ;
  for (int idx = t; idx < kQ * kQ; idx += 256) S.u.w.T[(idx / kQ) * (kQ + 1) + idx % kQ] = Tg[idx];
  __syncthreads();
  // W2 = T^H W (factorisation) or T W (apply), T upper triangular; stored
  // negated in real-extended form
  for (int idx = t; idx < kQ * kQ; idx += 256) {
    const int i = idx / kQ, j = idx % kQ;
    cplx z = make_double2(0.0, 0.0);
    if (kApply) {
      for (int k = i; k < kQ; ++k) cfma(z, S.u.w.T[i * (kQ + 1) + k], S.u.w.W[k * (kQ + 1) + j]);
    } else {
      for (int k = 0; k <= i; ++k) cfmac(z, S.u.w.T[k * (kQ + 1) + i], S.u.w.W[k * (kQ + 1) + j]);
    }
    S.W2[i * kQPitchW + j] = make_double2(-z.x, -z.y);
  }
  __syncthreads();

  // ---- pass 2: A_ext += V_ext (-W2_ext), -W2_ext = [[Re, Im], [-Im, Re]] of -W2
  // formed from one 16-byte load per k-step. Warp w: row tiles 2 (w & 1) +
  // {0, 1}, complex column tile w / 2 (real tiles w/2 and 4 + w/2).
  const int rbase = 2 * (warp & 1), cj = warp >> 1;
  const int jb = 8 * cj + fr;
  // chunks last to first (L2 reuse of pass 1's most recent rows)
  ld.issue(S.u.buf[0], c0 + (nchunks - 1) * kQC);
  for (int k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) {
      ld.issue(S.u.buf[(k + 1) & 1], c0 + (nchunks - 2 - k) * kQC);
      pg::wait<1>();
    } else {
      pg::wait<0>();
    }
    __syncthreads();
    const double* B = S.u.buf[k & 1];
    double o[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = 8 * (rbase + a) + fr, j = 8 * cj + 2 * fk + v;
        o[a][0][v] = B[2 * kQPlane + j * kQPitch + e];
        o[a][1][v] = B[3 * kQPlane + j * kQPitch + e];
      }
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int cc = (4 * s + fk) & (kQ - 1);
      const double* plane = B + (s < 8 ? 0 : kQPlane) + cc * kQPitch;
      const double a0 = plane[8 * rbase + fr], a1 = plane[8 * (rbase + 1) + fr];
      const cplx w2 = S.W2[cc * kQPitchW + jb];
      const double b0 = s < 8 ? w2.x : -w2.y, b1 = s < 8 ? w2.y : w2.x;
      pg::dmma(o[0][0][0], o[0][0][1], a0, b0);
      pg::dmma(o[0][1][0], o[0][1][1], a0, b1);
      pg::dmma(o[1][0][0], o[1][0][1], a1, b0);
      pg::dmma(o[1][1][0], o[1][1][1], a1, b1);
    }
    const int r0 = c0 + (nchunks - 1 - k) * kQC;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int e = 8 * (rbase + a) + fr, j = 8 * cj + 2 * fk + v;
        double* aj = reinterpret_cast<double*>(A + (long long)j * ald);
        aj[r0 + e] = o[a][0][v];
        aj[ald + r0 + e] = o[a][1][v];
      }
    __syncthreads();
  }
}

// X = R^H: X[j][i] = conj(R[j][i]) = conj(A_i[j]) for j <= i < n, else 0,
// i < m_pad (= round64(n)), j < n_pad. Grid (m_pad / 32, n_pad / 32, gates).
// second_step: this is the second QR of pre = 2 (R2^H -> the Jacobi operand);
// either way the target is split planes (common.cuh).
__global__ void __launch_bounds__(256) qrp_form_rh_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                          int second_step) {
  const GateDesc& g = gates[blockIdx.z];
  if (!g.pre) return;
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  if (i0 >= g.m_pad || j0 >= g.n_pad) return;
  const cplx* A = ws + g.qr_off;
  cplx* X = ws + g.ws_off;
  __shared__ cplx tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // read A_i[j] along j (rows of A), i.e. tile[ii][jj]
  for (int ii = ty; ii < 32; ii += 8) {
    const int i = i0 + ii, j = j0 + tx;
    cplx v = make_double2(0.0, 0.0);
    if (i < g.n && j < g.n && j <= i) {
      const cplx a = xs_get(A + (long long)i * g.qr_m_pad, g.qr_m_pad, j);
      v = make_double2(a.x, -a.y);
    }
    tile[ii][tx] = v;
  }
  __syncthreads();
  for (int jj = ty; jj < 32; jj += 8) {
    const int j = j0 + jj, i = i0 + tx;
    xs_set(X + (long long)j * g.m_pad, g.m_pad, i, tile[tx][jj]);
  }
}

// Z[j][r] = X[order[j]][r] for r < n (X: stride m_pad, the converged R2^H
// side, order: the truncation's descending-sigma order), 0 for n <= r <
// qr_m_pad; kept columns j < k only. Grid (qr_m_pad / 256, n_pad, gates).
__global__ void __launch_bounds__(256) qrp_zinit_kernel(const GateDesc* __restrict__ gates, cplx* __restrict__ ws,
                                                        const int* __restrict__ order, long long sig_stride,
                                                        const GateOut* __restrict__ out) {
  const GateDesc& g = gates[blockIdx.z];
  if (!g.pre) return;
  const long long r = blockIdx.x * 256LL + threadIdx.x;
  const int j = blockIdx.y;
  if (r >= g.qr_m_pad || j >= out[blockIdx.z].k) return;
  const cplx* X = ws + g.ws_off + (long long)(g.zsrc_ordered ? j : order[blockIdx.z * sig_stride + j]) * g.m_pad;
  cplx* Z = ws + g.qr_off + (long long)j * g.qr_m_pad;
  xs_set(Z, g.qr_m_pad, r, r < g.n ? xs_get(X, g.m_pad, r) : make_double2(0.0, 0.0));
}

// MPSIM_PANEL=legacy selects the L2-streaming panel kernel (A/B only).
static bool panel_legacy() {
  static const bool v = [] {
    const char* e = ab_knob("MPSIM_PANEL");
    return e != nullptr && std::string(e) == "legacy";
  }();
  return v;
}

void qrp_init() {
  cudaFuncSetAttribute(qrp_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PanelSmem));
  cudaFuncSetAttribute(qrp_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(qrp_update_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(QrUpdSmem));
  cudaFuncSetAttribute(qrp_update_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(QrUpdSmem));
}

// Householder QR of every descriptor with pre != 0 (panels, trailing
// updates), then X = R^H (qrp_form_rh_kernel: from qr_off into ws_off).
// max_n_pad: largest n_pad; max_x_pad: largest X stride; vbuf / tbuf hold
// npan panel slots per gate.
void launch_qr_factor(const GateDesc* d_gates, int n_gates, int max_n_pad, int max_x_pad, cplx* ws, cplx* vbuf,
                      long long vld, cplx* tbuf, int npan, int second_step, cudaStream_t st) {
  const int panels = max_n_pad / kQ;
  const int cs = (int)((vld + kPR - 1) / kPR);
  // The cluster kernel holds one SM per CTA (128 KB of reflector slices): use
  // it while all clusters fit in one wave, else one streaming CTA per gate.
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool cluster = cs <= 8 && (long long)cs * n_gates <= sms && !panel_legacy();
  for (int p = 0; p < panels; ++p) {
    if (cluster) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, n_gates);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = sizeof(PanelSmem);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, qrp_panel_cluster_kernel, d_gates, ws, p, vbuf, vld, tbuf, npan);
    } else {
      qrp_panel_kernel<<<n_gates, 1024, sizeof(cplx) * vld, st>>>(d_gates, ws, p, vbuf, vld, tbuf, npan);
    }
    const int blocks = panels - p - 1;
    if (blocks > 0)
      qrp_update_kernel<false><<<dim3(blocks, n_gates), 256, sizeof(QrUpdSmem), st>>>(d_gates, ws, p, vbuf, vld,
                                                                                      tbuf, npan, nullptr);
  }
  qrp_form_rh_kernel<<<dim3(max_x_pad / 32, max_n_pad / 32, n_gates), 256, 0, st>>>(d_gates, ws, second_step);
}

// Z = Q1 [X_kept; 0] (kept columns in descending-sigma order) with the
// reflectors kept by launch_qr_factor; runs after the truncation.
void launch_qr_apply(const GateDesc* d_gates, int n_gates, int max_n_pad, int max_qr_m_pad, cplx* ws,
                     const cplx* vbuf, long long vld, const cplx* tbuf, int npan, const int* order,
                     long long sig_stride, const GateOut* out, cudaStream_t st) {
  qrp_zinit_kernel<<<dim3((max_qr_m_pad + 255) / 256, max_n_pad, n_gates), 256, 0, st>>>(d_gates, ws, order,
                                                                                        sig_stride, out);
  const int panels = max_n_pad / kQ;
  for (int p = panels - 1; p >= 0; --p)
    qrp_update_kernel<true><<<dim3(panels, n_gates), 256, sizeof(QrUpdSmem), st>>>(d_gates, ws, p, vbuf, vld, tbuf,
                                                                                  npan, out);
}

}  // namespace mpsim_gpu
