// Householder QR of one tall site matrix for the centre moves (thin_qr,
// mps.cpp:57-65, in sweep_left_of / sweep_right_of, mps.cpp:69-95), shaped
// for latency: a centre move is a chain of site QRs where each site waits for
// the previous one's R, so nothing batches and the cost is the length of the
// dependent reflector chain (one per column).
//
//   site_qr_factor_kernel  one persistent launch per site: CTA c owns the
//                          8 columns of panel c in registers, applies the
//                          published block reflectors of panels 0..c-1 and
//                          factors its own panel (zlarfg / zlarft), chained
//                          by release / acquire flags;
//   site_qr_q_kernel       Q = H_0 ... H_{np-1} [I; 0], CTA c forming its 8
//                          columns independently, on a second stream so it
//                          overlaps the next site's factorisation.
// Any exact QR gives the same state; only k = min(m, n) is fixed by the
// reference (mps.cpp:57-65), and the reflector convention is zlarfg's.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cmath>
#include <string>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

namespace {

constexpr int kSW = 8;     // panel width (warps per panel CTA)
constexpr int kSL = 32;    // m <= 32 * 32 = 1024 rows (four warps x 8 rows per lane per column)

__device__ __forceinline__ cplx warp_sum(cplx v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

}  // namespace

// left (right = 0): A_c[r] = site[r chi + c] (r < 2 dl, c < dr); right:
// A_l[e] = conj(site[(l 2 + p) chi + r]), e = p dr + r. Column-major, lda.
__global__ void site_matrix_kernel(const cplx* __restrict__ site, int chi, int dl, int dr, int right,
                                   cplx* __restrict__ A, int lda) {
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * m;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / m), r = (int)(i % m);
    cplx v;
    if (!right) {
      v = site[(long long)r * chi + c];
    } else {
      const int p = r / dr, rr = r % dr;
      v = site[(long long)(c * 2 + p) * chi + rr];
      v.y = -v.y;
    }
    A[(long long)c * lda + r] = v;
  }
}

// ---- one persistent launch per site QR (factor) and one for Q formation.
// CTA c (1024 threads) owns columns [8c, 8c + 8) for the whole
// factorisation, in registers: warp w holds column 8c + (w & 7), rows
// 256 (w >> 3) + lane + 32 s (s < 8), i.e. four warps per column. It applies
// the block reflectors of panels 0 .. c-1 as each one is published (flag[p],
// release / acquire at gpu scope; V_p staged once in shared memory), factors
// its own panel in place (three block barriers per reflector, reductions
// over a column's four warps through shared memory), publishes V_c / T_c and
// releases flag[c]. The serial chain is panel p -> apply to panel p+1's
// columns -> factor panel p+1. Q = H_0 ... H_{np-1} [I; 0]: CTA c forms Q
// columns [8c, 8c + 8) by applying Q_c, ..., Q_0 (no cross-CTA dependencies).
namespace {
constexpr int kG = 4;   // warps (row groups of 256) per column
constexpr int kRL = 8;  // rows per lane

struct SiteQrSmem {
  cplx vs[kSW][kG * 256];  // a staged V_p (rows relative to 8p) or this CTA's own V_c
  cplx part[kSW][kSW][kG]; // per-group partials: V^H A (apply), v_j^H a_c and v_w^H v_j (factor)
  double pn[kG];
  cplx w2[kSW][kSW];
  cplx taus[kSW];
  cplx gv[kSW][kSW];
  cplx ts[kSW][kSW];
  cplx xr[2][kG * 256];    // raw column j below its diagonal (rows relative to c0), by reflector parity
  cplx adg[2][kSW];        // a_col(dg) of the reflector being formed, by reflector parity
  cplx inv;                // 1 / (alpha - beta) of the reflector being formed
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp sum of 4 complex values at once (reduce-scatter butterfly: 5 complex
// shuffles instead of 20): lane l ends with the total of value
// 2 ((l >> 4) & 1) + ((l >> 3) & 1).
__device__ __forceinline__ cplx warp_sum4(cplx (&v)[4], int lane) {
  auto sx = [](cplx x, int o) {
    return make_double2(__shfl_xor_sync(0xffffffffu, x.x, o), __shfl_xor_sync(0xffffffffu, x.y, o));
  };
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool up = lane & 16;
    const cplx r = sx(up ? v[k] : v[k + 2], 16);
    v[k] = cadd(up ? v[k + 2] : v[k], r);
  }
  {
    const bool up = lane & 8;
    const cplx r = sx(up ? v[0] : v[1], 8);
    v[0] = cadd(up ? v[1] : v[0], r);
  }
  v[0] = cadd(v[0], sx(v[0], 4));
  v[0] = cadd(v[0], sx(v[0], 2));
  v[0] = cadd(v[0], sx(v[0], 1));
  return v[0];
}

// a (this thread's rows of column `col`) <- ((I - V op(T) V^H) A) for rows >=
// r0. V (global, column i at V + i * ldv, rows relative to r0) and T are read
// with ld.global.cg: during the factorisation other CTAs of this launch wrote
// them (published by flags).
__device__ __forceinline__ void apply_block(SiteQrSmem& S, cplx (&a)[kRL], const cplx* V, int ldv, const cplx* T,
                                            int r0, int m, bool adjoint) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, col = warp & 7, grp = warp >> 3;
  const int L = m - r0;
#pragma unroll
  for (int i = 0; i < kSW; ++i)
    for (int rr = t; rr < L; rr += 1024) S.vs[i][rr] = __ldcg(V + (long long)i * ldv + rr);
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // V^H a in two halves of four reflectors (register budget of 1024 threads)
    cplx acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int s = 0; s < kRL; ++s) {
      const int r = 256 * grp + lane + 32 * s;
      if (r >= r0 && r < m) {
#pragma unroll
        for (int i = 0; i < 4; ++i) cfmac(acc[i], S.vs[4 * h + i][r - r0], a[s]);
      }
    }
    const cplx tot = warp_sum4(acc, lane);
    if ((lane & 7) == 0) S.part[4 * h + ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1)][col][grp] = tot;
  }
  __syncthreads();
  if (t < 64) {
    const int i = t >> 3, c = t & 7;
    cplx x = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kSW; ++k) {
      const cplx wk = cadd(cadd(S.part[k][c][0], S.part[k][c][1]), cadd(S.part[k][c][2], S.part[k][c][3]));
      const cplx tk = adjoint ? conjc(__ldcg(T + k * kSW + i)) : __ldcg(T + i * kSW + k);
      cfma(x, tk, wk);
    }
    S.w2[i][c] = x;
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < kRL; ++s) {
    const int r = 256 * grp + lane + 32 * s;
    if (r >= r0 && r < m) {
#pragma unroll
      for (int i = 0; i < kSW; ++i) {
        const cplx u = cmul(S.vs[i][r - r0], S.w2[i][col]);  // w2: a shared-memory broadcast
        a[s].x -= u.x;
        a[s].y -= u.y;
      }
    }
  }
  __syncthreads();  // vs is restaged by the next block
}
}  // namespace

// A (column-major, lda, m x n, m >= n, m <= 1024): R (n x n row-major,
// upper) written; V (np panels x 8 columns x ldv, rows relative to the
// panel) and T (np x 64) published; flags (np ints, zeroed by the caller).
__global__ void __launch_bounds__(1024, 1) site_qr_factor_kernel(const cplx* __restrict__ A, int lda, int m, int n,
                                                                 cplx* __restrict__ Vall, int ldv,
                                                                 cplx* __restrict__ Tall, int* __restrict__ flags,
                                                                 cplx* __restrict__ R,
                                                                 unsigned long long* __restrict__ trace) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SiteQrSmem& S = *reinterpret_cast<SiteQrSmem*>(smem_raw);
  const int cta = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, col = warp & 7, grp = warp >> 3;
  const int c0 = kSW * cta, jb = min(kSW, n - c0);
  auto stamp = [&](int k) {  // A/B timeline (tools/qr_case.py with MPSIM_QR_TRACE): %globaltimer ns
    if (trace && t == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      trace[cta * 6 + k] = g;
    }
  };
  stamp(0);
  cplx a[kRL];
#pragma unroll
  for (int s = 0; s < kRL; ++s) {
    const int r = 256 * grp + lane + 32 * s;
    a[s] = (col < jb && r < m) ? A[(long long)(c0 + col) * lda + r] : make_double2(0.0, 0.0);
  }
  for (int p = 0; p < cta; ++p) {
    if (t == 0)
      while (ld_acquire(flags + p) == 0) __nanosleep(20);
    __syncthreads();
    if (p == cta - 1) stamp(1);
    apply_block(S, a, Vall + (long long)p * kSW * ldv, ldv, Tall + (long long)p * kSW * kSW, kSW * p, m, true);
  }
  stamp(2);
  // Two block barriers per reflector: (1) column j's warps publish the raw
  // column (rows >= its diagonal) and partial norms, and the warp owning row
  // dg of every column publishes a_col(dg); (2) every warp forms zlarfg
  // redundantly and its partial x_j^H a_col (v = [1; x / (alpha - beta)], so
  // v^H a = a(dg) + conj(inv) x^H a below the diagonal); after the second
  // barrier the partials are summed and a_col is updated.
  for (int j = 0; j < jb; ++j) {
    const int dg = c0 + j;  // absolute diagonal row of reflector j
    const int pb = j & 1;   // xr / adg buffer: the previous reflector's update may still read the other
    const bool own_dg = dg >= 256 * grp && dg < 256 * grp + 256;
    if (own_dg) {
      cplx x = make_double2(0.0, 0.0);
#pragma unroll
      for (int s = 0; s < kRL; ++s)
        if (256 * grp + 32 * s + (dg & 31) == dg) x = a[s];
      x = make_double2(__shfl_sync(0xffffffffu, x.x, dg & 31), __shfl_sync(0xffffffffu, x.y, dg & 31));
      if (lane == 0) S.adg[pb][col] = x;
    }
    if (col == j) {
      double sn = 0.0;
#pragma unroll
      for (int s = 0; s < kRL; ++s) {
        const int r = 256 * grp + lane + 32 * s;
        if (r > dg && r < m) {
          sn += cabs2(a[s]);
          S.xr[pb][r - c0] = a[s];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sn += __shfl_xor_sync(0xffffffffu, sn, o);
      if (lane == 0) S.pn[grp] = sn;
    }
    __syncthreads();
    if (col == j) {  // zlarfg on column j's warps; tau / inv / beta published with v
      const double sn = (S.pn[0] + S.pn[1]) + (S.pn[2] + S.pn[3]);
      const cplx al = S.adg[pb][j];
      cplx tau = make_double2(0.0, 0.0), inv = make_double2(0.0, 0.0);
      double beta = al.x;
      if (!(sn == 0.0 && al.y == 0.0)) {
        beta = -copysign(sqrt(cabs2(al) + sn), al.x);
        const double rb = 1.0 / beta;
        tau = make_double2((beta - al.x) * rb, -al.y * rb);
        const cplx d = make_double2(al.x - beta, al.y);
        const double rdd = 1.0 / cabs2(d);
        inv = make_double2(d.x * rdd, -d.y * rdd);
      }
      const bool refl = tau.x != 0.0 || tau.y != 0.0;
#pragma unroll
      for (int s = 0; s < kRL; ++s) {  // v_j into the reflector store; R diagonal
        const int r = 256 * grp + lane + 32 * s;
        cplx v = make_double2(0.0, 0.0);
        if (r == dg) {
          v = make_double2(1.0, 0.0);
          if (refl) a[s] = make_double2(beta, 0.0);
        } else if (r > dg && r < m && refl) {
          v = cmul(a[s], inv);
        }
        if (r >= c0 && r < m) S.vs[j][r - c0] = v;
      }
      if (t == 32 * j) {
        S.taus[j] = tau;
        S.inv = inv;
      }
    }
    cplx d = make_double2(0.0, 0.0);  // partial x_j^H a_col (col > j) or v_col^H x_j (col < j), rows > dg
    if (col > j && col < jb) {
#pragma unroll
      for (int s = 0; s < kRL; ++s) {
        const int r = 256 * grp + lane + 32 * s;
        if (r > dg && r < m) cfmac(d, S.xr[pb][r - c0], a[s]);
      }
    } else if (col < j) {
#pragma unroll
      for (int s = 0; s < kRL; ++s) {
        const int r = 256 * grp + lane + 32 * s;
        if (r > dg && r < m) cfmac(d, S.vs[col][r - c0], S.xr[pb][r - c0]);
      }
    }
    if (col != j && col < jb) {
      d = warp_sum(d);
      if (lane == 0) S.part[0][col][grp] = d;
    }
    __syncthreads();
    if (col != j && col < jb) {
      const cplx tau = S.taus[j], inv = S.inv;
      const cplx tot = cadd(cadd(S.part[0][col][0], S.part[0][col][1]), cadd(S.part[0][col][2], S.part[0][col][3]));
      if (col > j) {
        if (tau.x != 0.0 || tau.y != 0.0) {
          // H^H a = a - conj(tau) v (v^H a), v^H a = a(dg) + conj(inv) tot, v = x inv below dg
          const cplx vha = cadd(S.adg[pb][col], cmul(conjc(inv), tot));
          const cplx coef = cmul(make_double2(tau.x, -tau.y), vha);
          const cplx cc = cmul(inv, coef);
#pragma unroll
          for (int s = 0; s < kRL; ++s) {
            const int r = 256 * grp + lane + 32 * s;
            if (r > dg && r < m) {
              const cplx x = S.xr[pb][r - c0];
              a[s].x = fma(-x.x, cc.x, fma(x.y, cc.y, a[s].x));
              a[s].y = fma(-x.x, cc.y, fma(-x.y, cc.x, a[s].y));
            } else if (r == dg) {
              a[s].x -= coef.x;
              a[s].y -= coef.y;
            }
          }
        }
      } else if (grp == 0 && lane == 0) {  // zlarft's v_col^H v_j
        S.gv[col][j] = cadd(conjc(S.vs[col][dg - c0]), cmul(tot, inv));
      }
    }
  }
  stamp(3);
  // columns >= jb of a short last panel: zero reflectors
  for (int jj = jb; jj < kSW; ++jj)
    for (int rr = t; rr < m - c0; rr += 1024) S.vs[jj][rr] = make_double2(0.0, 0.0);
  __syncthreads();
  const int L = m - c0;
  cplx* V = Vall + (long long)cta * kSW * ldv;
#pragma unroll
  for (int jj = 0; jj < kSW; ++jj)
    for (int rr = t; rr < L; rr += 1024) V[(long long)jj * ldv + rr] = S.vs[jj][rr];
  if (warp == 0) {  // zlarft (forward, columnwise)
    for (int j = 0; j < kSW; ++j) {
      cplx v = make_double2(0.0, 0.0);
      if (lane < j && j < jb) {
        for (int q = lane; q < j; ++q) cfma(v, S.ts[lane][q], S.gv[q][j]);
        const cplx tj = S.taus[j];
        v = make_double2(-(tj.x * v.x - tj.y * v.y), -(tj.x * v.y + tj.y * v.x));
      } else if (lane == j && j < jb) {
        v = S.taus[j];
      }
      if (lane < kSW) S.ts[lane][j] = (lane <= j && j < jb) ? v : make_double2(0.0, 0.0);
      __syncwarp();
    }
    if (lane < kSW)
      for (int j = 0; j < kSW; ++j) Tall[(long long)cta * kSW * kSW + lane * kSW + j] = S.ts[lane][j];
  }
  __syncthreads();
  stamp(4);
  if (t == 0) {
    __threadfence();
    st_release(flags + cta, 1);
  }
  stamp(5);
  // R[r][c0 + col] for r <= c0 + col (R is n x n row-major)
  if (col < jb) {
#pragma unroll
    for (int s = 0; s < kRL; ++s) {
      const int r = 256 * grp + lane + 32 * s;
      if (r < n) R[(long long)r * n + c0 + col] = r <= c0 + col ? a[s] : make_double2(0.0, 0.0);
    }
  }
}

// Q = H_0 ... H_{np-1} [I; 0] (m x n): CTA c forms columns [8c, 8c + 8) and
// writes them into the site (left: site[r chi + j] = Q[r][j]; right: site[(j 2 + p) chi + r] = conj(Q[p dr + r][j])).
__global__ void __launch_bounds__(1024, 1) site_qr_q_kernel(int m, int n, const cplx* __restrict__ Vall, int ldv,
                                                            const cplx* __restrict__ Tall, int dl, int dr, int right,
                                                            cplx* __restrict__ site, int chi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SiteQrSmem& S = *reinterpret_cast<SiteQrSmem*>(smem_raw);
  const int cta = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, col = warp & 7, grp = warp >> 3;
  const int c0 = kSW * cta, jb = min(kSW, n - c0);
  const int j = c0 + col;
  cplx a[kRL];
#pragma unroll
  for (int s = 0; s < kRL; ++s) a[s] = make_double2(256 * grp + lane + 32 * s == j ? 1.0 : 0.0, 0.0);
  for (int p = cta; p >= 0; --p)
    apply_block(S, a, Vall + (long long)p * kSW * ldv, ldv, Tall + (long long)p * kSW * kSW, kSW * p, m, false);
  if (col >= jb) return;
#pragma unroll
  for (int s = 0; s < kRL; ++s) {
    const int r = 256 * grp + lane + 32 * s;
    if (r >= m) continue;
    cplx v = a[s];
    if (!right) {
      site[(long long)r * chi + j] = v;
    } else {
      const int pp = r / dr, rr = r % dr;
      v.y = -v.y;
      site[(long long)(j * 2 + pp) * chi + rr] = v;
    }
  }
}

namespace {
unsigned grid_of(long long n) { return (unsigned)std::max(1LL, std::min((n + 255) / 256, 8LL * 148)); }
#define CKQ(x)                                                                             \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
}  // namespace

// persistent kernels: one CTA per 8-column panel, all resident (one per SM)
bool site_qr_supported(int m, int n) { return m >= n && m <= kSL * 32 && n >= 16 && (n + kSW - 1) / kSW <= 148; }

// QR of the site's matricisation (left: (2 Dl x Dr); right: (Dl x 2 Dr)^H):
// R (k x n, row-major) into R, Q (or Q^H) written into the site. Work
// buffers grow as needed. Launched on s.st (panels, look-ahead updates) and
// aux (trailing updates, Q formation); on return aux has been joined back
// into s.st.
// V / T come in two sets used by alternate sites: the Q formation of site i
// runs on `aux` concurrently with the factorisation of site i + 1 (only R
// gates the next site); evs[0] orders Q after the factorisation, evs[1 + set]
// keeps a set from being refactored while its Q formation still reads it.
// The caller joins aux back into s.st at the end of the sweep.
int site_qr(State& s, cplx* site, int dl, int dr, int right, DeviceBuf& Abuf, DeviceBuf& Vbuf, DeviceBuf& Tbuf,
            DeviceBuf& Qbuf, cplx* R, cudaStream_t aux, cudaEvent_t* evs, int set) {
  NvtxRange nv("mpsim: site qr");
  static bool init = false;
  if (!init) {
    CKQ(cudaFuncSetAttribute(site_qr_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SiteQrSmem)));
    CKQ(cudaFuncSetAttribute(site_qr_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SiteQrSmem)));
    init = true;
  }
  const int m = right ? 2 * dr : 2 * dl, n = right ? dl : dr, k = std::min(m, n);
  const int lda = (m + 31) / 32 * 32;
  const int np = (n + kSW - 1) / kSW;
  Abuf.ensure(sizeof(cplx) * (size_t)lda * n);
  Vbuf.ensure(sizeof(cplx) * (size_t)np * kSW * lda);
  Tbuf.ensure(sizeof(cplx) * (size_t)np * kSW * kSW);
  Qbuf.ensure(sizeof(int) * (size_t)np);
  cplx* A = (cplx*)Abuf.p;
  cudaStream_t st = s.st;
  CKQ(cudaStreamWaitEvent(st, evs[1 + set], 0));  // this V / T set's previous Q formation is done
  site_matrix_kernel<<<grid_of((long long)n * m), 256, 0, st>>>(site, s.chi, dl, dr, right, A, lda);
  CKQ(cudaMemsetAsync(Qbuf.p, 0, sizeof(int) * (size_t)np, st));
  static const bool trace_on = ab_knob("MPSIM_QR_TRACE") != nullptr;
  static DeviceBuf tbuf;
  if (trace_on) tbuf.ensure(sizeof(unsigned long long) * 6 * 160);
  site_qr_factor_kernel<<<np, 1024, sizeof(SiteQrSmem), st>>>(A, lda, m, n, (cplx*)Vbuf.p, lda, (cplx*)Tbuf.p,
                                                             (int*)Qbuf.p, R,
                                                             trace_on ? (unsigned long long*)tbuf.p : nullptr);
  if (trace_on) {  // per panel: start, last flag seen, applies done, published (us from launch start)
    std::vector<unsigned long long> h(6 * (size_t)np);
    CKQ(cudaMemcpyAsync(h.data(), tbuf.p, sizeof(unsigned long long) * 6 * np, cudaMemcpyDeviceToHost, st));
    CKQ(cudaStreamSynchronize(st));
    unsigned long long t0 = h[0];
    for (int c = 0; c < np; ++c) t0 = std::min(t0, h[6 * c]);
    std::fprintf(stderr, "[qr trace m=%d n=%d]", m, n);
    for (int c = 0; c < np; c += std::max(1, np / 16)) {
      std::fprintf(stderr, " %d:", c);
      for (int k = 0; k < 6; ++k)
        std::fprintf(stderr, "%s%.1f", k ? "/" : "", (k == 1 && c == 0) ? 0.0 : (h[6 * c + k] - t0) * 1e-3);
    }
    std::fprintf(stderr, "\n");
  }
  CKQ(cudaEventRecord(evs[0], st));
  CKQ(cudaStreamWaitEvent(aux, evs[0], 0));
  site_qr_q_kernel<<<np, 1024, sizeof(SiteQrSmem), aux>>>(m, n, (const cplx*)Vbuf.p, lda, (const cplx*)Tbuf.p, dl,
                                                         dr, right, site, s.chi);
  CKQ(cudaEventRecord(evs[1 + set], aux));
  s.launches += 3;
  return k;
}

}  // namespace mpsim_gpu
