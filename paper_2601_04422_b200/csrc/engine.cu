// Host-side engine: the HBM site store, the layer scheduler that turns a
// brick layer of disjoint gates into one batched launch sequence, the
// transfer-matrix queries, and the extern "C" boundary (include/mpsim_gpu.h).
//
// Reference correspondence (paths relative to /root/reference/proj):
//   MpsState                     include/mpsim/mps.hpp:33-75, src/mps.cpp
//   apply_1q / apply_2q_local    src/gate_apply.cpp:99-147
//   apply_2q_swap                src/gate_apply.cpp:149-179
//   execute_serial / _parallel   src/executor.cpp:73-232
//   decompose_nonlocal/layerize  src/fusion.cpp:137-190
//   norm/amplitude/overlap/...   src/mps.cpp:189-256
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

// ---- launchers implemented in the kernel translation units
int launch_theta(const GateDesc*, const GateDesc*, int, int, const cplx*, long long, int, cplx*, double*, CUtensorMap*,
                 CUtensorMap*, cudaStream_t);
int theta_tiles(int dl, int dr);
void jacobi_split_init();
#ifdef MPSIM_AB_KNOBS
void jacobi_phase_clocks(unsigned long long*, bool);
void jacobi_w32_phase_clocks(unsigned long long*, bool);
#endif
void launch_jacobi_sweep(const GateDesc*, int, int, cplx*, const int*, int*, double, double, const double*, double,
                         const int*, long long, double*, int*, cplx*, cplx*, double*, cplx*, int*, int, int,
                         cudaStream_t);
// L2 eviction priorities in the persistent sweep (jacobi_split.cu RoundArgs::l2hint).
static int l2hint_policy() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_L2HINT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
// One persistent launch per sweep (jacobi_split.cu); MPSIM_SWEEP=rounds selects
// one launch per tournament round.
static bool sweep_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_SWEEP");
    return !(v != nullptr && std::string(v) == "rounds");
  }();
  return on;
}
void launch_jacobi_sweep_cl(const GateDesc*, int, int, cplx*, const int*, const int*, int, int, int*, double, double,
                            const double*, double, const int*, long long, double*, int*, double*, cplx*, int*,
                            cudaStream_t);
// Persistent sweeps with one CTA per visit over the whole layer (default), or
// as 4-CTA cluster visits claimed gate group by gate group (MPSIM_SWEEP_CL=1).
static bool cluster_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_SWEEP_CL");
    return v != nullptr && std::string(v) == "1";
  }();
  return on;
}
// Gates per claim group of the cluster sweep: the group's operands (16 MB per
// gate at chi = 512) stay in L2 between rounds.
static int group_policy() {
  static const int g = [] {
    const char* v = ab_knob("MPSIM_GROUP");
    const int x = v ? std::atoi(v) : 0;
    return x > 0 ? x : 6;
  }();
  return g;
}
void launch_jacobi_sweep_w32(const GateDesc*, int, int, cplx*, const int*, int*, double, double, const double*, double,
                             const int*, long long, double*, double*, cplx*, int*, cudaStream_t);
// Persistent sweeps with 32-vector blocks (jacobi_w32.cu) for batches whose
// largest operand has at least kW32MinN vectors (every n_pad is a multiple of
// 64). Measured (profiles/sweep_ab_r02.txt): half the DRAM
// traffic per sweep keeps the SM clock off the power cap (1965 MHz vs
// 1717-1845 for 16-vector blocks): with the symmetric EVD update, the cross
// test, three-product cross Grams and two-in-three cross-only EVD rounds,
// 1024-vector thetas (chi = 512) run 119-120 gates/s vs 115 on the same box,
// 2048-vector thetas (chi = 1024) 16.5 vs 14.7. 256-vector thetas (C2) keep
// 16-vector blocks for their amplitude margin.
// A/B: MPSIM_W32=0 never, =1 from 512 vectors.
constexpr int kW32MinN = 1024;
// Vector-count padding of gate and plain-SVD operands (a multiple of both
// block pair widths, so either sweep kernel can run the batch).
constexpr int kNAlign = 64;
static int w32_min_n() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_W32");
    if (e == nullptr) return kW32MinN;
    return std::string(e) == "0" ? (1 << 30) : 512;
  }();
  return v;
}
// Pair EVDs with FP32 Gram updates (bit 64) in the first sweep and in sweeps
// whose predecessor's largest relative off-diagonal exceeded this; 0 = off
// (A/B: MPSIM_EVD32_MAXOFF).
constexpr int kEvd32MinN = 512;  // (operands with fewer vectors keep the FP64 inner sweep)
static double evd32_maxoff() {
  static const double v = [] {
    const char* e = ab_knob("MPSIM_EVD32_MAXOFF");
    return e ? std::atof(e) : 0.0;
  }();
  return v;
}
// Relative orthogonality a pair must reach (times max(sqrt(m), 32)): 4 eps;
// A/B: MPSIM_JTOL (in units of eps).
static double jacobi_tol() {
  static const double v = [] {
    const char* e = ab_knob("MPSIM_JTOL");
    return (e ? std::atof(e) : 4.0) * 2.220446049250313e-16;
  }();
  return v;
}
void launch_orthonormalize(const GateDesc*, int, int, int, cplx*, const double*, const int*, long long,
                           const GateOut*, const double*, double, float2*, float2*, long long, cudaStream_t);
// First-order orthonormalisation of the kept vectors before the split
// (split.cu); A/B: MPSIM_ORTHO=0 skips it.
static bool ortho_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_ORTHO");
    return !(v != nullptr && std::string(v) == "0");
  }();
  return on;
}
void qrp_init();
void split_init();
void theta_init();
void launch_qr_factor(const GateDesc*, int, int, int, cplx*, cplx*, long long, cplx*, int, int, cudaStream_t);
void launch_qr_apply(const GateDesc*, int, int, int, cplx*, const cplx*, long long, const cplx*, int, const int*,
                     long long, const GateOut*, cudaStream_t);
// QR preconditioning (qr_pre.cu) of gates whose SVD operand has at least
// kQrMinN vectors: MPSIM_QR=2 (default) two QR steps, 1 one, 0 none.
constexpr int kQrMinN = 128;
constexpr int kMaxSvdN = kMaxSortN;  // derijk_kernel / truncate_kernel: one CTA, keys in shared memory
// Default: two steps. A/B: MPSIM_QR=0, 1, 2, 4 force that many steps; -1 =
// four for operands with >= kQr4MinN vectors (measured at chi = 512: 10 sweep
// launches per layer instead of 11, but the bench step 1.3 % slower — the two
// extra QR steps cost more than the sweep they save).
constexpr int kQr4MinN = 512;
static int qr_policy() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_QR");
    if (e == nullptr) return 2;
    const int x = std::atoi(e);
    return x < 0 ? -1 : (x >= 4 ? 4 : (x > 2 ? 2 : x));
  }();
  return v;
}
void launch_jacobi_round_split(const GateDesc*, int, int, cplx*, const int*, int*, int, double, double, const double*,
                               double, const int*, long long, double*, int*, cplx*, cplx*, double*, int, cplx*,
                               int, cudaStream_t);
// Cross-only pair EVDs (evd.cuh) in a sweep whose predecessor measured an rms
// relative off-norm above this (the pre-asymptotic phase); MPSIM_CROSS=0 disables.
constexpr double kCrossRmsDefault = 0.35;
constexpr int kCrossSweepsDefault = 4;  // cross-only EVDs in sweeps 1 .. kCrossSweeps - 1 at most
// (MPSIM_CROSS_RMS / MPSIM_CROSS_SWEEPS override both, A/B only)
static double cross_rms() {
  static const double v = [] {
    const char* e = ab_knob("MPSIM_CROSS_RMS");
    return e ? std::atof(e) : kCrossRmsDefault;
  }();
  return v;
}
static int cross_sweeps() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_CROSS_SWEEPS");
    return e ? std::atoi(e) : kCrossSweepsDefault;
  }();
  return v;
}
// Stored in-block Grams while the previous sweep's largest relative
// off-diagonal exceeds this; MPSIM_INBLOCK=0 disables.
constexpr double kInblockMaxoff = 1e-4;
static bool inblock_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_INBLOCK");
    return !(v != nullptr && v[0] == '0');
  }();
  return on;
}
static bool cross_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_CROSS");
    return !(v != nullptr && v[0] == '0');
  }();
  return on;
}
// Jacobi round implementation: default = the whole pair visit in one kernel
// (one persistent launch per sweep, see sweep_policy); "split2" (Gram + pair
// EVD / rotation) and "split3" (Gram / EVD / rotation) launch per round (A/B).
static int jacobi_mode() {
  static const int m = [] {
    const char* v = ab_knob("MPSIM_JACOBI");
    if (v != nullptr && std::string(v) == "split3") return 2;
    if (v != nullptr && std::string(v) == "split2") return 3;
    return 4;
  }();
  return m;
}
void launch_derijk(const GateDesc*, int, const cplx*, const int*, int*, long long, int, cudaStream_t);
void launch_norms(const GateDesc*, int, int, const cplx*, double*, long long, cudaStream_t);
void launch_truncate(const GateDesc*, int, double*, int*, long long, GateOut*, const double*, double, int,
                     cudaStream_t);
void launch_write_factors(const GateDesc*, int, int, int, int, const cplx*, const double*, const int*, long long,
                          const GateOut*, const double*, double, cudaStream_t);
void launch_apply1q(const Gate1Desc*, int, long long, cplx*, long long, int, cudaStream_t);
void launch_regrow(const cplx*, long long, int, cplx*, long long, int, const int*, int, cudaStream_t);
void launch_cgemm(const GemmArgs&, cudaStream_t);
void launch_amp_step(const cplx*, long long, cplx*, long long, const char*, int, int, int, const cplx*, int, int,
                     int, cudaStream_t);
void launch_fill(cplx*, long long, cplx, cudaStream_t);

Error::Error(int c, std::string m) : std::runtime_error(std::move(m)), code(c) {}

[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }

std::string& last_error_slot() {
  thread_local std::string s;
  return s;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// MPSIM_SYNC_DEBUG=1 synchronises after every checked launch so a device
// fault is attributed to the kernel that raised it.
static bool sync_debug() {
  static const bool on = [] {
    const char* v = std::getenv("MPSIM_SYNC_DEBUG");
    return v != nullptr && v[0] == '1';
  }();
  return on;
}

// MPSIM_PHASE_PROBE=1|2 (profiling only): Jacobi rounds stop after the Gram
// (1) or after the pair EVD (2), with a single sweep, to time the phases.
static int phase_probe() {
  static const int v = [] {
    const char* e = ab_knob("MPSIM_PHASE_PROBE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

#ifndef MPSIM_W32_ALT
#define MPSIM_W32_ALT 3
#endif
constexpr int kW32AltCross = MPSIM_W32_ALT;
// Cross-block-only pair EVDs outside a period of rounds in the asymptotic
// sweeps: MPSIM_ALT_CROSS=2 (odd rounds, default), 3 (two rounds in three)
// or 0 (full EVDs every round, A/B). Returns the active bits to add.
// The 32-vector-block sweep defaults to two rounds in three: its 64 x 64 full
// EVD is relatively dearer (chi = 1024: +0.55 % for one more sweep launch per
// three layers, parity green; profiles/sweep_ab_r02.txt). MPSIM_W32_ALT_CROSS (A/B).
static int alt_cross_bits(bool w32 = false) {
  if (w32) {
    static const int bits32 = [] {
      const char* v = ab_knob("MPSIM_W32_ALT_CROSS");
      const int p = v ? std::atoi(v) : kW32AltCross;
      return p == 2 ? 16 : p == 3 ? (16 | 32) : 0;
    }();
    return bits32;
  }
  static const int bits = [] {
    const char* v = ab_knob("MPSIM_ALT_CROSS");
    const int p = v ? std::atoi(v) : 2;
    return p == 2 ? 16 : p == 3 ? (16 | 32) : 0;
  }();
  return bits;
}

// MPSIM_FIRST_INBLOCK=0 computes every Gram tile in the first sweep (A/B).
static bool first_sweep_inblock() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_FIRST_INBLOCK");
    return !(v != nullptr && v[0] == '0');
  }();
  return on;
}

// MPSIM_EXACT_CACHE=0 recomputes all 36 Gram tiles in closing sweeps (A/B).
static bool exact_cache_policy() {
  static const bool on = [] {
    const char* v = ab_knob("MPSIM_EXACT_CACHE");
    return !(v != nullptr && v[0] == '0');
  }();
  return on;
}

// MPSIM_SWEEP_DEBUG=1 prints per-sweep Jacobi convergence to stderr.
static bool sweep_debug() {
  static const bool on = [] {
    const char* v = std::getenv("MPSIM_SWEEP_DEBUG");
    return v != nullptr && v[0] == '1';
  }();
  return on;
}

static void check_launch(const char* what = "kernel") {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_debug()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) fail(MPSIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void DeviceBuf::ensure(size_t b) {
  if (b <= bytes) return;
  size_t nb = std::max(b, bytes + bytes / 2);
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  if (cudaMalloc(&p, nb) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&p, b) != cudaSuccess) {
      cudaGetLastError();
      fail(MPSIM_ECUDA, "device allocation of " + std::to_string(b) + " bytes failed");
    }
    nb = b;
  }
  bytes = nb;
}
void DeviceBuf::release() {
  if (p) {
    int dev = -1;  // the owning device may not be current (multi-GPU hosts)
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess) dev = a.device;
    cudaGetLastError();
    int cur = -1;
    cudaGetDevice(&cur);
    if (dev >= 0 && dev != cur) cudaSetDevice(dev);
    cudaFree(p);
    if (dev >= 0 && dev != cur) cudaSetDevice(cur);
  }
  p = nullptr;
  bytes = 0;
}
void PinnedBuf::ensure(size_t b) {
  if (b <= bytes) return;
  if (p) cudaFreeHost(p);
  p = nullptr;
  size_t nb = std::max(b, bytes + bytes / 2);
  CK(cudaMallocHost(&p, nb));
  bytes = nb;
}
void PinnedBuf::release() {
  if (p) cudaFreeHost(p);
  p = nullptr;
  bytes = 0;
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  if (prev != dev) CK(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != prev) cudaSetDevice(prev);
}

static int next_pow2(long long x) {
  int c = 1;
  while (c < x) c <<= 1;
  return c;
}

}  // namespace mpsim_gpu

using namespace mpsim_gpu;
using cd = std::complex<double>;

// ============================================================== state

State::State(int n_, long long chi_hint, int dev) : n(n_), device(dev) {
  if (n_ < 1) fail(MPSIM_EINVAL, "state needs at least one qubit");
  DeviceGuard g(dev);
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventCreate(&evj0));
  CK(cudaEventCreate(&evj1));
  {
    // split-K GEMM workspaces (queries.cu) come from the stream-ordered pool:
    // keep up to 1 GiB cached across stream syncs instead of trimming it
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  static bool inited = false;
  if (!inited) {
    jacobi_split_init();
    qrp_init();
    split_init();
    theta_init();
    inited = true;
  }
  chi = next_pow2(std::max<long long>(2, std::min<long long>(chi_hint, 1 << 14)));
  stride = (long long)chi * 2 * chi;
  sites_buf.ensure((size_t)n * stride * sizeof(cplx));
  sites = (cplx*)sites_buf.p;
  // |0...0>: every site (1,2,1) = [1, 0] (mps.cpp:99-110)
  CK(cudaMemsetAsync(sites, 0, (size_t)n * stride * sizeof(cplx), st));
  launch_fill_sites_zero_state();
  bonds.assign((size_t)n + 1, 1);
  sdl.assign((size_t)n, 1);
  sdr.assign((size_t)n, 1);
  CK(cudaStreamSynchronize(st));
}

void State::launch_fill_sites_zero_state() {
  // element (0,0,0) of every site = 1: a strided 2D copy from a pinned pattern.
  const cplx one = make_double2(1.0, 0.0);
  h_small.ensure(sizeof(cplx) * (size_t)n);
  cplx* h = (cplx*)h_small.p;
  for (int i = 0; i < n; ++i) h[i] = one;
  CK(cudaMemcpy2DAsync(sites, stride * sizeof(cplx), h, sizeof(cplx), sizeof(cplx), n, cudaMemcpyHostToDevice, st));
}

State::~State() {
  DeviceGuard g(device);
  cudaStreamSynchronize(st);
  // every DeviceBuf / PinnedBuf member frees itself (RAII)
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaEventDestroy(evj0);
  cudaEventDestroy(evj1);
  if (aux) {
    cudaStreamSynchronize(aux);
    cudaStreamDestroy(aux);
  }
  for (cudaEvent_t e : evq)
    if (e) cudaEventDestroy(e);
  cudaStreamDestroy(st);
}

void State::grow(int new_chi) {
  if (new_chi <= chi) return;
  DeviceGuard g(device);
  const long long nstride = (long long)new_chi * 2 * new_chi;
  DeviceBuf nb;
  nb.ensure((size_t)n * nstride * sizeof(cplx));
  CK(cudaMemsetAsync(nb.p, 0, (size_t)n * nstride * sizeof(cplx), st));
  std::vector<int> dims(2 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    dims[2 * i] = (int)sdl[i];
    dims[2 * i + 1] = (int)sdr[i];
  }
  DeviceBuf dd;
  dd.ensure(dims.size() * sizeof(int));
  CK(cudaMemcpyAsync(dd.p, dims.data(), dims.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  launch_regrow(sites, stride, chi, (cplx*)nb.p, nstride, new_chi, (const int*)dd.p, n, st);
  check_launch();
  ++launches;
  CK(cudaStreamSynchronize(st));
  sites_buf = std::move(nb);
  sites = (cplx*)sites_buf.p;
  chi = new_chi;
  stride = nstride;
}

static void check_policy(const mpsim_policy& p) {  // gate_apply.cpp:26-33
  if (p.max_bond < 1) fail(MPSIM_EINVAL, "truncation policy needs max_bond >= 1");
  if (!(p.cutoff >= 0.0 && p.cutoff < 1.0)) fail(MPSIM_EINVAL, "truncation cutoff must lie in [0, 1)");
}

static void update_center(State& s, int lo, int hi) {  // gate_apply.cpp:70-77
  if (s.center < 0) return;
  s.center = (s.center >= lo && s.center <= hi) ? hi : -1;
}

// ============================================================== layer execution

namespace {

struct G2 {
  int q;
  cplx u[16];
  int idx;
};
struct G1 {
  int q;
  cplx u[4];
  int idx;
};
struct Rep {
  double w = 0.0;
  long long k = 1;
  int svd = 0;
};

constexpr int kMaxSweeps = 60;
constexpr double kEps = 2.220446049250313e-16;
// Rounding-noise floor for Jacobi vectors: sigma^2 <= (64 eps)^2 ||theta||_F^2.
constexpr double kFloorRel2 = (64.0 * kEps) * (64.0 * kEps);
// Largest relative off-diagonal entering a sweep after which that sweep's
// rotations are final (quadratic convergence; see run_two_chunk).
// (1e-9 measured too loose: on the C4 window's truncating 2048 x 2048 thetas
// the kept subspace then sat 4e-11..2e-9 from LAPACK's at relative gaps of
// 0.75..0.07, since the rounding of the final sweep's own rotations keeps the
// convergence short of quadratic; at 1e-12 it is 3e-14, LAPACK's level)
constexpr double kQuadFinish = 1e-12;
// A/B: MPSIM_QUAD overrides kQuadFinish (0 disables the quadratic-phase exit).
static double quad_finish() {
  static const double v = [] {
    const char* e = ab_knob("MPSIM_QUAD");
    return e ? std::atof(e) : kQuadFinish;
  }();
  return v;
}

}  // namespace

// Runs the batched Jacobi SVD + truncation + split for the descriptors: the
// operand comes from the theta kernel (src == nullptr) or from a row-major
// device matrix (plain SVDs, bond-propagation carriers); descriptors with
// pre = 1 are QR-preconditioned (qr_pre.cu) before the sweeps.
int mpsim_gpu::use_qr_precondition(int n) {
  if (n < kQrMinN) return 0;
  const int p = qr_policy();
  return p >= 0 ? p : (n >= kQr4MinN ? 4 : 2);
}

// The descriptor as each phase of run_two_chunk sees it (desc_layout holds the
// Jacobi-phase view): 0 theta / load + first QR (R^H -> y2 for pre = 2),
// 1 second QR (pre = 2 only), 2 Jacobi sweeps, 3 Z = Q1 [X; 0] (pre = 2 only),
// 4 split epilogue.
// pre = 4 adds 5 third QR (y3 -> R3^H into y4), 6 fourth QR (y4 -> R4^H
// into X), 7 Q3 applied to the kept X (into y3, before phase 3 maps y3 by Q1).
static GateDesc phase_desc(const GateDesc& d, int phase) {
  GateDesc e = d;
  auto qr_on = [&](long long off) {
    e.qr_off = off;
    e.qr_m = d.n;
    e.qr_m_pad = d.m_pad;
  };
  if (d.pre >= 2) {
    if (phase == 0) {
      e.ws_off = d.y2_off;
    } else if (phase == 1) {
      qr_on(d.y2_off);
      if (d.pre == 4) e.ws_off = d.y3_off;
    } else if (phase == 3 && d.pre == 4) {
      e.ws_off = d.y3_off;  // Q3 X_kept, already in kept order
      e.zsrc_ordered = 1;
    } else if (phase == 4) {
      e.ws_off = d.qr_off;
      e.m = d.qr_m;
      e.m_pad = (int)d.qr_m_pad;
    } else if (phase == 5 || phase == 6 || phase == 7) {
      if (d.pre != 4) {
        e.pre = 0;
      } else if (phase == 5) {
        qr_on(d.y3_off);
        e.ws_off = d.y4_off;
      } else if (phase == 6) {
        qr_on(d.y4_off);
      } else {
        qr_on(d.y3_off);
      }
    }
  } else if (phase == 1 || phase == 3 || phase >= 5) {
    e.pre = 0;
  }
  return e;
}
constexpr int kPhases = 8;

void mpsim_gpu::run_two_chunk(State& s, const std::vector<GateDesc>& descs, std::vector<GateOut>& outs,
                              const cplx* src, long long src_ld) {
  NvtxRange nv("mpsim: theta + svd + truncate (apply_2q_local batch)");
  const int ng = (int)descs.size();
  for (const GateDesc& d : descs)
    if (d.n_pad > kMaxSvdN)  // de Rijk / truncation sort one gate's vectors in one CTA
      fail(MPSIM_EINVAL, "SVD operand with " + std::to_string(d.n) + " vectors (min dimension) exceeds the " +
                             std::to_string(kMaxSvdN) + " this build supports (bond dimension <= 8192)");
  long long ws_elems = 0;
  int max_tiles = 1, max_nb = 2, max_m = 1, max_n = 1;
  int max_n0 = 1, qr_n_pad = 0, qr_m_pad = 0, qr_jm_pad = 0, max_out_m = 1, max_out_m_pad = 1;
  bool any_pre2 = false, any_pre4 = false;
  for (const GateDesc& d : descs) {
    long long end = d.x0_off + (long long)d.n_pad * d.x0_ld;
    if (d.pre == 1) end = d.qr_off + (long long)d.n_pad * d.qr_m_pad;
    if (d.pre == 2) end = d.y2_off + (long long)d.n_pad * d.m_pad;
    if (d.pre == 4) end = d.y4_off + (long long)d.n_pad * d.m_pad;
    ws_elems = std::max(ws_elems, end);
    max_n0 = std::max(max_n0, d.n0);
    if (d.pre) {
      qr_n_pad = std::max(qr_n_pad, d.n_pad);
      qr_m_pad = std::max(qr_m_pad, (int)d.qr_m_pad);
      qr_jm_pad = std::max(qr_jm_pad, d.m_pad);
    }
    any_pre2 = any_pre2 || d.pre >= 2;
    any_pre4 = any_pre4 || d.pre == 4;
    max_tiles = std::max(max_tiles, theta_tiles(d.dl, d.dr));
    max_nb = std::max(max_nb, d.nb);
    max_m = std::max(max_m, d.m);
    max_n = std::max(max_n, d.n);
    max_out_m = std::max(max_out_m, phase_desc(d, 4).m);
    max_out_m_pad = std::max(max_out_m_pad, phase_desc(d, 4).m_pad);
  }
  const long long sig_stride = ((max_n + 31) / 32) * 32;
  long long perm_stride = 32;
  for (const GateDesc& d : descs) perm_stride = std::max<long long>(perm_stride, d.n_pad);
  s.d_perm.ensure(sizeof(int) * perm_stride * ng);
  s.ws.ensure((size_t)ws_elems * sizeof(cplx));
  s.d_gates.ensure(sizeof(GateDesc) * kPhases * ng);
  s.d_out.ensure(sizeof(GateOut) * ng);
  s.d_sigma.ensure(sizeof(double) * sig_stride * ng);
  s.d_order.ensure(sizeof(int) * sig_stride * ng);
  s.d_active.ensure(sizeof(int) * 2 * ng);  // active flags, then the active-gate list
  s.d_rot.ensure(sizeof(int) * ng);
  s.d_frob.ensure(sizeof(double) * ng);
  s.h_gates.ensure(sizeof(GateDesc) * kPhases * ng);
  s.h_out.ensure(sizeof(GateOut) * ng);
  s.h_rot.ensure(sizeof(int) * 2 * ng);
  {
    GateDesc* h = (GateDesc*)s.h_gates.p;
    for (int ph = 0; ph < kPhases; ++ph)
      for (int i = 0; i < ng; ++i) h[ph * ng + i] = phase_desc(descs[i], ph);
  }
  cudaStream_t st = s.st;
  CK(cudaMemcpyAsync(s.d_gates.p, s.h_gates.p, sizeof(GateDesc) * kPhases * ng, cudaMemcpyHostToDevice, st));
  s.h2d_bytes += (long long)sizeof(GateDesc) * kPhases * ng + (long long)sizeof(int) * ng;
  CK(cudaMemsetAsync(s.ws.p, 0, (size_t)ws_elems * sizeof(cplx), st));
  const GateDesc* dph = (const GateDesc*)s.d_gates.p;
  const GateDesc* dg = dph + 2 * ng;  // Jacobi phase
  cplx* ws = (cplx*)s.ws.p;
  CK(cudaMemsetAsync(s.d_frob.p, 0, sizeof(double) * ng, st));
  if (src == nullptr) {
    s.h_maps.ensure(sizeof(CUtensorMap) * 2 * ng);
    s.d_maps.ensure(sizeof(CUtensorMap) * 2 * ng);
    const int tv = launch_theta(dph, (const GateDesc*)s.h_gates.p, ng, max_tiles, s.sites, s.stride, s.chi, ws,
                                (double*)s.d_frob.p, (CUtensorMap*)s.h_maps.p, (CUtensorMap*)s.d_maps.p, st);
    if (tv == 0) s.h2d_bytes += (long long)sizeof(CUtensorMap) * 2 * ng;
    check_launch("theta_kernel");
    ++s.launches;
  } else {
    // A device-resident row-major matrix (plain SVDs, bond-propagation carriers)
    const GateDesc d = phase_desc(descs[0], 0);
    const int big = d.pre ? d.qr_m : d.m;
    launch_load_matrix(src, src_ld, d.trans == 0 ? big : d.n, d.trans == 0 ? d.n : big, d.trans,
                       ws + (d.pre ? d.qr_off : d.ws_off), d.pre ? d.qr_m_pad : d.m_pad, d.pre ? 0 : 1, d.f,
                       ws + d.x0_off, d.x0_ld,
                       (double*)s.d_frob.p, st);
    check_launch("load_matrix_kernel");
    ++s.launches;
  }
  const int npan = qr_n_pad / 32;
  if (qr_n_pad > 0) {
    // first QR (its reflectors stay in d_qrv / d_qrt for Z = Q1 [X; 0])
    s.d_qrv.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * qr_m_pad);
    s.d_qrt.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * 32);
    launch_qr_factor(dph, ng, qr_n_pad, qr_jm_pad, ws, (cplx*)s.d_qrv.p, qr_m_pad, (cplx*)s.d_qrt.p, npan, 0, st);
    check_launch("qr_factor");
    s.launches += 2 * npan;
  }
  if (any_pre2) {
    s.d_qrv2.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * qr_jm_pad);
    s.d_qrt2.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * 32);
    launch_qr_factor(dph + ng, ng, qr_n_pad, qr_jm_pad, ws, (cplx*)s.d_qrv2.p, qr_jm_pad, (cplx*)s.d_qrt2.p, npan,
                     1, st);
    check_launch("qr_factor (second step)");
    s.launches += 2 * npan;
  }
  if (any_pre4) {
    // third step (reflectors kept for Z), fourth step (scratch reflectors)
    s.d_qrv3.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * qr_jm_pad);
    s.d_qrt3.ensure(sizeof(cplx) * (size_t)ng * npan * 32 * 32);
    launch_qr_factor(dph + 5 * ng, ng, qr_n_pad, qr_jm_pad, ws, (cplx*)s.d_qrv3.p, qr_jm_pad, (cplx*)s.d_qrt3.p,
                     npan, 1, st);
    launch_qr_factor(dph + 6 * ng, ng, qr_n_pad, qr_jm_pad, ws, (cplx*)s.d_qrv2.p, qr_jm_pad, (cplx*)s.d_qrt2.p,
                     npan, 1, st);
    check_launch("qr_factor (third / fourth step)");
    s.launches += 4 * npan;
  }

  int* h_rot = (int*)s.h_rot.p;
  bool use_w32 = max_nb * kW >= w32_min_n();
  for (const GateDesc& d : descs) use_w32 = use_w32 && d.n_pad % (4 * kW) == 0;
  const bool w32_sweeps = use_w32 && jacobi_mode() == 4 && sweep_policy() && !phase_probe();
  // The first sweep of a fresh theta is pre-asymptotic: it reuses the pair
  // EVDs' in-block Grams from round 1 on (bit 4) like the sweeps the maxoff
  // policy below flags. It cannot end the iteration through kQuadFinish (its
  // maxoff saw in-block values that may be stale); only a sweep without any
  // rotation — whose Grams were then all computed exactly — ends it.
  const int first = ((jacobi_mode() >= 3 && inblock_policy() && first_sweep_inblock()) ? (1 | 4) : 1) |
                    alt_cross_bits(w32_sweeps) | (evd32_maxoff() > 0.0 ? 64 : 0);
  for (int i = 0; i < ng; ++i) h_rot[i] = descs[i].n >= kEvd32MinN ? first : first & ~64;
  int n_list = 0;
  // flags h_rot[0, ng) -> device, with the list of active gates after them
  // (the cluster sweep claims its visits gate group by gate group over it)
  auto upload_active = [&]() {
    n_list = 0;
    for (int i = 0; i < ng; ++i)
      if (h_rot[i]) h_rot[ng + n_list++] = i;
    CK(cudaMemcpyAsync(s.d_active.p, h_rot, sizeof(int) * (ng + n_list), cudaMemcpyHostToDevice, st));
  };
  upload_active();
  bool converged = false;
  std::vector<int> still(ng, 1);
  s.d_maxoff.ensure(sizeof(double) * ng);
  {
    const size_t slots = (size_t)ng * (max_nb / 2);
    s.d_need.ensure(sizeof(int) * slots);
    s.d_gbuf.ensure(sizeof(cplx) * slots * kP * kP);
    s.d_rbuf.ensure(sizeof(cplx) * slots * kP * kP);
    s.d_gblk.ensure(sizeof(cplx) * slots * 2 * kW * kW * 2);  // (twice: 32 x 32 blocks of the W = 32 sweep)
  }
  s.h_maxoff.ensure(sizeof(double) * ng);
  double* h_maxoff = (double*)s.h_maxoff.p;
  s.d_offsum.ensure(sizeof(double) * ng);
  s.h_offsum.ensure(sizeof(double) * ng);
  double* h_offsum = (double*)s.h_offsum.p;
  const int max_sweeps = phase_probe() ? 1 : kMaxSweeps;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    NvtxRange nvs("mpsim: jacobi sweep");
    CK(cudaMemsetAsync(s.d_rot.p, 0, sizeof(int) * ng, st));
    CK(cudaMemsetAsync(s.d_maxoff.p, 0, sizeof(double) * ng, st));
    CK(cudaMemsetAsync(s.d_offsum.p, 0, sizeof(double) * ng, st));
    launch_derijk(dg, ng, ws, (const int*)s.d_active.p, (int*)s.d_perm.p, perm_stride, (int)perm_stride, st);
    ++s.launches;
    CK(cudaEventRecord(s.evj0, st));
    // One cyclic sweep of the inner 2W x 2W eigensolver per pair visit: the
    // outer iteration needs the same number of sweeps as with a fully
    // converged inner EVD (measured in emulation and on the B200), at a
    // fraction of the cost. Final orthogonality is at the tol level.
    // (phase probes 1-2 run per round; probe 4, the visit without its EVD, runs persistent)
    const bool persistent = jacobi_mode() == 4 && sweep_policy();
    const double jtol = jacobi_tol();
    if (persistent && use_w32 && !phase_probe()) {
      s.d_sweepctl.ensure(sizeof(int) * (1 + 2 * (size_t)ng * max_nb));
      launch_jacobi_sweep_w32(dg, ng, max_nb / 4, ws, (const int*)s.d_active.p, (int*)s.d_rot.p, 4.0 * kEps,
                              2.0 * kEps, (const double*)s.d_frob.p, kFloorRel2, (const int*)s.d_perm.p, perm_stride,
                              (double*)s.d_maxoff.p, (double*)s.d_offsum.p, (cplx*)s.d_gblk.p,
                              (int*)s.d_sweepctl.p, st);
      s.launches += 1;
      ++s.jacobi_launches;
    } else if (persistent && cluster_policy() && !phase_probe()) {
      s.d_sweepctl.ensure(sizeof(int) * (1 + 2 * (size_t)ng * max_nb));
      launch_jacobi_sweep_cl(dg, ng, max_nb / 2, ws, (const int*)s.d_active.p, (const int*)s.d_active.p + ng, n_list,
                             group_policy(), (int*)s.d_rot.p, jtol, 2.0 * kEps, (const double*)s.d_frob.p,
                             kFloorRel2, (const int*)s.d_perm.p, perm_stride, (double*)s.d_maxoff.p,
                             (int*)s.d_need.p, (double*)s.d_offsum.p, (cplx*)s.d_gblk.p, (int*)s.d_sweepctl.p, st);
      s.launches += 1;
      ++s.jacobi_launches;
    } else if (persistent) {
      s.d_sweepctl.ensure(sizeof(int) * (1 + 2 * (size_t)ng * max_nb));
      launch_jacobi_sweep(dg, ng, max_nb / 2, ws, (const int*)s.d_active.p, (int*)s.d_rot.p, jtol, 2.0 * kEps,
                          (const double*)s.d_frob.p, kFloorRel2, (const int*)s.d_perm.p, perm_stride,
                          (double*)s.d_maxoff.p, (int*)s.d_need.p, (cplx*)s.d_gbuf.p, (cplx*)s.d_rbuf.p,
                          (double*)s.d_offsum.p, (cplx*)s.d_gblk.p, (int*)s.d_sweepctl.p, phase_probe(), l2hint_policy(), st);
      s.launches += 1;
      ++s.jacobi_launches;
    }
    for (int round = 0; round < (persistent ? 0 : max_nb - 1); ++round) {
      // (per-round launches: A/B and phase probes)
      {
        launch_jacobi_round_split(dg, ng, max_nb / 2, ws, (const int*)s.d_active.p, (int*)s.d_rot.p, round,
                                  jtol, 2.0 * kEps, (const double*)s.d_frob.p, kFloorRel2,
                                  (const int*)s.d_perm.p, perm_stride, (double*)s.d_maxoff.p, (int*)s.d_need.p,
                                  (cplx*)s.d_gbuf.p, (cplx*)s.d_rbuf.p, (double*)s.d_offsum.p, jacobi_mode() - 2,
                                  (cplx*)s.d_gblk.p, phase_probe(), st);
        s.launches += 4 - jacobi_mode();  // kernels per round beyond the one counted below
      }
      ++s.launches;
      ++s.jacobi_launches;
      if (sync_debug()) check_launch("jacobi round");
    }
    CK(cudaEventRecord(s.evj1, st));
    check_launch("jacobi sweep");
    ++s.sweeps;
    CK(cudaMemcpyAsync(h_rot, s.d_rot.p, sizeof(int) * ng, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_maxoff, s.d_maxoff.p, sizeof(double) * ng, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_offsum, s.d_offsum.p, sizeof(double) * ng, cudaMemcpyDeviceToHost, st));
    s.d2h_bytes += (long long)(sizeof(int) + 2 * sizeof(double)) * ng;
    CK(cudaStreamSynchronize(st));
    {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, s.evj0, s.evj1));
      s.jacobi_ms += ms;
    }
    // A gate is done when no pair rotated, or (DMMA kernel, which reports the
    // largest relative off-diagonal it saw) when every pair entered this sweep
    // with off <= kQuadFinish (1e-12, within ~50x of the test's tolerance):
    // the rotations of this sweep then leave the pairs at the rounding level
    // and the otherwise Gram-only confirmation sweep is skipped.
#ifdef MPSIM_AB_KNOBS
    if (sweep_debug()) {
      unsigned long long c[8], c2[8];
      jacobi_phase_clocks(c, true);
      jacobi_w32_phase_clocks(c2, true);
      if (c2[6] > 0) std::memcpy(c, c2, sizeof(c));
      if (c[6] > 0)
        std::fprintf(stderr,
                     "[mpsim]   per visit (SM clocks, thread 0): total %.0f = wait %.0f + gram %.0f + test %.0f + "
                     "evd %.0f (%.0f per EVD, %llu EVDs) + rotation %.0f\n",
                     (double)c[0] / c[6], (double)c[1] / c[6], (double)c[2] / c[6], (double)c[3] / c[6],
                     (double)c[4] / c[6], c[7] ? (double)c[4] / c[7] : 0.0, c[7], (double)c[5] / c[6]);
    }
#endif
    if (sweep_debug()) {
      double mx = 0.0, mn = 1e300;
      long long act = 0, pairs = 0;
      for (int i = 0; i < ng; ++i) {
        mx = std::max(mx, h_maxoff[i]);
        mn = std::min(mn, h_maxoff[i]);
        act += h_rot[i] > 0;
        pairs += h_rot[i];
      }
      long long total = 0;
      for (const GateDesc& d : descs) total += (long long)d.nb * (d.nb - 1) / 2;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, s.evj0, s.evj1);
      std::fprintf(stderr,
                   "[mpsim] sweep %d: %lld/%d gates rotated, %lld/%lld pairs rotated, max rel off in [%.3e, %.3e], "
                   "rms off[0] %.3f, %.3f ms\n",
                   sweep, act, ng, pairs, total, mn, mx, std::sqrt(2.0 * h_offsum[0] / std::max(1, descs[0].n)), ms);
    }
    bool any = false;
    for (int i = 0; i < ng; ++i) {
      const bool quad_done = h_maxoff[i] <= quad_finish() && !(sweep == 0 && (first & 4));
      h_rot[i] = h_rot[i] && !quad_done;
      still[i] = h_rot[i];
      any = any || h_rot[i];
      // pre-asymptotic (rms relative off-norm of the sweep above kCrossRms):
      // the next sweep's pair EVDs rotate the cross-block pairs only
      const double rms = std::sqrt(2.0 * h_offsum[i] / std::max(1, descs[i].n));
      // (bounded: at most kCrossSweeps sweeps and only with >= 8 blocks, where the
      // de Rijk reordering keeps reshuffling the blocks; with few blocks two
      // nearly parallel vectors could share a block for good and a cross-only
      // EVD would never rotate them — measured on a SWAP-routed 32 x 32 theta)
      if (h_rot[i] && cross_policy() && rms > cross_rms() && h_maxoff[i] > 1e-3 && sweep < cross_sweeps() &&
          descs[i].nb >= 8)
        h_rot[i] |= 2;
      if (h_rot[i]) h_rot[i] |= alt_cross_bits(w32_sweeps);
      // pre-asymptotic and early asymptotic sweeps reuse the in-block Grams the
      // pair EVDs leave behind (jacobi_split.cu); the closing sweeps recompute all
      if (h_rot[i] && jacobi_mode() >= 3 && inblock_policy() && h_maxoff[i] > kInblockMaxoff) h_rot[i] |= 4;
      // closing sweeps: reuse in-block Grams only while they are exact (flags
      // kept by the persistent sweep kernel; bit-for-bit the recomputed values)
      else if (h_rot[i] && exact_cache_policy()) h_rot[i] |= 8;
      // pre-asymptotic sweeps: pair EVDs with FP32 Gram updates (evd.cuh pair_evd_f32)
      if (h_rot[i] && evd32_maxoff() > 0.0 && h_maxoff[i] > evd32_maxoff() && descs[i].n >= kEvd32MinN)
        h_rot[i] |= 64;
    }
    if (!any) {
      converged = true;
      break;
    }
    upload_active();
  }
  launch_norms(dg, ng, max_n, ws, (double*)s.d_sigma.p, sig_stride, st);
  check_launch("norms_kernel");
  launch_truncate(dg, ng, (double*)s.d_sigma.p, (int*)s.d_order.p, sig_stride, (GateOut*)s.d_out.p,
                  (const double*)s.d_frob.p, kFloorRel2, max_n, st);
  check_launch("truncate_kernel");
  if (any_pre4) {  // Q3 X_kept into y3 (phase 3 then maps it by Q1)
    launch_qr_apply(dph + 7 * ng, ng, qr_n_pad, qr_jm_pad, ws, (const cplx*)s.d_qrv3.p, qr_jm_pad,
                    (const cplx*)s.d_qrt3.p, npan, (const int*)s.d_order.p, sig_stride, (const GateOut*)s.d_out.p,
                    st);
    check_launch("qr_apply (Q3)");
    s.launches += 1 + npan;
  }
  if (any_pre2) {
    launch_qr_apply(dph + 3 * ng, ng, qr_n_pad, qr_m_pad, ws, (const cplx*)s.d_qrv.p, qr_m_pad,
                    (const cplx*)s.d_qrt.p, npan, (const int*)s.d_order.p, sig_stride, (const GateOut*)s.d_out.p,
                    st);
    check_launch("qr_apply");
    s.launches += 1 + npan;
  }
  const GateDesc* dout = dph + 4 * ng;
  if (ortho_policy()) {
    // kept vectors orthonormalised to O(E^2) before the split (split.cu)
    long long kcap = 1;
    for (const GateDesc& d : descs) kcap = std::max<long long>(kcap, std::min<long long>(d.n, d.max_bond));
    const long long tstride = (long long)max_out_m_pad * kcap;
    s.d_fcorr.ensure(sizeof(float2) * (size_t)ng * kcap * kcap);
    s.d_tcorr.ensure(sizeof(float2) * (size_t)ng * tstride);
    launch_orthonormalize(dout, ng, max_out_m, (int)kcap, ws, (const double*)s.d_sigma.p, (const int*)s.d_order.p,
                          sig_stride, (const GateOut*)s.d_out.p, (const double*)s.d_frob.p, kFloorRel2,
                          (float2*)s.d_fcorr.p, (float2*)s.d_tcorr.p, tstride, st);
    check_launch("orthonormalize");
    s.launches += 3;
  }
  launch_write_factors(dout, ng, max_out_m, max_n, max_n0, ws, (const double*)s.d_sigma.p, (const int*)s.d_order.p, sig_stride,
                       (const GateOut*)s.d_out.p, (const double*)s.d_frob.p, kFloorRel2, st);
  check_launch("write_factors");
  s.launches += 4;
  CK(cudaMemcpyAsync(s.h_out.p, s.d_out.p, sizeof(GateOut) * ng, cudaMemcpyDeviceToHost, st));
  s.d2h_bytes += (long long)sizeof(GateOut) * ng;
  CK(cudaStreamSynchronize(st));
  outs.assign((GateOut*)s.h_out.p, (GateOut*)s.h_out.p + ng);
  for (const GateDesc& d : descs) {
    // F_2q = 32 Dl Dm Dr + 128 Dl Dr + 32 M N^2 (M = max, N = min of 2Dl, 2Dr)
    const double M = d.pre ? d.qr_m : d.m, N = d.n;
    s.svd_flops += 32.0 * M * N * N;
    if (src == nullptr) s.gate_flops +=32.0 * d.dl * (double)d.dm * d.dr + 128.0 * d.dl * (double)d.dr + 32.0 * M * N * N;
  }
  if (!converged)
    for (int i = 0; i < ng; ++i)
      if (still[i]) outs[i].status = 3;
}

namespace {

// Applies disjoint local gates. reports[idx] is filled for every gate.
void run_layer(State& s, const std::vector<G2>& two, const std::vector<G1>& one, const mpsim_policy& pol,
               std::vector<Rep>& reports) {
  NvtxRange nv("mpsim: layer (execute_parallel barrier interval)");
  cudaStream_t st = s.st;
  if (!one.empty()) {
    const int ng = (int)one.size();
    s.h_g1.ensure(sizeof(Gate1Desc) * ng);
    s.d_g1.ensure(sizeof(Gate1Desc) * ng);
    Gate1Desc* h = (Gate1Desc*)s.h_g1.p;
    long long max_elems = 1;
    for (int i = 0; i < ng; ++i) {
      const G1& g = one[i];
      h[i].q = g.q;
      h[i].dl = (int)s.sdl[g.q];
      h[i].dr = (int)s.sdr[g.q];
      std::memcpy(h[i].u, g.u, sizeof(g.u));
      max_elems = std::max(max_elems, (long long)h[i].dl * h[i].dr);
      Rep r;
      r.k = std::max(s.bonds[g.q], s.bonds[g.q + 1]);  // gate_apply.cpp:107
      reports[g.idx] = r;
    }
    CK(cudaMemcpyAsync(s.d_g1.p, h, sizeof(Gate1Desc) * ng, cudaMemcpyHostToDevice, st));
    s.h2d_bytes += (long long)sizeof(Gate1Desc) * ng;
    launch_apply1q((const Gate1Desc*)s.d_g1.p, ng, max_elems, s.sites, s.stride, s.chi, st);
    check_launch();
    ++s.launches;
    // The pinned descriptor buffer is reused by the next call: fence here.
    CK(cudaStreamSynchronize(st));
  }
  if (two.empty()) return;
  check_policy(pol);
  // Capacity: the kept rank is at most min(2Dl, 2Dr, max_bond).
  long long need = 1;
  for (const G2& g : two) {
    if (s.sdr[g.q] != s.sdl[g.q + 1])
      fail(MPSIM_EINVAL, "contract: extent mismatch between sites " + std::to_string(g.q) + " and " +
                             std::to_string(g.q + 1));
    long long k = std::min(2 * s.sdl[g.q], 2 * s.sdr[g.q + 1]);
    k = std::min<long long>(k, pol.max_bond);
    need = std::max(need, k);
  }
  if (need > s.chi) s.grow(next_pow2(need));

  // Build descriptors, chunked so the Jacobi workspace fits the budget.
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const long long budget_elems =
      (long long)(std::min<double>((double)free_b * 0.6 + (double)s.ws.bytes, 64e9) / sizeof(cplx));
  std::vector<GateDesc> chunk;
  std::vector<const G2*> chunk_src;
  long long off = 0, extra_used = 0;
  auto flush = [&]() {
    if (chunk.empty()) return;
    std::vector<GateOut> outs;
    run_two_chunk(s, chunk, outs);
    for (size_t i = 0; i < chunk.size(); ++i) {
      const GateDesc& d = chunk[i];
      const GateOut& o = outs[i];
      if (o.status != 0)
        fail(MPSIM_ENUMERIC, "singular value decomposition did not converge for (" + std::to_string(2 * d.dl) + "," +
                                 std::to_string(2 * d.dr) + ") matrix");
      s.sdr[d.q] = o.k;
      s.sdl[d.q + 1] = o.k;
      s.bonds[d.q + 1] = o.k;
      update_center(s, d.q, d.q + 1);
      Rep r;
      r.w = o.w;
      r.k = o.k;
      r.svd = 1;
      reports[chunk_src[i]->idx] = r;
    }
    chunk.clear();
    chunk_src.clear();
    off = 0;
    extra_used = 0;
  };
  for (const G2& g : two) {
    GateDesc d{};
    d.q = g.q;
    d.dl = (int)s.sdl[g.q];
    d.dm = (int)s.sdr[g.q];
    d.dr = (int)s.sdr[g.q + 1];
    const int M = 2 * d.dl, N = 2 * d.dr;
    d.trans = M >= N ? 0 : 1;
    d.m = std::max(M, N);
    d.n = std::min(M, N);
    d.n_pad = ((d.n + kNAlign - 1) / kNAlign) * kNAlign;
    d.m_pad = ((d.m + kE - 1) / kE) * kE;
    d.nb = d.n_pad / kW;
    d.max_bond = pol.max_bond;
    d.cutoff = pol.cutoff;
    std::memcpy(d.u, g.u, sizeof(d.u));
    d.u_out = s.sites + (long long)g.q * s.stride;        // U -> site q (2Dl x k), ld chi
    d.ldu = s.chi;
    d.v_out = s.sites + (long long)(g.q + 1) * s.stride;  // S V^dag -> site q+1 (k, 2, Dr)
    d.ldv = 2LL * s.chi;
    d.vsplit = d.dr;
    d.vsplit_ld = s.chi;
    const int pre = use_qr_precondition(d.n);
    GateDesc probe = d;
    const long long sz = desc_layout(probe, 0, pre);
    long long extra = 0;
    if (ortho_policy()) {  // the split's orthonormalisation buffers (FP32 complex: half a cplx each)
      const long long kc = std::min<long long>(d.n, d.max_bond), mo = phase_desc(probe, 4).m_pad;
      extra = (kc * kc + mo * kc + 1) / 2;
    }
    if (!chunk.empty() && off + extra_used + sz + extra > budget_elems) flush();
    desc_layout(d, off, pre);
    off += sz;
    extra_used += extra;
    chunk.push_back(d);
    chunk_src.push_back(&g);
  }
  flush();
}

void to_cplx(const double* u, int count, cplx* out) {
  for (int i = 0; i < count; ++i) out[i] = make_double2(u[2 * i], u[2 * i + 1]);
}

// SWAP conjugation (gate_apply.cpp:86-95): (high, low) -> (low, high) basis.
void swap_conjugate4(cplx* m) {
  cplx o[16];
  auto rev = [](int x) { return ((x & 1) << 1) | (x >> 1); };
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) o[r * 4 + c] = m[rev(r) * 4 + rev(c)];
  std::memcpy(m, o, sizeof(o));
}

void swap_matrix(cplx* m) {  // gate_apply.cpp:79-84
  for (int i = 0; i < 16; ++i) m[i] = make_double2(0.0, 0.0);
  m[0] = m[6] = m[9] = m[15] = make_double2(1.0, 0.0);
}

// A lowered, local gate with the index of the input gate it belongs to.
struct Lowered {
  int q0, q1;  // q1 = -1 or q0+1
  cplx u[16];
  int src;
};

void lower(const mpsim_gate* gates, int count, int n, std::vector<Lowered>& out) {
  for (int i = 0; i < count; ++i) {
    const mpsim_gate& g = gates[i];
    Lowered L{};
    L.src = i;
    if (g.q1 < 0) {
      if (g.q0 < 0 || g.q0 >= n) fail(MPSIM_EINVAL, "qubit " + std::to_string(g.q0) + " out of range");
      L.q0 = g.q0;
      L.q1 = -1;
      to_cplx(g.u, 4, L.u);
      out.push_back(L);
      continue;
    }
    int a = g.q0, b = g.q1;
    cplx m[16];
    to_cplx(g.u, 16, m);
    if (a == b) fail(MPSIM_EINVAL, "two-qubit gate needs two distinct qubits");
    if (a > b) {
      std::swap(a, b);
      swap_conjugate4(m);
    }
    if (a < 0 || b >= n) fail(MPSIM_EINVAL, "gate qubits out of range");
    // fusion.cpp:137-161: SWAPs i = a..b-2, the gate on (b-1, b), SWAPs back.
    cplx sw[16];
    swap_matrix(sw);
    for (int q = a; q < b - 1; ++q) {
      Lowered s{};
      s.q0 = q;
      s.q1 = q + 1;
      std::memcpy(s.u, sw, sizeof(sw));
      s.src = i;
      out.push_back(s);
    }
    L.q0 = b - 1;
    L.q1 = b;
    std::memcpy(L.u, m, sizeof(m));
    out.push_back(L);
    for (int q = b - 2; q >= a; --q) {
      Lowered s{};
      s.q0 = q;
      s.q1 = q + 1;
      std::memcpy(s.u, sw, sizeof(sw));
      s.src = i;
      out.push_back(s);
    }
  }
}

// fusion.cpp:163-190 — greedy ASAP layering; in-layer order = input order.
std::vector<std::vector<int>> layerize(const std::vector<Lowered>& g, int n) {
  std::vector<int> last((size_t)n, -1);
  std::vector<std::vector<int>> plan;
  for (int i = 0; i < (int)g.size(); ++i) {
    const int lo = g[i].q0, hi = g[i].q1 < 0 ? g[i].q0 : g[i].q1;
    int layer = 0;
    for (int q = lo; q <= hi; ++q) layer = std::max(layer, last[q] + 1);
    if ((size_t)layer >= plan.size()) plan.resize((size_t)layer + 1);
    plan[(size_t)layer].push_back(i);
    for (int q = lo; q <= hi; ++q) last[q] = layer;
  }
  return plan;
}

// Runs a list of local lowered gates layer by layer; returns per-lowered reports.
void run_plan(State& s, const std::vector<Lowered>& low, const mpsim_policy& pol, std::vector<Rep>& rep,
              int* n_layers, long long* peak) {
  const auto plan = layerize(low, s.n);
  rep.assign(low.size(), Rep{});
  long long pk = *std::max_element(s.bonds.begin(), s.bonds.end());
  for (const auto& layer : plan) {
    std::vector<G2> two;
    std::vector<G1> one;
    for (int i : layer) {
      const Lowered& L = low[(size_t)i];
      if (L.q1 < 0) {
        G1 g;
        g.q = L.q0;
        std::memcpy(g.u, L.u, sizeof(g.u));
        g.idx = i;
        one.push_back(g);
      } else {
        G2 g;
        g.q = L.q0;
        std::memcpy(g.u, L.u, sizeof(g.u));
        g.idx = i;
        two.push_back(g);
      }
    }
    run_layer(s, two, one, pol, rep);
    pk = std::max(pk, *std::max_element(s.bonds.begin(), s.bonds.end()));
  }
  if (n_layers) *n_layers = (int)plan.size();
  if (peak) *peak = pk;
}

}  // namespace

// ============================================================== bond propagation
// (apply_2q_bondprop, gate_apply.cpp:181-255) lives in bondprop.cu.
namespace mpsim_gpu {
void apply_bondprop(State& s, const cplx* u_lowhigh, int q0, int q1, const mpsim_policy& pol, double* w,
                    long long* k, int* svd);
}

// ============================================================== queries

namespace {

// E' = sum_p A_p^H op_p(E B_p) over one site; op = optional 2x2 operator on the
// ket side (B'_p = sum_p' O[p][p'] B_p').
void transfer_step(State& a, int i, const State& b, const cplx* E, long long ldE, cplx* E2, long long ldE2, cplx* T0,
                   cplx* T1, long long ldT, const cd* op, cudaStream_t st) {
  const int dla = (int)a.sdl[i], dra = (int)a.sdr[i];
  const int dlb = (int)b.sdl[i], drb = (int)b.sdr[i];
  const cplx* As = a.sites + (long long)i * a.stride;
  const cplx* Bs = b.sites + (long long)i * b.stride;
  auto gemm = [&](int M, int N, int K, const cplx* A, long long lda, int opA, const cplx* B, long long ldb,
                  int opB, cplx* C, long long ldc, cplx alpha, int acc) {
    GemmArgs g{M, N, K, A, lda, opA, B, ldb, opB, C, ldc, alpha, acc};
    launch_cgemm(g, st);
    ++a.launches;
  };
  const cplx one = make_double2(1.0, 0.0);
  // T_p' = E (dla x dlb) * B_p' (dlb x drb)
  gemm(dla, drb, dlb, E, ldE, 0, Bs, 2LL * b.chi, 0, T0, ldT, one, 0);
  gemm(dla, drb, dlb, E, ldE, 0, Bs + b.chi, 2LL * b.chi, 0, T1, ldT, one, 0);
  bool first = true;
  for (int p = 0; p < 2; ++p) {
    const cplx* Ap = As + (long long)p * a.chi;
    if (!op) {
      gemm(dra, drb, dla, Ap, 2LL * a.chi, 1, p == 0 ? T0 : T1, ldT, 0, E2, ldE2, one, first ? 0 : 1);
      first = false;
    } else {
      for (int pp = 0; pp < 2; ++pp) {
        const cd o = op[p * 2 + pp];
        if (o == cd(0.0, 0.0)) continue;
        gemm(dra, drb, dla, Ap, 2LL * a.chi, 1, pp == 0 ? T0 : T1, ldT, 0, E2, ldE2, make_double2(o.real(), o.imag()),
             first ? 0 : 1);
        first = false;
      }
    }
  }
  if (first) launch_fill(E2, (long long)dra * ldE2, make_double2(0.0, 0.0), st);
}

// E' = sum_p A_p^H E B_p over every site (mps.cpp:223-239), optional 2x2
// operators on B's physical index. env_in (host, sdl_a[0] x sdl_b[0],
// row-major; nullptr = [[1]]) / env_out (host, sdr_a[n-1] x sdr_b[n-1]):
// a shard of a longer chain contracts from its left neighbour's environment
// (SURVEY 8(e) queries).
void chain_env(State& a, const State& b, const std::map<int, const cd*>& ops, const cplx* env_in, cplx* env_out,
               int i0 = 0, int i1 = -1) {
  if (a.n != b.n) fail(MPSIM_EINVAL, "overlap requires equal qubit counts");
  if (a.device != b.device) fail(MPSIM_EINVAL, "overlap requires both states on one device");
  if (i1 < 0) i1 = a.n;
  if (i0 < 0 || i1 > a.n || i0 >= i1) fail(MPSIM_EINVAL, "site range out of bounds");
  if (!env_in && (a.sdl[i0] != 1 || b.sdl[i0] != 1)) fail(MPSIM_EINVAL, "open left bond needs an input environment");
  DeviceGuard g(a.device);
  cudaStream_t st = a.st;
  if (&a != &b) CK(cudaStreamSynchronize(b.st));
  const long long c = std::max(a.chi, b.chi);
  a.q1.ensure(sizeof(cplx) * c * c);
  a.q2.ensure(sizeof(cplx) * c * c);
  a.q3.ensure(sizeof(cplx) * c * c);
  a.q4.ensure(sizeof(cplx) * c * c);
  cplx* E = (cplx*)a.q1.p;
  cplx* E2 = (cplx*)a.q2.p;
  const cplx one = make_double2(1.0, 0.0);
  if (env_in)
    CK(cudaMemcpy2DAsync(E, sizeof(cplx) * c, env_in, sizeof(cplx) * b.sdl[i0], sizeof(cplx) * b.sdl[i0], a.sdl[i0],
                         cudaMemcpyDefault, st));  // host or device (UVA): sharded chains pass HBM
  else
    CK(cudaMemcpyAsync(E, &one, sizeof(cplx), cudaMemcpyHostToDevice, st));
  for (int i = i0; i < i1; ++i) {
    auto it = ops.find(i);
    transfer_step(a, i, b, E, c, E2, c, (cplx*)a.q3.p, (cplx*)a.q4.p, c, it == ops.end() ? nullptr : it->second, st);
    std::swap(E, E2);
  }
  check_launch();
  const long long ra = a.sdr[i1 - 1], rb = b.sdr[i1 - 1];
  CK(cudaMemcpy2DAsync(env_out, sizeof(cplx) * rb, E, sizeof(cplx) * c, sizeof(cplx) * rb, ra, cudaMemcpyDefault,
                       st));
  CK(cudaStreamSynchronize(st));
}

cd chain_contract(State& a, const State& b, const std::map<int, const cd*>& ops) {
  if (a.n != b.n) fail(MPSIM_EINVAL, "overlap requires equal qubit counts");
  if (a.sdr[a.n - 1] != 1 || b.sdr[b.n - 1] != 1) fail(MPSIM_EINVAL, "open right bond: use the environment form");
  cplx r;
  chain_env(a, b, ops, nullptr, &r);
  return cd(r.x, r.y);
}

}  // namespace

// ============================================================== C ABI

namespace {
// The calling thread's message slot (shared with the sampler translation unit).
#define g_err (last_error_slot())

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MPSIM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return MPSIM_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MPSIM_ELOGIC;
  }
}

State& S(mpsim_gpu_state* s) {
  if (!s) fail(MPSIM_EINVAL, "null state");
  return *reinterpret_cast<State*>(s);
}
const State& S(const mpsim_gpu_state* s) {
  if (!s) fail(MPSIM_EINVAL, "null state");
  return *reinterpret_cast<const State*>(s);
}

void put_rep(mpsim_report* r, const Rep& x) {
  if (!r) return;
  r->discarded_weight = x.w;
  r->new_bond = x.k;
  r->svd_count = x.svd;
  r->reserved = 0;
}

}  // namespace

extern "C" {

const char* mpsim_gpu_last_error(void) { return g_err.c_str(); }

int mpsim_gpu_state_create(int32_t n, int64_t chi_hint, int32_t device, mpsim_gpu_state** out) {
  return guarded([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    *out = reinterpret_cast<mpsim_gpu_state*>(new State(n, chi_hint, device));
  });
}

int mpsim_gpu_state_destroy(mpsim_gpu_state* s) {
  return guarded([&] { delete reinterpret_cast<State*>(s); });
}

int mpsim_gpu_state_copy(const mpsim_gpu_state* src, mpsim_gpu_state** out) {
  return guarded([&] {
    const State& a = S(src);
    DeviceGuard g(a.device);
    State* b = new State(a.n, a.chi, a.device);
    CK(cudaStreamSynchronize(a.st));
    CK(cudaMemcpyAsync(b->sites, a.sites, (size_t)a.n * a.stride * sizeof(cplx), cudaMemcpyDeviceToDevice, b->st));
    CK(cudaStreamSynchronize(b->st));
    b->bonds = a.bonds;
    b->sdl = a.sdl;
    b->sdr = a.sdr;
    b->center = a.center;
    *out = reinterpret_cast<mpsim_gpu_state*>(b);
  });
}

int mpsim_gpu_num_qubits(const mpsim_gpu_state* s, int32_t* out) {
  return guarded([&] { *out = S(s).n; });
}

int mpsim_gpu_bond_dims(const mpsim_gpu_state* s, int64_t* out) {
  return guarded([&] {
    const State& a = S(s);
    std::memcpy(out, a.bonds.data(), a.bonds.size() * sizeof(int64_t));
  });
}

int mpsim_gpu_chi_capacity(const mpsim_gpu_state* s, int64_t* out) {
  return guarded([&] { *out = S(s).chi; });
}

int mpsim_gpu_ortho_center(const mpsim_gpu_state* s, int32_t* out) {
  return guarded([&] { *out = S(s).center; });
}

int mpsim_gpu_set_ortho_center(mpsim_gpu_state* s, int32_t c) {
  return guarded([&] { S(s).center = c < 0 ? -1 : c; });
}

int mpsim_gpu_set_bond_dim(mpsim_gpu_state* s, int32_t i, int64_t d) {
  return guarded([&] {
    State& a = S(s);
    if (i < 0 || i > a.n) fail(MPSIM_EINVAL, "bond index out of range");
    a.bonds[(size_t)i] = d;
  });
}

int mpsim_gpu_set_open_boundaries(mpsim_gpu_state* s, int32_t open) {
  return guarded([&] { S(s).open_boundaries = open != 0; });
}

int mpsim_gpu_site_slot(const mpsim_gpu_state* s, int32_t i, void** device_ptr, int64_t* chi) {
  return guarded([&] {
    const State& a = S(s);
    if (i < 0 || i >= a.n) fail(MPSIM_EINVAL, "site index out of range");
    *device_ptr = (void*)(a.sites + (long long)i * a.stride);
    *chi = a.chi;
  });
}

int mpsim_gpu_set_site_dims(mpsim_gpu_state* s, int32_t i, int64_t dl, int64_t dr) {
  return guarded([&] {
    State& a = S(s);
    if (i < 0 || i >= a.n) fail(MPSIM_EINVAL, "site index out of range");
    if (dl < 1 || dr < 1 || dl > a.chi || dr > a.chi) fail(MPSIM_EINVAL, "site extents outside the slot");
    a.sdl[i] = dl;
    a.sdr[i] = dr;
    a.bonds[(size_t)i] = dl;
    a.bonds[(size_t)i + 1] = dr;
  });
}

int mpsim_gpu_validate(const mpsim_gpu_state* s) {  // mps.cpp:150-169
  return guarded([&] {
    const State& a = S(s);
    if (a.bonds.size() != (size_t)a.n + 1) fail(MPSIM_ELOGIC, "bond bookkeeping has wrong length");
    if (!a.open_boundaries && (a.bonds.front() != 1 || a.bonds.back() != 1))
      fail(MPSIM_ELOGIC, "boundary bonds must have dimension 1");
    for (int i = 0; i < a.n; ++i)
      if (a.sdl[i] != a.bonds[i] || a.sdr[i] != a.bonds[i + 1])
        fail(MPSIM_ELOGIC, "site " + std::to_string(i) + " disagrees with recorded bond dimensions");
  });
}

int mpsim_gpu_get_site(const mpsim_gpu_state* s, int32_t i, int64_t* dl, int64_t* dr, double* out) {
  return guarded([&] {
    const State& a = S(s);
    if (i < 0 || i >= a.n) fail(MPSIM_EINVAL, "site index out of range");
    *dl = a.sdl[i];
    *dr = a.sdr[i];
    if (!out) return;
    DeviceGuard g(a.device);
    CK(cudaMemcpy2DAsync(out, (size_t)a.sdr[i] * sizeof(cplx), a.sites + (long long)i * a.stride,
                         (size_t)a.chi * sizeof(cplx), (size_t)a.sdr[i] * sizeof(cplx), (size_t)a.sdl[i] * 2,
                         cudaMemcpyDeviceToHost, a.st));
    CK(cudaStreamSynchronize(a.st));
  });
}

int mpsim_gpu_set_site(mpsim_gpu_state* s, int32_t i, int64_t dl, int64_t dr, const double* data) {
  return guarded([&] {
    State& a = S(s);
    if (i < 0 || i >= a.n) fail(MPSIM_EINVAL, "site index out of range");
    if (dl < 1 || dr < 1) fail(MPSIM_EINVAL, "tensor extents must be positive");
    DeviceGuard g(a.device);
    if (std::max(dl, dr) > a.chi) a.grow(next_pow2(std::max(dl, dr)));
    CK(cudaMemcpy2DAsync(a.sites + (long long)i * a.stride, (size_t)a.chi * sizeof(cplx), data,
                         (size_t)dr * sizeof(cplx), (size_t)dr * sizeof(cplx), (size_t)dl * 2,
                         cudaMemcpyHostToDevice, a.st));
    CK(cudaStreamSynchronize(a.st));
    a.sdl[i] = dl;
    a.sdr[i] = dr;
    a.bonds[(size_t)i] = dl;
    a.bonds[(size_t)i + 1] = dr;
  });
}

int mpsim_gpu_apply_1q(mpsim_gpu_state* s, const double* u, int32_t q, mpsim_report* rep) {
  return guarded([&] {
    State& a = S(s);
    if (q < 0 || q >= a.n) fail(MPSIM_EINVAL, "qubit " + std::to_string(q) + " out of range");
    DeviceGuard g(a.device);
    G1 g1;
    g1.q = q;
    g1.idx = 0;
    to_cplx(u, 4, g1.u);
    std::vector<Rep> r(1);
    run_layer(a, {}, {g1}, mpsim_policy{MPSIM_UNBOUNDED, 0.0}, r);
    put_rep(rep, r[0]);
  });
}

int mpsim_gpu_apply_2q(mpsim_gpu_state* s, const double* u, int32_t q0, int32_t q1, int32_t method,
                       const mpsim_policy* policy, mpsim_report* rep) {
  return guarded([&] {
    State& a = S(s);
    if (!policy) fail(MPSIM_EINVAL, "null policy");
    DeviceGuard g(a.device);
    if (q0 == q1) fail(MPSIM_EINVAL, "two-qubit gate needs two distinct qubits");
    if (method == MPSIM_NONLOCAL_BONDPROP) {
      check_policy(*policy);
      cplx m[16];
      to_cplx(u, 16, m);
      int a0 = q0, b0 = q1;
      if (a0 > b0) {
        std::swap(a0, b0);
        swap_conjugate4(m);
      }
      if (a0 < 0 || b0 >= a.n)
        fail(MPSIM_EINVAL, "qubit pair (" + std::to_string(a0) + "," + std::to_string(b0) + ") out of range");
      Rep r;
      apply_bondprop(a, m, a0, b0, *policy, &r.w, &r.k, &r.svd);
      put_rep(rep, r);
      return;
    }
    if (std::min(q0, q1) < 0 || std::max(q0, q1) >= a.n)
      fail(MPSIM_EINVAL, "adjacent pair (" + std::to_string(std::min(q0, q1)) + "," +
                             std::to_string(std::max(q0, q1)) + ") out of range");
    check_policy(*policy);
    mpsim_gate gate;
    gate.q0 = q0;
    gate.q1 = q1;
    std::memcpy(gate.u, u, sizeof(double) * 32);
    std::vector<Lowered> low;
    lower(&gate, 1, a.n, low);
    Rep tot;
    tot.k = 1;
    // Sequential single-gate layers, in SWAP-chain order (gate_apply.cpp:171-177).
    for (size_t i = 0; i < low.size(); ++i) {
      G2 g2;
      g2.q = low[i].q0;
      std::memcpy(g2.u, low[i].u, sizeof(g2.u));
      g2.idx = 0;
      std::vector<Rep> r(1);
      run_layer(a, {g2}, {}, *policy, r);
      tot.w += r[0].w;
      tot.k = std::max(tot.k, r[0].k);
      tot.svd += r[0].svd;
    }
    put_rep(rep, tot);
  });
}

int mpsim_gpu_apply_layer(mpsim_gpu_state* s, const mpsim_gate* gates, int32_t count, const mpsim_policy* policy,
                          mpsim_report* reports) {
  return guarded([&] {
    State& a = S(s);
    DeviceGuard g(a.device);
    std::vector<char> busy((size_t)a.n, 0);
    std::vector<G2> two;
    std::vector<G1> one;
    for (int i = 0; i < count; ++i) {
      const mpsim_gate& gt = gates[i];
      int lo = gt.q0, hi = gt.q1 < 0 ? gt.q0 : gt.q1;
      if (gt.q1 >= 0 && lo > hi) std::swap(lo, hi);
      if (lo < 0 || hi >= a.n) fail(MPSIM_EINVAL, "gate qubits out of range");
      if (gt.q1 >= 0 && hi != lo + 1) fail(MPSIM_EINVAL, "parallel execution requires a local-gate plan");
      // SpanGuard (executor.cpp:41-69): disjoint spans inside one layer.
      for (int q = lo; q <= hi; ++q) {
        if (busy[(size_t)q])
          fail(MPSIM_ELOGIC, "layer contract violated: two in-flight gates touch site " + std::to_string(q));
        busy[(size_t)q] = 1;
      }
      if (gt.q1 < 0) {
        G1 g1;
        g1.q = gt.q0;
        to_cplx(gt.u, 4, g1.u);
        g1.idx = i;
        one.push_back(g1);
      } else {
        G2 g2;
        g2.q = lo;
        to_cplx(gt.u, 16, g2.u);
        if (gt.q0 > gt.q1) swap_conjugate4(g2.u);
        g2.idx = i;
        two.push_back(g2);
      }
    }
    if (!two.empty() && !policy) fail(MPSIM_EINVAL, "null policy");
    std::vector<Rep> r((size_t)count);
    run_layer(a, two, one, policy ? *policy : mpsim_policy{MPSIM_UNBOUNDED, 0.0}, r);
    if (reports)
      for (int i = 0; i < count; ++i) put_rep(&reports[i], r[(size_t)i]);
  });
}

int mpsim_gpu_execute(mpsim_gpu_state* s, const mpsim_gate* gates, int32_t count, const mpsim_policy* policy,
                      int32_t method, mpsim_exec_stats* stats, mpsim_report* reports) {
  return guarded([&] {
    State& a = S(s);
    if (!policy) fail(MPSIM_EINVAL, "null policy");
    DeviceGuard g(a.device);
    const long long l0 = a.launches;
    CK(cudaEventRecord(a.ev0, a.st));
    std::vector<Rep> per_input((size_t)count);
    long long peak = *std::max_element(a.bonds.begin(), a.bonds.end());
    int n_layers = 0, n_local = 0;
    if (method == MPSIM_NONLOCAL_BONDPROP) {
      // execute_serial with BondProp: gate by gate (executor.cpp:84-92).
      for (int i = 0; i < count; ++i) {
        const mpsim_gate& gt = gates[i];
        const bool nonlocal = gt.q1 >= 0 && std::abs(gt.q1 - gt.q0) != 1;
        if (nonlocal) {
          mpsim_report r;
          const int rc = mpsim_gpu_apply_2q(s, gt.u, gt.q0, gt.q1, MPSIM_NONLOCAL_BONDPROP, policy, &r);
          if (rc != MPSIM_OK) fail(rc, g_err);
          per_input[(size_t)i] = Rep{r.discarded_weight, r.new_bond, r.svd_count};
          ++n_layers;
          ++n_local;
        } else {
          std::vector<Lowered> low;
          lower(&gt, 1, a.n, low);
          std::vector<Rep> rep;
          int nl = 0;
          run_plan(a, low, *policy, rep, &nl, nullptr);
          per_input[(size_t)i] = rep[0];
          n_layers += nl;
          n_local += (int)low.size();
        }
        peak = std::max(peak, *std::max_element(a.bonds.begin(), a.bonds.end()));
      }
    } else {
      std::vector<Lowered> low;
      lower(gates, count, a.n, low);
      bool any2 = false;
      for (const Lowered& L : low) any2 = any2 || L.q1 >= 0;
      if (any2) check_policy(*policy);
      std::vector<Rep> rep;
      long long pk = 0;
      run_plan(a, low, *policy, rep, &n_layers, &pk);
      peak = std::max(peak, pk);
      n_local = (int)low.size();
      // Aggregate SWAP chains per input gate (gate_apply.cpp:163-167).
      std::vector<char> seen((size_t)count, 0);
      for (size_t i = 0; i < low.size(); ++i) {
        Rep& t = per_input[(size_t)low[i].src];
        const Rep& x = rep[i];
        if (!seen[(size_t)low[i].src]) {
          t = x;
          seen[(size_t)low[i].src] = 1;
        } else {
          t.w += x.w;
          t.k = std::max(t.k, x.k);
          t.svd += x.svd;
        }
      }
    }
    CK(cudaEventRecord(a.ev1, a.st));
    CK(cudaEventSynchronize(a.ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a.ev0, a.ev1));
    a.device_ms += ms;
    double total_w = 0.0;
    for (const Rep& r : per_input) total_w += r.w;  // executor.cpp:90, input order
    if (stats) {
      stats->peak_bond = peak;
      stats->total_discarded_weight = total_w;
      stats->layers = n_layers;
      stats->gates = n_local;
      stats->kernel_launches = a.launches - l0;
      stats->device_ms = ms;
    }
    if (reports)
      for (int i = 0; i < count; ++i) put_rep(&reports[i], per_input[(size_t)i]);
    // executor.cpp:93 validates the final state.
    if (mpsim_gpu_validate(s) != MPSIM_OK) fail(MPSIM_ELOGIC, g_err);
  });
}

int mpsim_gpu_move_center(mpsim_gpu_state* s, int32_t center) {  // mps.cpp:177-187
  return guarded([&] { move_center_impl(S(s), center); });
}

int mpsim_gpu_sweep_left(mpsim_gpu_state* s, int32_t i0, int32_t i1) {  // mps.cpp:69-80, sites [i0, i1)
  return guarded([&] { sweep_left_impl(S(s), i0, i1); });
}

int mpsim_gpu_sweep_right(mpsim_gpu_state* s, int32_t i0, int32_t i1) {  // mps.cpp:84-95, sites i1 .. i0
  return guarded([&] { sweep_right_impl(S(s), i0, i1); });
}

int mpsim_gpu_site_norm2(const mpsim_gpu_state* s, int32_t i, double* out) {
  return guarded([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    *out = site_norm2_impl(const_cast<State&>(S(s)), i);
  });
}

int mpsim_gpu_norm(const mpsim_gpu_state* s, double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    const cd v = chain_contract(a, a, {});
    *out = std::sqrt(std::max(0.0, v.real()));
  });
}

int mpsim_gpu_overlap(const mpsim_gpu_state* x, const mpsim_gpu_state* y, double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(x));
    const cd v = chain_contract(a, S(y), {});
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int mpsim_gpu_expect_1q(const mpsim_gpu_state* s, const double* op, int32_t q, double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    if (q < 0 || q >= a.n) fail(MPSIM_EINVAL, "qubit out of range");
    cd o[4];
    for (int i = 0; i < 4; ++i) o[i] = cd(op[2 * i], op[2 * i + 1]);
    const cd v = chain_contract(a, a, {{q, o}});
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int mpsim_gpu_expect_2q(const mpsim_gpu_state* s, const double* op_a, int32_t qa, const double* op_b, int32_t qb,
                        double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    if (qa < 0 || qa >= a.n || qb < 0 || qb >= a.n || qa == qb) fail(MPSIM_EINVAL, "invalid qubit pair");
    cd oa[4], ob[4];
    for (int i = 0; i < 4; ++i) {
      oa[i] = cd(op_a[2 * i], op_a[2 * i + 1]);
      ob[i] = cd(op_b[2 * i], op_b[2 * i + 1]);
    }
    const cd v = chain_contract(a, a, {{qa, oa}, {qb, ob}});
    out[0] = v.real();
    out[1] = v.imag();
  });
}

// Row environments of `count` bit strings through every site (mps.cpp:204-221):
// env_in (host, count x sdl[0]; nullptr = ones at a chain start), env_out
// (host, count x sdr[n-1]); amplitudes are the 1 x 1 case.
static void amplitude_env(State& a, const char* bits, int32_t count, const cplx* env_in, cplx* env_out, int i0 = 0,
                          int i1 = -1) {
  if (count < 0) fail(MPSIM_EINVAL, "negative count");
  if (i1 < 0) i1 = a.n;
  if (i0 < 0 || i1 > a.n || i0 >= i1) fail(MPSIM_EINVAL, "site range out of bounds");
  for (long long i = 0; i < (long long)count * a.n; ++i)
    if (bits[i] != '0' && bits[i] != '1') fail(MPSIM_EINVAL, "bit string must contain only 0 and 1");
  if (!env_in && a.sdl[i0] != 1) fail(MPSIM_EINVAL, "open left bond needs an input environment");
  if (count == 0) return;
  DeviceGuard g(a.device);
  cudaStream_t st = a.st;
  const int chunk = 4096;
  const long long l0 = a.sdl[i0], rn = a.sdr[i1 - 1];
  a.qbits.ensure((size_t)std::min(count, chunk) * a.n);
  a.q1.ensure(sizeof(cplx) * (size_t)std::min(count, chunk) * a.chi);
  a.q2.ensure(sizeof(cplx) * (size_t)std::min(count, chunk) * a.chi);
  for (int c0 = 0; c0 < count; c0 += chunk) {
    const int c = std::min(chunk, count - c0);
    CK(cudaMemcpyAsync(a.qbits.p, bits + (long long)c0 * a.n, (size_t)c * a.n, cudaMemcpyHostToDevice, st));
    cplx* E = (cplx*)a.q1.p;
    cplx* E2 = (cplx*)a.q2.p;
    long long ld = l0;
    if (env_in)
      CK(cudaMemcpyAsync(E, env_in + (long long)c0 * l0, sizeof(cplx) * c * l0, cudaMemcpyDefault, st));
    else
      launch_fill(E, c, make_double2(1.0, 0.0), st);  // env = ones(1) per string, ld = 1 at site 0
    for (int i = i0; i < i1; ++i) {
      launch_amp_step(E, ld, E2, a.sdr[i], (const char*)a.qbits.p, a.n, i, c, a.sites + (long long)i * a.stride,
                      a.chi, (int)a.sdl[i], (int)a.sdr[i], st);
      ++a.launches;
      ld = a.sdr[i];
      std::swap(E, E2);
    }
    check_launch();
    CK(cudaMemcpyAsync(env_out + (long long)c0 * rn, E, sizeof(cplx) * c * rn, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  }
}

int mpsim_gpu_amplitudes_env(const mpsim_gpu_state* s, int32_t i0, int32_t i1, const char* bits, int32_t count,
                             const double* env_in, double* env_out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    if (!env_out) fail(MPSIM_EINVAL, "null output");
    amplitude_env(a, bits, count, reinterpret_cast<const cplx*>(env_in), reinterpret_cast<cplx*>(env_out), i0, i1);
  });
}

int mpsim_gpu_transfer_env(const mpsim_gpu_state* x, const mpsim_gpu_state* y, int32_t i0, int32_t i1,
                           const double* op2x2, int32_t q, const double* env_in, double* env_out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(x));
    if (!env_out) fail(MPSIM_EINVAL, "null output");
    cd o[4];
    std::map<int, const cd*> ops;
    if (op2x2) {
      if (q < 0 || q >= a.n) fail(MPSIM_EINVAL, "qubit out of range");
      for (int i = 0; i < 4; ++i) o[i] = cd(op2x2[2 * i], op2x2[2 * i + 1]);
      ops[q] = o;
    }
    chain_env(a, S(y), ops, reinterpret_cast<const cplx*>(env_in), reinterpret_cast<cplx*>(env_out), i0, i1);
  });
}

int mpsim_gpu_amplitudes(const mpsim_gpu_state* s, const char* bits, int32_t count, double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    if (a.sdr[a.n - 1] != 1) fail(MPSIM_EINVAL, "open right bond: use mpsim_gpu_amplitudes_env");
    amplitude_env(a, bits, count, nullptr, reinterpret_cast<cplx*>(out));
  });
}

int mpsim_gpu_to_statevector(const mpsim_gpu_state* s, int32_t max_qubits, double* out) {
  return guarded([&] {
    State& a = const_cast<State&>(S(s));
    if (a.n > max_qubits)
      fail(MPSIM_EINVAL, "statevector export capped at " + std::to_string(max_qubits) + " qubits, got " +
                             std::to_string(a.n));
    DeviceGuard g(a.device);
    cudaStream_t st = a.st;
    const size_t cap = (size_t)1 << a.n;
    size_t need = cap;
    // acc is (rows x dl); grown is (rows x 2dr) = (2 rows x dr).
    long long rows = 1;
    for (int i = 0; i < a.n; ++i) {
      need = std::max(need, (size_t)(rows * 2 * a.sdr[i]));
      rows *= 2;
    }
    a.q1.ensure(sizeof(cplx) * need);
    a.q2.ensure(sizeof(cplx) * need);
    cplx* acc = (cplx*)a.q1.p;
    cplx* nx = (cplx*)a.q2.p;
    const cplx one = make_double2(1.0, 0.0);
    CK(cudaMemcpyAsync(acc, &one, sizeof(cplx), cudaMemcpyHostToDevice, st));
    rows = 1;
    for (int i = 0; i < a.n; ++i) {
      const int dl = (int)a.sdl[i], dr = (int)a.sdr[i];
      const cplx* site = a.sites + (long long)i * a.stride;
      for (int p = 0; p < 2; ++p) {
        GemmArgs ga{(int)rows, dr, dl, acc, dl, 0, site + (long long)p * a.chi, 2LL * a.chi, 0, nx + (long long)p * dr,
                    2LL * dr, one, 0};
        launch_cgemm(ga, st);
        ++a.launches;
      }
      rows *= 2;
      std::swap(acc, nx);
    }
    check_launch();
    CK(cudaMemcpyAsync(out, acc, sizeof(cplx) * cap, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int mpsim_gpu_svd(int32_t rows, int32_t cols, const double* a, int64_t max_rank, double cutoff, int32_t device,
                  int64_t* k, double* s_out, double* u_out, double* vdag_out, double* w) {
  return guarded([&] {
    // svd.hpp:79-110 argument contract
    if (rows < 1 || cols < 1) fail(MPSIM_EINVAL, "svd requires a rank-2 tensor with positive extents");
    if (max_rank < 1) fail(MPSIM_EINVAL, "svd max_rank must be >= 1");
    if (!(cutoff >= 0.0 && cutoff < 1.0)) fail(MPSIM_EINVAL, "svd cutoff must lie in [0, 1)");
    static std::map<int, State*> scratch;  // per-device buffers for plain SVDs
    State*& sc = scratch[device];
    if (!sc) sc = new State(1, 2, device);
    DeviceGuard g(device);
    GateDesc d{};
    d.dl = 1;
    d.dm = 1;
    d.dr = 1;
    d.trans = rows >= cols ? 0 : 1;
    d.m = std::max(rows, cols);
    d.n = std::min(rows, cols);
    d.n_pad = ((d.n + kNAlign - 1) / kNAlign) * kNAlign;
    d.m_pad = ((d.m + kE - 1) / kE) * kE;
    d.nb = d.n_pad / kW;
    d.max_bond = max_rank;
    d.cutoff = cutoff;
    desc_layout(d, 0, use_qr_precondition(d.n));
    DeviceBuf dU, dV, dA;
    dU.ensure(sizeof(cplx) * (size_t)rows * d.n);
    dV.ensure(sizeof(cplx) * (size_t)d.n * cols);
    dA.ensure(sizeof(cplx) * (size_t)rows * cols);
    d.u_out = (cplx*)dU.p;
    d.ldu = d.n;
    d.v_out = (cplx*)dV.p;
    d.ldv = cols;
    d.vsplit = cols;
    d.vsplit_ld = 0;
    CK(cudaMemcpy(dA.p, a, sizeof(cplx) * (size_t)rows * cols, cudaMemcpyHostToDevice));
    std::vector<GateOut> outs;
    run_two_chunk(*sc, {d}, outs, (const cplx*)dA.p, cols);
    dA.release();
    const GateOut& o = outs[0];
    if (o.status != 0)
      fail(MPSIM_ENUMERIC, "singular value decomposition did not converge for (" + std::to_string(rows) + "," +
                               std::to_string(cols) + ") matrix");
    const int kk = o.k;
    *k = kk;
    *w = o.w;
    std::vector<double> sv((size_t)kk);
    std::vector<cplx> hu((size_t)rows * d.n), hv((size_t)d.n * cols);
    CK(cudaMemcpy(sv.data(), sc->d_sigma.p, sizeof(double) * kk, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hu.data(), dU.p, sizeof(cplx) * hu.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv.data(), dV.p, sizeof(cplx) * hv.size(), cudaMemcpyDeviceToHost));
    dU.release();
    dV.release();
    for (int j = 0; j < kk; ++j) s_out[j] = sv[(size_t)j];
    if (u_out)
      for (int r = 0; r < rows; ++r)
        for (int j = 0; j < kk; ++j) {
          u_out[2 * ((size_t)r * kk + j)] = hu[(size_t)r * d.n + j].x;
          u_out[2 * ((size_t)r * kk + j) + 1] = hu[(size_t)r * d.n + j].y;
        }
    if (vdag_out)
      for (int j = 0; j < kk; ++j) {
        // The split epilogue writes scale * S V^dag; svd() returns V^dag alone.
        const double f = sv[(size_t)j] > 0.0 ? 1.0 / (sv[(size_t)j] * o.scale) : 0.0;
        for (int c = 0; c < cols; ++c) {
          cplx v = hv[(size_t)j * cols + c];
          if (f == 0.0) v = make_double2(c == j ? 1.0 : 0.0, 0.0);
          vdag_out[2 * ((size_t)j * cols + c)] = f == 0.0 ? v.x : v.x * f;
          vdag_out[2 * ((size_t)j * cols + c) + 1] = f == 0.0 ? v.y : v.y * f;
        }
      }
  });
}

int mpsim_gpu_counters(const mpsim_gpu_state* s, int64_t* launches, double* device_ms, int64_t* sweeps) {
  return guarded([&] {
    const State& a = S(s);
    if (launches) *launches = a.launches;
    if (device_ms) *device_ms = a.device_ms;
    if (sweeps) *sweeps = a.sweeps;
  });
}

int mpsim_gpu_kernel_counters(const mpsim_gpu_state* s, int64_t* jacobi_launches, double* jacobi_ms,
                              double* svd_flops, double* gate_flops) {
  return guarded([&] {
    const State& a = S(s);
    if (jacobi_launches) *jacobi_launches = a.jacobi_launches;
    if (jacobi_ms) *jacobi_ms = a.jacobi_ms;
    if (svd_flops) *svd_flops = a.svd_flops;
    if (gate_flops) *gate_flops = a.gate_flops;
  });
}

int mpsim_gpu_reset_counters(mpsim_gpu_state* s) {
  return guarded([&] {
    State& a = S(s);
    a.launches = 0;
    a.device_ms = 0.0;
    a.sweeps = 0;
    a.jacobi_launches = 0;
    a.jacobi_ms = 0.0;
    a.svd_flops = 0.0;
    a.gate_flops = 0.0;
    a.h2d_bytes = 0;
    a.d2h_bytes = 0;
  });
}

int mpsim_gpu_transfer_counters(const mpsim_gpu_state* s, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  return guarded([&] {
    const State& a = S(s);
    if (h2d_bytes) *h2d_bytes = a.h2d_bytes;
    if (d2h_bytes) *d2h_bytes = a.d2h_bytes;
  });
}

int mpsim_gpu_synchronize(mpsim_gpu_state* s) {
  return guarded([&] {
    State& a = S(s);
    DeviceGuard g(a.device);
    CK(cudaStreamSynchronize(a.st));
  });
}

}  // extern "C"
