// Host-side engine types shared by the engine translation units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace mpsim_gpu {

struct Error : std::runtime_error {
  int code;
  Error(int c, std::string m);
};
[[noreturn]] void fail(int code, const std::string& msg);
std::string& last_error_slot();  // mpsim_gpu_last_error() of the calling thread

// Owning device / pinned-host buffers: move-only, freed by the destructor, so
// a workspace added later (or a local left on an error path) cannot leak.
// ensure() grows by at least 1.5x so buffers that grow step by step (the
// sampler's prefix environments) reallocate O(log) times.
struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DeviceBuf() = default;
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
  DeviceBuf(DeviceBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DeviceBuf& operator=(DeviceBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DeviceBuf() { release(); }
  void ensure(size_t b);
  void release();
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  PinnedBuf(PinnedBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  PinnedBuf& operator=(PinnedBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~PinnedBuf() { release(); }
  void ensure(size_t b);
  void release();
};

// NVTX range for Nsight timelines (header-only NVTX v3: a no-op unless a
// tool is attached). Named after the reference step each range replaces.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

// The HBM-resident MPS (MpsState, mps.hpp:33-75): n sites of (chi x 2 x chi)
// complex128 slots; real dims per site in sdl/sdr; bonds as the reference
// records them (bond_dims_, mps.hpp:73).
struct State {
  int n = 0;
  int device = 0;
  int chi = 0;          // padded capacity (power of two)
  long long stride = 0; // complex elements per site slot
  cplx* sites = nullptr;
  DeviceBuf sites_buf;
  std::vector<long long> bonds;   // n+1
  std::vector<long long> sdl, sdr;  // site extents
  int center = -1;
  bool open_boundaries = false;  // shard of a longer chain (multi-GPU)
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // workspaces
  DeviceBuf ws, d_gates, d_out, d_sigma, d_order, d_active, d_rot, d_frob, d_perm, d_maxoff, d_g1, q1, q2, q3, q4,
      qbits, d_need, d_gbuf, d_rbuf, d_offsum, d_qrv, d_qrt, d_gblk, d_qrv2, d_qrt2, d_sweepctl, d_fcorr, d_tcorr, d_qrv3, d_qrt3;
  PinnedBuf h_gates, h_out, h_rot, h_g1, h_small, h_maxoff, h_offsum, h_maps;
  DeviceBuf d_maps;  // per-gate TMA tensor maps of the theta kernel
  // instrumentation
  long long launches = 0;
  double device_ms = 0.0;
  long long sweeps = 0;
  long long jacobi_launches = 0;  // Jacobi sweep (or round) launches
  double jacobi_ms = 0.0;         // CUDA-event time of those launches
  double svd_flops = 0.0;         // algorithmic SVD flops of the decomposed matrices (32 M N^2)
  double gate_flops = 0.0;        // algorithmic F_2q of applied gates
  cudaEvent_t evj0 = nullptr, evj1 = nullptr;
  // centre moves (qr_site.cu): a second stream for trailing updates, two join events
  cudaStream_t aux = nullptr;
  cudaEvent_t evq[3] = {nullptr, nullptr, nullptr};
  long long h2d_bytes = 0, d2h_bytes = 0;  // gate-path host<->device traffic

  State(int n, long long chi_hint, int device);
  ~State();
  State(const State&) = delete;
  State& operator=(const State&) = delete;
  void grow(int new_chi);
  void launch_fill_sites_zero_state();
};

// QR sweeps of move_center (canon.cu).
void move_center_impl(State& s, int center);
void sweep_left_impl(State& s, int i0, int i1);
void sweep_right_impl(State& s, int i0, int i1);
double site_norm2_impl(State& s, int i);

// Batched Jacobi SVD + truncation + split of the descriptors (engine.cu). The
// operand comes from the theta kernel (src == nullptr) or, for a single
// descriptor, from a row-major device matrix src (leading dimension src_ld).
void run_two_chunk(State& s, const std::vector<GateDesc>& descs, std::vector<GateOut>& outs,
                   const cplx* src = nullptr, long long src_ld = 0);
// X (orientation xtrans, stride ldx, split planes if xsplit) and X0 (orientation f, stride ldx0) of a
// row-major device matrix A (rows x cols), ||A||_F^2 added to *frob2.
void launch_load_matrix(const cplx* A, long long lda, int rows, int cols, int xtrans, cplx* X, long long ldx,
                        int xsplit, int f, cplx* X0, long long ldx0, double* frob2, cudaStream_t st);
// QR preconditioning steps (0, 1, 2) for a descriptor with n vectors (engine.cu).
int use_qr_precondition(int n);
void launch_cgemm(const GemmArgs&, cudaStream_t);

}  // namespace mpsim_gpu
