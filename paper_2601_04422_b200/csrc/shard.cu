// Site-sharded chains across GPUs, host C++ in the library.
//
// Replaces, in the reference's terms, the execute_parallel worker pool
// (src/executor.cpp:99-232) when a chain spans several GPUs, and the paper's
// TAMM / GlobalArrays layer distribution. One process per
// GPU; NCCL (loaded at run time, libnccl.so.2) over NVLink / NVSwitch moves
// the data; nothing else (no torch) is on the data plane.
//
// Rank r owns global sites [lo, hi) with even boundaries (cost-weighted,
// shard_bounds), so even brick layers never straddle a shard and odd layers
// straddle at exactly world - 1 gates. A shard that is not the last keeps one
// "ghost" slot after its last site. For a layer with a gate on (hi-1, hi):
//   1. rank r+1 sends its first site (the whole padded slot) and its extents
//      to rank r, which records it in the ghost slot;
//   2. every rank applies its own gates (the straddling one included on rank
//      r) as one batched launch sequence (mpsim_gpu_execute);
//   3. rank r sends the updated ghost site (k, 2, Dr) back; rank r+1 stores it
//      as its first site, whose left bond is now k.
// Gates of a layer are disjoint, so the per-gate inputs never change with the
// shard count: N GPUs reproduce the one-GPU result bit for bit. All NCCL
// calls are enqueued on the shard state's stream, so the exchange is ordered
// with the gate kernels without host round trips; the host reads back only
// the 16-byte extents of a received site.
//
// Queries follow the chain: each rank continues its left neighbour's
// environment (row environments for amplitudes, transfer environments for
// norm / overlap / <O_q>) over its sites and sends it right, device to device;
// the last rank broadcasts the result. Centre moves run the same QR steps in
// the same order as move_center (mps.cpp:171-187), handing boundary sites back
// and forth. Perfect sampling canonicalises a copy that way and walks shot
// chunks rank by rank, handing over the distinct-prefix environments.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {
namespace {

// ---- NCCL, resolved at run time (the process may already hold torch's copy;
// the loader then hands back that one: same soname, same API)
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.error = e ? e : "dlopen failed";
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f && api.error.empty()) api.error = std::string("missing symbol ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Broadcast, "ncclBroadcast");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GetErrorString, "ncclGetErrorString");
  });
  if (!api.error.empty()) fail(MPSIM_ECUDA, "NCCL unavailable: " + api.error);
  return api;
}

#define NC(x)                                                                                        \
  do {                                                                                               \
    ncclResult_t r_ = (x);                                                                           \
    if (r_ != ncclSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + nccl().GetErrorString(r_));    \
  } while (0)
#define CKH(x)                                                                             \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
// a C-ABI call on the local state from inside a guarded function
#define ABI(x)                                    \
  do {                                            \
    const int rc_ = (x);                          \
    if (rc_ != MPSIM_OK) fail(rc_, last_error_slot()); \
  } while (0)

template <class F>
int sguard(F&& f) {
  try {
    f();
    return MPSIM_OK;
  } catch (const Error& e) {
    last_error_slot() = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    last_error_slot() = "host allocation failed";
    return MPSIM_ECUDA;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return MPSIM_ELOGIC;
  }
}

// ---- host planning (no device): the pieces tests/test_sharding.py drives on CPU

// Even-aligned contiguous ranges [b_r, b_{r+1}). With a bond cap chi > 0 the
// cut points split the steady-state gate cost (theta merge and SVD of the gate
// on (q, q+1) scale as D_q D_{q+1} D_{q+2}, bonds min(chi, 2^q, 2^(n-q))) into
// equal parts, so the cheap edge gates do not leave the edge shards idle;
// without it the sites are split evenly.
std::vector<int> shard_bounds(int n, int world, long long chi) {
  if (world < 1 || n < 2 * world) fail(MPSIM_EINVAL, "need at least two sites per shard");
  std::vector<double> cum((size_t)n + 1, 0.0);
  if (chi <= 0 || world == 1) {
    for (int q = 0; q <= n; ++q) cum[(size_t)q] = q;
  } else {
    std::vector<double> bond((size_t)n + 1);
    for (int q = 0; q <= n; ++q) bond[(size_t)q] = (double)std::min<long long>(chi, 1LL << std::min({q, n - q, 60}));
    for (int q = 0; q < n; ++q)
      cum[(size_t)q + 1] = cum[(size_t)q] + bond[(size_t)q] * bond[(size_t)q + 1] * bond[(size_t)std::min(q + 2, n)];
  }
  std::vector<int> b{0};
  for (int r = 1; r < world; ++r) {
    const double target = r * cum[(size_t)n] / world;
    int x = 0;
    double best = std::abs(cum[0] - target);
    for (int q = 1; q <= n; ++q)
      if (std::abs(cum[(size_t)q] - target) < best) {
        best = std::abs(cum[(size_t)q] - target);
        x = q;
      }
    x -= x % 2;
    x = std::max(b.back() + 2, x);
    x = std::min(x, n - 2 * (world - r));  // leave room for the remaining shards
    b.push_back(x);
  }
  b.push_back(n);
  return b;
}

// One layer (global indices) for the shard [lo, hi): the gates this rank
// applies (local indices; a gate on (hi-1, hi) uses the ghost slot) and
// whether it lends its first site left / borrows the right neighbour's.
void partition_layer(const mpsim_gate* gates, int count, int lo, int hi, int rank, int world,
                     std::vector<mpsim_gate>& local, bool& straddle_left, bool& straddle_right) {
  local.clear();
  straddle_left = straddle_right = false;
  for (int i = 0; i < count; ++i) {
    mpsim_gate g = gates[i];
    if (g.q1 < 0) {
      if (lo <= g.q0 && g.q0 < hi) {
        g.q0 -= lo;
        local.push_back(g);
      }
      continue;
    }
    const int a = std::min(g.q0, g.q1), b = std::max(g.q0, g.q1);
    if (b != a + 1) fail(MPSIM_EINVAL, "sharded layers take local gates (lower non-local gates to SWAP chains first)");
    if (lo <= a && b < hi) {
      g.q0 -= lo;
      g.q1 -= lo;
      local.push_back(g);
    } else if (rank < world - 1 && a == hi - 1) {
      g.q0 -= lo;
      g.q1 -= lo;
      local.push_back(g);
      straddle_right = true;
    } else if (rank > 0 && b == lo) {
      straddle_left = true;
    }
  }
}

}  // namespace
}  // namespace mpsim_gpu

using namespace mpsim_gpu;

struct mpsim_gpu_shard {
  int n = 0, rank = 0, world = 1, device = 0;
  long long chi = 0;
  int lo = 0, hi = 0, n_local = 0;
  bool has_right = false;
  mpsim_gpu_state* state = nullptr;  // owned sites [lo, hi) + ghost
  ncclComm_t comm = nullptr;
  bool owns_comm = false;
  DeviceBuf dims_send, dims_recv, scratch, scratch2, red;
  PinnedBuf dims_host, red_host;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int center = -1;
  bool capacity_agreed = false;  // slot capacities equal on every rank (reset by set_site)
  std::vector<std::pair<std::string, uint64_t>> result;  // last sample()
  State& st() { return *reinterpret_cast<State*>(state); }
  cudaStream_t stream() { return st().st; }
  ~mpsim_gpu_shard() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (state) mpsim_gpu_state_destroy(state);
    if (comm && owns_comm) nccl().CommDestroy(comm);
  }
};

namespace {

mpsim_gpu_shard& SH(mpsim_gpu_shard* s) {
  if (!s) fail(MPSIM_EINVAL, "null shard");
  return *s;
}

void sync(mpsim_gpu_shard& s) { CKH(cudaStreamSynchronize(s.stream())); }

// ---- collectives on the shard stream (host scalars in and out)
void allreduce(mpsim_gpu_shard& s, double* v, int count, ncclRedOp_t op) {
  if (s.world == 1) return;
  s.red.ensure(sizeof(double) * count);
  s.red_host.ensure(sizeof(double) * count);
  std::memcpy(s.red_host.p, v, sizeof(double) * count);
  CKH(cudaMemcpyAsync(s.red.p, s.red_host.p, sizeof(double) * count, cudaMemcpyHostToDevice, s.stream()));
  NC(nccl().AllReduce(s.red.p, s.red.p, count, ncclFloat64, op, s.comm, s.stream()));
  CKH(cudaMemcpyAsync(s.red_host.p, s.red.p, sizeof(double) * count, cudaMemcpyDeviceToHost, s.stream()));
  sync(s);
  std::memcpy(v, s.red_host.p, sizeof(double) * count);
}

// One point-to-point round: send local slot `send_li` (with its extents) to
// rank `dst` and / or receive a slot into local slot `recv_li` from `src`, in
// one NCCL group (both directions at once cannot deadlock).
void p2p(mpsim_gpu_shard& s, int send_li, int dst, int recv_li, int src) {
  NvtxRange nv("mpsim: shard boundary exchange (NCCL)");
  State& a = s.st();
  const auto& api = nccl();
  const size_t slot = (size_t)a.stride * 2;  // doubles per padded slot
  s.dims_send.ensure(2 * sizeof(int64_t));
  s.dims_recv.ensure(2 * sizeof(int64_t));
  s.dims_host.ensure(4 * sizeof(int64_t));
  int64_t* hd = (int64_t*)s.dims_host.p;
  if (send_li >= 0) {
    hd[0] = a.sdl[send_li];
    hd[1] = a.sdr[send_li];
    CKH(cudaMemcpyAsync(s.dims_send.p, hd, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, s.stream()));
  }
  NC(api.GroupStart());
  if (send_li >= 0) {
    NC(api.Send(s.dims_send.p, 2, ncclInt64, dst, s.comm, s.stream()));
    NC(api.Send(a.sites + (long long)send_li * a.stride, slot, ncclFloat64, dst, s.comm, s.stream()));
  }
  if (recv_li >= 0) {
    NC(api.Recv(s.dims_recv.p, 2, ncclInt64, src, s.comm, s.stream()));
    NC(api.Recv(a.sites + (long long)recv_li * a.stride, slot, ncclFloat64, src, s.comm, s.stream()));
  }
  NC(api.GroupEnd());
  if (recv_li >= 0) {
    CKH(cudaMemcpyAsync(hd + 2, s.dims_recv.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s.stream()));
    sync(s);
    ABI(mpsim_gpu_set_site_dims(s.state, recv_li, hd[2], hd[3]));
  } else {
    sync(s);  // the pinned extents are reused by the next call
  }
}

// All ranks agree on the slot capacity before slots move (a rank whose bonds
// outgrew chi regrew its store; the neighbours follow).
void agree_capacity(mpsim_gpu_shard& s) {
  if (s.world == 1) return;
  double c = (double)s.st().chi;
  allreduce(s, &c, 1, ncclMax);
  if ((long long)c > s.st().chi) s.st().grow((int)c);
  s.capacity_agreed = true;
}

void apply_layer(mpsim_gpu_shard& s, const mpsim_gate* gates, int count, const mpsim_policy& pol,
                 mpsim_exec_stats* stats) {
  NvtxRange nv("mpsim: shard layer (exchange, layer, exchange)");
  DeviceGuard g(s.device);
  std::vector<mpsim_gate> local;
  bool sl = false, sr = false;
  partition_layer(gates, count, s.lo, s.hi, s.rank, s.world, local, sl, sr);
  if (s.world > 1 && (!s.capacity_agreed || pol.max_bond > s.st().chi)) agree_capacity(s);
  CKH(cudaEventRecord(s.e0, s.stream()));
  if (sl || sr) p2p(s, sl ? 0 : -1, s.rank - 1, sr ? s.n_local - 1 : -1, s.rank + 1);  // exchange in
  mpsim_exec_stats es{};
  if (!local.empty())
    ABI(mpsim_gpu_execute(s.state, local.data(), (int)local.size(), &pol, MPSIM_NONLOCAL_SWAP, &es, nullptr));
  if (sl || sr) p2p(s, sr ? s.n_local - 1 : -1, s.rank + 1, sl ? 0 : -1, s.rank - 1);  // exchange out
  CKH(cudaEventRecord(s.e1, s.stream()));
  CKH(cudaEventSynchronize(s.e1));
  float ms = 0.f;
  CKH(cudaEventElapsedTime(&ms, s.e0, s.e1));
  s.center = -1;  // the gates moved or scrambled the gauge (gate_apply.cpp:70-77 per gate)
  if (stats) {
    *stats = es;
    stats->device_ms = ms;  // exchange in + layer + exchange out
    stats->layers = 1;
  }
}

// Environment hand-off down the chain: compute(env_in device or nullptr,
// env_out device) on every rank in order; the last rank's `result` values
// (complex) are broadcast to every rank.
template <class F>
void env_chain(mpsim_gpu_shard& s, size_t in_elems, size_t out_elems, size_t result, F&& compute, double* out) {
  const auto& api = nccl();
  s.scratch.ensure(sizeof(cplx) * std::max<size_t>(in_elems, 1));
  s.scratch2.ensure(sizeof(cplx) * std::max<size_t>(std::max(out_elems, result), 1));
  cplx* ein = (cplx*)s.scratch.p;
  cplx* eout = (cplx*)s.scratch2.p;
  if (s.rank > 0) NC(api.Recv(ein, 2 * in_elems, ncclFloat64, s.rank - 1, s.comm, s.stream()));
  sync(s);
  compute(s.rank > 0 ? ein : nullptr, eout);
  if (s.rank < s.world - 1) NC(api.Send(eout, 2 * out_elems, ncclFloat64, s.rank + 1, s.comm, s.stream()));
  NC(api.Broadcast(eout, eout, 2 * result, ncclFloat64, s.world - 1, s.comm, s.stream()));
  CKH(cudaMemcpyAsync(out, eout, sizeof(cplx) * result, cudaMemcpyDeviceToHost, s.stream()));
  sync(s);
}

// <a| O_q |b> over both shard sets (same bounds): transfer environments.
void transfer(mpsim_gpu_shard& a, mpsim_gpu_shard& b, const double* op, int q_global, double* out) {
  DeviceGuard g(a.device);
  const int k = a.hi - a.lo;
  const int q = (op && a.lo <= q_global && q_global < a.hi) ? q_global - a.lo : -1;
  const double* o = q >= 0 ? op : nullptr;
  if (a.world == 1) {
    ABI(mpsim_gpu_transfer_env(a.state, b.state, 0, k, o, q, nullptr, out));
    return;
  }
  const State& x = a.st();
  const State& y = b.st();
  const size_t din = (size_t)x.sdl[0] * y.sdl[0], dout = (size_t)x.sdr[k - 1] * y.sdr[k - 1];
  env_chain(a, din, dout, 1, [&](const cplx* ein, cplx* eout) {
    ABI(mpsim_gpu_transfer_env(a.state, b.state, 0, k, o, q, (const double*)ein, (double*)eout));
  }, out);
}

// Centre moves across the shards (move_center, mps.cpp:177-187) on state
// `a` (the shard's own, or a canonicalised copy with the same layout).
void move_center(mpsim_gpu_shard& s, int c) {
  if (c < 0 || c >= s.n) fail(MPSIM_EINVAL, "center out of range");
  DeviceGuard g(s.device);
  if (s.world == 1) {
    ABI(mpsim_gpu_move_center(s.state, c));
    s.center = c;
    return;
  }
  agree_capacity(s);
  const std::vector<int> bounds = shard_bounds(s.n, s.world, s.chi);
  int rc = 0;
  for (int r = 0; r < s.world; ++r)
    if (bounds[(size_t)r] <= c) rc = r;
  const int k = s.hi - s.lo, ghost = k, r = s.rank;
  if (r <= rc) {  // left sweep (mps.cpp:69-80), ranks 0 .. rc in order
    if (r > 0) {
      p2p(s, 0, r - 1, -1, -1);  // my first site becomes r-1's ghost ...
      p2p(s, -1, -1, 0, r - 1);  // ... and comes back with its R absorbed
    }
    if (r < rc) {
      p2p(s, -1, -1, ghost, r + 1);
      ABI(mpsim_gpu_sweep_left(s.state, 0, k));
      p2p(s, ghost, r + 1, -1, -1);
    } else {
      ABI(mpsim_gpu_sweep_left(s.state, 0, c - s.lo));
    }
  }
  if (r >= rc) {  // right sweep (mps.cpp:84-95), ranks world-1 .. rc in order
    if (r < s.world - 1) {
      p2p(s, -1, -1, ghost, r + 1);
      ABI(mpsim_gpu_sweep_right(s.state, ghost, ghost));
      p2p(s, ghost, r + 1, -1, -1);
    }
    const int lo_step = r > rc ? 1 : c - s.lo + 1;
    if (k - 1 >= lo_step) ABI(mpsim_gpu_sweep_right(s.state, lo_step, k - 1));
    if (r > rc) {
      p2p(s, 0, r - 1, -1, -1);
      p2p(s, -1, -1, 0, r - 1);
    }
  }
  double bad = 0.0;  // mps.cpp:183-185, decided on the centre's rank, raised everywhere
  if (r == rc) {
    double n2 = 0.0;
    ABI(mpsim_gpu_site_norm2(s.state, c - s.lo, &n2));
    if (std::sqrt(n2) < 1e-14) bad = 1.0;
  }
  allreduce(s, &bad, 1, ncclMax);
  if (bad > 0.0) fail(MPSIM_ENUMERIC, "cannot canonicalize a zero-norm state");
  s.center = c;
}

// A shard handle over a copy of the local state, sharing the communicator.
mpsim_gpu_shard* clone(mpsim_gpu_shard& s) {
  auto* c = new mpsim_gpu_shard();
  c->n = s.n;
  c->rank = s.rank;
  c->world = s.world;
  c->device = s.device;
  c->chi = s.chi;
  c->lo = s.lo;
  c->hi = s.hi;
  c->n_local = s.n_local;
  c->has_right = s.has_right;
  c->comm = s.comm;
  c->owns_comm = false;
  try {
    ABI(mpsim_gpu_state_copy(s.state, &c->state));
    if (s.world > 1) ABI(mpsim_gpu_set_open_boundaries(c->state, 1));
    CKH(cudaEventCreate(&c->e0));
    CKH(cudaEventCreate(&c->e1));
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

// Perfect sampling across the shards (Sampler, sampler.cpp:35-143): a left +
// right canonicalised copy, then shot chunks walked rank by rank; each rank
// starts from the distinct-prefix environments and per-shot prefix indices its
// left neighbour hands over. Variates: the reference's shot-major
// mt19937_64 stream (one engine across chunks), restricted to the rank's sites.
void sample(mpsim_gpu_shard& s, uint64_t shots, uint64_t seed, uint64_t chunk) {
  if (shots == 0) fail(MPSIM_EINVAL, "shots must be positive");
  if (chunk == 0) chunk = 4096;
  DeviceGuard g(s.device);
  const auto& api = nccl();
  double nv[2];
  transfer(s, s, nullptr, -1, nv);
  const double nrm = std::sqrt(std::max(0.0, nv[0]));
  if (std::abs(nrm - 1.0) > 1e-8)  // sampler.cpp:36-40
    fail(MPSIM_ENUMERIC, "sampling requires a normalized state, norm is " + std::to_string(nrm));
  mpsim_gpu_shard* prep = clone(s);
  try {
    move_center(*prep, s.n - 1);  // left_canonicalize (sampler.cpp:46)
    move_center(*prep, 0);        // right_canonicalize (sampler.cpp:47)
    State& ps = prep->st();
    const int k = s.hi - s.lo, n = s.n;
    const long long d0 = ps.sdl[0], dk = ps.sdr[k - 1];
    std::mt19937_64 eng(seed);
    std::vector<double> uall, u;
    std::vector<char> mine((size_t)shots * k);
    std::vector<int32_t> node_in, node_out;
    DeviceBuf env_in, env_out, meta, nodes;
    PinnedBuf meta_h;
    meta.ensure(sizeof(int64_t));
    meta_h.ensure(sizeof(int64_t));
    for (uint64_t c0 = 0; c0 < shots; c0 += chunk) {
      const uint64_t cs = std::min(chunk, shots - c0);
      uall.resize((size_t)cs * n);
      for (double& x : uall) x = static_cast<double>(eng() >> 11) * 0x1.0p-53;
      u.resize((size_t)cs * k);
      for (uint64_t sh = 0; sh < cs; ++sh)
        std::memcpy(&u[(size_t)sh * k], &uall[(size_t)sh * n + s.lo], sizeof(double) * k);
      int32_t U = 1;
      const cplx* ein = nullptr;
      const int32_t* nin = nullptr;
      nodes.ensure(sizeof(int32_t) * cs);
      if (s.rank > 0) {
        NC(api.Recv(meta.p, 1, ncclInt64, s.rank - 1, prep->comm, ps.st));
        CKH(cudaMemcpyAsync(meta_h.p, meta.p, sizeof(int64_t), cudaMemcpyDeviceToHost, ps.st));
        CKH(cudaStreamSynchronize(ps.st));
        U = (int32_t) * (int64_t*)meta_h.p;
        env_in.ensure(sizeof(cplx) * (size_t)U * d0);
        NC(api.GroupStart());
        NC(api.Recv(env_in.p, 2 * (size_t)U * d0, ncclFloat64, s.rank - 1, prep->comm, ps.st));
        NC(api.Recv(nodes.p, cs, ncclInt32, s.rank - 1, prep->comm, ps.st));
        NC(api.GroupEnd());
        node_in.resize(cs);
        CKH(cudaMemcpyAsync(node_in.data(), nodes.p, sizeof(int32_t) * cs, cudaMemcpyDeviceToHost, ps.st));
        CKH(cudaStreamSynchronize(ps.st));
        ein = (const cplx*)env_in.p;
        nin = node_in.data();
      }
      env_out.ensure(sizeof(cplx) * (size_t)cs * dk);
      node_out.resize(cs);
      int32_t U_out = 0;
      ABI(mpsim_gpu_sample_segment_dev(prep->state, 0, k, cs, u.data(), U, (const double*)ein, nin, &U_out,
                                       (double*)env_out.p, node_out.data(), &mine[(size_t)c0 * k]));
      if (s.rank < s.world - 1) {
        *(int64_t*)meta_h.p = U_out;
        CKH(cudaMemcpyAsync(meta.p, meta_h.p, sizeof(int64_t), cudaMemcpyHostToDevice, ps.st));
        CKH(cudaMemcpyAsync(nodes.p, node_out.data(), sizeof(int32_t) * cs, cudaMemcpyHostToDevice, ps.st));
        NC(api.Send(meta.p, 1, ncclInt64, s.rank + 1, prep->comm, ps.st));
        NC(api.GroupStart());
        NC(api.Send(env_out.p, 2 * (size_t)U_out * dk, ncclFloat64, s.rank + 1, prep->comm, ps.st));
        NC(api.Send(nodes.p, cs, ncclInt32, s.rank + 1, prep->comm, ps.st));
        NC(api.GroupEnd());
        CKH(cudaStreamSynchronize(ps.st));  // meta_h / node_out are reused next chunk
      }
    }
    // every rank's bits of every shot -> ordered counts (sampler.cpp:140);
    // one all-gather per block of shots after the walk, padded to the widest shard
    const std::vector<int> b = shard_bounds(n, s.world, s.chi);
    int kmax = 0;
    for (int r = 0; r < s.world; ++r) kmax = std::max(kmax, b[(size_t)r + 1] - b[(size_t)r]);
    std::map<std::string, uint64_t> counts;
    const uint64_t block = std::max<uint64_t>(1, (64ull << 20) / ((uint64_t)kmax * s.world));
    DeviceBuf gsend, grecv;
    std::vector<char> pad, all;
    std::string key((size_t)n, '0');
    for (uint64_t s0 = 0; s0 < shots; s0 += block) {
      const uint64_t bs = std::min(block, shots - s0);
      pad.assign((size_t)bs * kmax, '0');
      for (uint64_t sh = 0; sh < bs; ++sh) std::memcpy(&pad[(size_t)sh * kmax], &mine[(size_t)(s0 + sh) * k], k);
      all.resize((size_t)bs * kmax * s.world);
      if (s.world == 1) {
        all = pad;
      } else {
        gsend.ensure(pad.size());
        grecv.ensure(all.size());
        CKH(cudaMemcpyAsync(gsend.p, pad.data(), pad.size(), cudaMemcpyHostToDevice, ps.st));
        NC(api.AllGather(gsend.p, grecv.p, pad.size(), ncclUint8, prep->comm, ps.st));
        CKH(cudaMemcpyAsync(all.data(), grecv.p, all.size(), cudaMemcpyDeviceToHost, ps.st));
        CKH(cudaStreamSynchronize(ps.st));
      }
      for (uint64_t sh = 0; sh < bs; ++sh) {
        for (int r = 0; r < s.world; ++r) {
          const int w = b[(size_t)r + 1] - b[(size_t)r];
          std::memcpy(&key[(size_t)b[(size_t)r]], &all[((size_t)r * bs + sh) * kmax], (size_t)w);
        }
        ++counts[key];
      }
    }
    s.result.assign(counts.begin(), counts.end());
  } catch (...) {
    delete prep;
    throw;
  }
  delete prep;
}

}  // namespace

extern "C" {

int mpsim_shard_bounds(int32_t n_qubits, int32_t world, int64_t chi, int32_t* out) {
  return sguard([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    const std::vector<int> b = shard_bounds(n_qubits, world, chi);
    for (size_t i = 0; i < b.size(); ++i) out[i] = b[i];
  });
}

int mpsim_shard_partition_layer(const mpsim_gate* gates, int32_t count, int32_t lo, int32_t hi, int32_t rank,
                                int32_t world, mpsim_gate* local, int32_t* n_local, int32_t* straddle_left,
                                int32_t* straddle_right) {
  return sguard([&] {
    if ((!gates && count) || !local || !n_local || !straddle_left || !straddle_right) fail(MPSIM_EINVAL, "null argument");
    std::vector<mpsim_gate> v;
    bool sl = false, sr = false;
    partition_layer(gates, count, lo, hi, rank, world, v, sl, sr);
    std::copy(v.begin(), v.end(), local);
    *n_local = (int32_t)v.size();
    *straddle_left = sl;
    *straddle_right = sr;
  });
}

int mpsim_gpu_nccl_unique_id(void* id_out) {
  return sguard([&] {
    if (!id_out) fail(MPSIM_EINVAL, "null output");
    ncclUniqueId id;
    NC(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int mpsim_gpu_shard_create(int32_t n_qubits, int64_t chi, int32_t rank, int32_t world, const void* nccl_id,
                           int32_t device, mpsim_gpu_shard** out) {
  return sguard([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    if (world < 1 || rank < 0 || rank >= world) fail(MPSIM_EINVAL, "rank out of range");
    if (world > 1 && !nccl_id) fail(MPSIM_EINVAL, "a multi-rank shard needs the NCCL unique id of rank 0");
    if (chi < 1) fail(MPSIM_EINVAL, "chi must be positive");
    auto* s = new mpsim_gpu_shard();
    try {
      s->n = n_qubits;
      s->rank = rank;
      s->world = world;
      s->device = device;
      s->chi = chi;
      const std::vector<int> b = shard_bounds(n_qubits, world, chi);
      s->lo = b[(size_t)rank];
      s->hi = b[(size_t)rank + 1];
      s->has_right = rank < world - 1;
      s->n_local = s->hi - s->lo + (s->has_right ? 1 : 0);
      DeviceGuard g(device);
      ABI(mpsim_gpu_state_create(s->n_local, chi, device, &s->state));
      if (world > 1) ABI(mpsim_gpu_set_open_boundaries(s->state, 1));
      CKH(cudaEventCreate(&s->e0));
      CKH(cudaEventCreate(&s->e1));
      if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        NC(nccl().CommInitRank(&s->comm, world, id, rank));
        s->owns_comm = true;
      }
      s->center = world == 1 ? 0 : -1;
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int mpsim_gpu_shard_destroy(mpsim_gpu_shard* s) {
  return sguard([&] { delete s; });
}

int mpsim_gpu_shard_info(const mpsim_gpu_shard* s, int32_t* lo, int32_t* hi, mpsim_gpu_state** local_state) {
  return sguard([&] {
    if (!s) fail(MPSIM_EINVAL, "null shard");
    if (lo) *lo = s->lo;
    if (hi) *hi = s->hi;
    if (local_state) *local_state = s->state;
  });
}

int mpsim_gpu_shard_set_site(mpsim_gpu_shard* s, int32_t i, int64_t dl, int64_t dr, const double* data) {
  return sguard([&] {
    mpsim_gpu_shard& a = SH(s);
    if (i < a.lo || i >= a.hi) fail(MPSIM_EINVAL, "site " + std::to_string(i) + " is not owned by this shard");
    ABI(mpsim_gpu_set_site(a.state, i - a.lo, dl, dr, data));
    a.capacity_agreed = false;
    if (a.has_right && i == a.hi - 1) {  // the ghost slot's extents follow the last owned bond
      ABI(mpsim_gpu_set_site_dims(a.state, a.n_local - 1, dr, 1));
    }
    a.center = -1;
  });
}

int mpsim_gpu_shard_get_site(mpsim_gpu_shard* s, int32_t i, int64_t* dl, int64_t* dr, double* out) {
  return sguard([&] {
    mpsim_gpu_shard& a = SH(s);
    if (i < a.lo || i >= a.hi) fail(MPSIM_EINVAL, "site " + std::to_string(i) + " is not owned by this shard");
    ABI(mpsim_gpu_get_site(a.state, i - a.lo, dl, dr, out));
  });
}

int mpsim_gpu_shard_bond_dims(mpsim_gpu_shard* s, int64_t* out) {
  return sguard([&] {
    mpsim_gpu_shard& a = SH(s);
    if (!out) fail(MPSIM_EINVAL, "null output");
    const State& x = a.st();
    for (int i = 0; i <= a.hi - a.lo; ++i) out[i] = x.bonds[(size_t)i];
  });
}

int mpsim_gpu_shard_apply_layer(mpsim_gpu_shard* s, const mpsim_gate* gates, int32_t count,
                                const mpsim_policy* policy, mpsim_exec_stats* stats) {
  return sguard([&] {
    if (!policy || (!gates && count)) fail(MPSIM_EINVAL, "null argument");
    apply_layer(SH(s), gates, count, *policy, stats);
  });
}

int mpsim_gpu_shard_execute(mpsim_gpu_shard* s, const mpsim_gate* gates, int32_t count, const mpsim_policy* policy,
                            mpsim_exec_stats* stats) {
  return sguard([&] {
    mpsim_gpu_shard& a = SH(s);
    if (!policy || (!gates && count)) fail(MPSIM_EINVAL, "null argument");
    // decompose_nonlocal + layerize over the whole chain (fusion.cpp:137-190):
    // every rank plans identically, then runs the layers in order.
    mpsim_gate* low = nullptr;
    int32_t* layer_of = nullptr;
    int32_t nlow = 0, nlayers = 0;
    ABI(mpsim_plan_layers(gates, count, a.n, &low, &layer_of, &nlow, &nlayers));
    std::vector<mpsim_gate> lg(low, low + nlow);
    std::vector<int32_t> lo(layer_of, layer_of + nlow);
    mpsim_free(low);
    mpsim_free(layer_of);
    double acc[2] = {0.0, 0.0};  // discarded weight (sum), device ms
    double peak = 1.0;
    long long launches = 0;
    for (int32_t i = 0, L = 0; L < nlayers; ++L) {
      int32_t j = i;
      while (j < nlow && lo[(size_t)j] == L) ++j;
      mpsim_exec_stats es{};
      apply_layer(a, lg.data() + i, j - i, *policy, &es);
      acc[0] += es.total_discarded_weight;
      acc[1] += es.device_ms;
      peak = std::max(peak, (double)es.peak_bond);
      launches += es.kernel_launches;
      i = j;
    }
    allreduce(a, acc, 1, ncclSum);
    allreduce(a, &peak, 1, ncclMax);
    if (stats) {
      stats->peak_bond = (int64_t)peak;
      stats->total_discarded_weight = acc[0];
      stats->layers = nlayers;
      stats->gates = nlow;
      stats->kernel_launches = launches;
      stats->device_ms = acc[1];
    }
  });
}

int mpsim_gpu_shard_amplitudes(mpsim_gpu_shard* s, const char* bits, int32_t count, double* out) {
  return sguard([&] {
    mpsim_gpu_shard& a = SH(s);
    if ((!bits && count) || !out) fail(MPSIM_EINVAL, "null argument");
    DeviceGuard g(a.device);
    const int k = a.hi - a.lo;
    std::vector<char> local((size_t)count * a.n_local, '0');
    for (int32_t c = 0; c < count; ++c)
      std::memcpy(&local[(size_t)c * a.n_local], bits + (size_t)c * a.n + a.lo, (size_t)k);
    if (a.world == 1) {
      ABI(mpsim_gpu_amplitudes_env(a.state, 0, k, local.data(), count, nullptr, out));
      return;
    }
    const State& x = a.st();
    env_chain(a, (size_t)count * x.sdl[0], (size_t)count * x.sdr[k - 1], (size_t)count,
              [&](const cplx* ein, cplx* eout) {
                ABI(mpsim_gpu_amplitudes_env(a.state, 0, k, local.data(), count, (const double*)ein, (double*)eout));
              },
              out);
  });
}

int mpsim_gpu_shard_overlap(mpsim_gpu_shard* a, mpsim_gpu_shard* b, double* out) {
  return sguard([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    if (SH(a).lo != SH(b).lo || SH(a).hi != SH(b).hi) fail(MPSIM_EINVAL, "overlap needs chains sharded alike");
    transfer(SH(a), SH(b), nullptr, -1, out);
  });
}

int mpsim_gpu_shard_norm(mpsim_gpu_shard* s, double* out) {
  return sguard([&] {
    if (!out) fail(MPSIM_EINVAL, "null output");
    double v[2];
    transfer(SH(s), SH(s), nullptr, -1, v);
    *out = std::sqrt(std::max(0.0, v[0]));
  });
}

int mpsim_gpu_shard_expect_1q(mpsim_gpu_shard* s, const double* op2x2, int32_t q, double* out) {
  return sguard([&] {
    if (!op2x2 || !out) fail(MPSIM_EINVAL, "null argument");
    if (q < 0 || q >= SH(s).n) fail(MPSIM_EINVAL, "qubit out of range");
    transfer(SH(s), SH(s), op2x2, q, out);
  });
}

int mpsim_gpu_shard_move_center(mpsim_gpu_shard* s, int32_t c) {
  return sguard([&] { move_center(SH(s), c); });
}

int mpsim_gpu_shard_ortho_center(const mpsim_gpu_shard* s, int32_t* out) {
  return sguard([&] {
    if (!s || !out) fail(MPSIM_EINVAL, "null argument");
    *out = s->center;
  });
}

int mpsim_gpu_shard_sample(mpsim_gpu_shard* s, uint64_t shots, uint64_t seed, uint64_t chunk, int32_t* unique) {
  return sguard([&] {
    sample(SH(s), shots, seed, chunk);
    if (unique) *unique = (int32_t)s->result.size();
  });
}

int mpsim_gpu_shard_sample_result(const mpsim_gpu_shard* s, int32_t i, char* bits, uint64_t* count) {
  return sguard([&] {
    if (!s || i < 0 || (size_t)i >= s->result.size() || !bits || !count) fail(MPSIM_EINVAL, "result index out of range");
    std::memcpy(bits, s->result[(size_t)i].first.data(), s->result[(size_t)i].first.size());
    *count = s->result[(size_t)i].second;
  });
}

int mpsim_gpu_shard_allreduce(mpsim_gpu_shard* s, double* values, int32_t count, int32_t op) {
  return sguard([&] {
    if (!values && count) fail(MPSIM_EINVAL, "null argument");
    DeviceGuard g(SH(s).device);
    allreduce(*s, values, count, op == MPSIM_REDUCE_MAX ? ncclMax : op == MPSIM_REDUCE_MIN ? ncclMin : ncclSum);
  });
}

int mpsim_gpu_shard_barrier(mpsim_gpu_shard* s) {
  return sguard([&] {
    DeviceGuard g(SH(s).device);
    double x = 0.0;
    allreduce(*s, &x, 1, ncclSum);
    CKH(cudaDeviceSynchronize());
  });
}

}  // extern "C"
