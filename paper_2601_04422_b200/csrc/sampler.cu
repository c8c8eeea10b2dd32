// Perfect sampling (Sampler, sampler.cpp:35-154) as a batched-shot
// transfer-matrix walk on the GPU.
//
// The reference walks shot by shot with a prefix memo. Here all shots advance
// together site by site; shots with an identical bit prefix share one left
// environment (a node of the prefix tree), so every distinct prefix's
// environment and P(0) are computed exactly once — the memo, in bulk. Per site:
//   T = E [A0 | A1]            (nodes x 2Dr, complex GEMM)
//   raw_b = ||T_b row||^2, P0 = raw0 / (raw0 + raw1)            (row kernel)
//   bit = u < P0, u = the reference's mt19937_64 variate for (shot, site)
//   E' = T_bit row / sqrt(raw_bit), one row per (node, bit) child (gather kernel)
// Variates are drawn on the host from std::mt19937_64 in the reference order
// (one per qubit per shot, shot-major, sampler.cpp:84/115), so counts match
// the reference for the same seed. Cache statistics (hits / size / cap) are
// replayed on a host trie in the reference's shot-major order.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "engine.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {

void launch_cgemm(const GemmArgs&, cudaStream_t);
void move_center_impl(State& s, int c);

__global__ void row_norms2_kernel(const cplx* __restrict__ T, long long ld, int rows, int dr, double* __restrict__ raw) {
  // raw[2*r + b] = ||T[r, b*dr:(b+1)*dr]||^2 ; one warp per (row, b)
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (w >= 2 * rows) return;
  const int r = w / 2, b = w % 2;
  const cplx* x = T + (long long)r * ld + (long long)b * dr;
  double s = 0.0;
  for (int i = lane; i < dr; i += 32) s += cabs2(x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) raw[w] = s;
}

// E'[c][j] = T[src[c]][bit[c]*dr + j] * scale[c]
__global__ void gather_env_kernel(const cplx* __restrict__ T, long long ldt, int dr, const int* __restrict__ src,
                                  const int* __restrict__ bit, const double* __restrict__ scale, int children,
                                  cplx* __restrict__ E, long long lde) {
  const long long total = (long long)children * dr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / dr), j = (int)(i % dr);
    const cplx v = T[(long long)src[c] * ldt + (long long)bit[c] * dr + j];
    E[(long long)c * lde + j] = make_double2(v.x * scale[c], v.y * scale[c]);
  }
}

}  // namespace mpsim_gpu

using namespace mpsim_gpu;

namespace {

template <class F>
int sguard(F&& f) {
  try {
    f();
    return MPSIM_OK;
  } catch (const Error& e) {
    last_error_slot() = e.what();
    return e.code;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return MPSIM_ELOGIC;
  }
}

#define CKS(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) fail(MPSIM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr double kDegenerate = 1e-12;  // sampler.cpp:31

// Host trie over bit prefixes: the reference's cache entries (prefix -> env,
// P0) for the statistics replay.
struct Trie {
  std::vector<int> child;  // 2 per node
  std::vector<char> entry, known;
  Trie() { reset(); }
  void reset() {
    child.assign(2, -1);
    entry.assign(1, 0);
    known.assign(1, 0);
  }
  int step(int node, int b) {
    int& c = child[2 * (size_t)node + b];
    if (c < 0) {
      c = (int)entry.size();
      child.push_back(-1);
      child.push_back(-1);
      entry.push_back(0);
      known.push_back(0);
    }
    return child[2 * (size_t)node + b];
  }
};

}  // namespace

struct mpsim_gpu_sampler {
  State* st = nullptr;  // canonicalised copy
  int n = 0;
  bool memoize = true;
  uint64_t cap = 0;
  Trie trie;
  bool root_known = false;
  uint64_t cache_size = 0, hits = 0;
  std::vector<std::pair<std::string, uint64_t>> result;
  ~mpsim_gpu_sampler() { delete st; }
};

namespace {

// The walk over sites [i0, i1): U distinct prefixes (nodes) with their left
// environments dE (U x sdl[i0], device, ld = sdl[i0]); node_of[shot] the
// shot's node; prefix[node] its bits so far; u(shot, site) the variate.
// On return dE holds the U' x sdr[i1 - 1] environments of the new nodes.
template <class Var>
void sample_walk(State& s, int i0, int i1, uint64_t shots, Var u, int& U, DeviceBuf& dE,
                 std::vector<int>& node_of, std::vector<std::string>& prefix) {
  DeviceBuf dE2, dT, dRaw, dSrc, dBit, dScale;
  const cplx one = make_double2(1.0, 0.0);
  std::vector<double> raw;
  for (int site = i0; site < i1; ++site) {
    const int dl = (int)s.sdl[site], dr = (int)s.sdr[site];
    const cplx* A = s.sites + (long long)site * s.stride;
    dT.ensure(sizeof(cplx) * (size_t)U * 2 * dr);
    dRaw.ensure(sizeof(double) * (size_t)U * 2);
    for (int p = 0; p < 2; ++p) {
      GemmArgs ga{U, dr, dl, (const cplx*)dE.p, dl, 0, A + (long long)p * s.chi, 2LL * s.chi, 0,
                  (cplx*)dT.p + (long long)p * dr, 2LL * dr, one, 0};
      launch_cgemm(ga, s.st);
      ++s.launches;
    }
    row_norms2_kernel<<<(unsigned)((2LL * U * 32 + 255) / 256), 256, 0, s.st>>>((const cplx*)dT.p, 2LL * dr, U, dr,
                                                                               (double*)dRaw.p);
    ++s.launches;
    raw.resize((size_t)U * 2);
    CKS(cudaMemcpyAsync(raw.data(), dRaw.p, sizeof(double) * U * 2, cudaMemcpyDeviceToHost, s.st));
    CKS(cudaStreamSynchronize(s.st));
    CKS(cudaGetLastError());
    std::vector<double> p0((size_t)U);
    for (int k = 0; k < U; ++k) {
      const double tot = raw[2 * (size_t)k] + raw[2 * (size_t)k + 1];
      if (tot < kDegenerate)
        fail(MPSIM_ENUMERIC, "degenerate state: total probability vanished at site " + std::to_string(site));
      p0[(size_t)k] = raw[2 * (size_t)k] / tot;
    }
    // children
    std::vector<int> child_id((size_t)U * 2, -1), src, bits;
    std::vector<double> scale;
    std::vector<std::string> nprefix;
    for (uint64_t sh = 0; sh < shots; ++sh) {
      const int k = node_of[sh];
      const int b = u(sh, site) < p0[(size_t)k] ? 0 : 1;  // sampler.cpp:116-117
      int& cid = child_id[2 * (size_t)k + b];
      if (cid < 0) {
        const double r = raw[2 * (size_t)k + b];
        if (r < kDegenerate * kDegenerate) fail(MPSIM_ENUMERIC, "degenerate state: chosen branch has no weight");
        cid = (int)src.size();
        src.push_back(k);
        bits.push_back(b);
        scale.push_back(1.0 / std::sqrt(r));
        nprefix.push_back(prefix[(size_t)k] + char('0' + b));
      }
      node_of[sh] = cid;
    }
    const int U2 = (int)src.size();
    dSrc.ensure(sizeof(int) * U2);
    dBit.ensure(sizeof(int) * U2);
    dScale.ensure(sizeof(double) * U2);
    dE2.ensure(sizeof(cplx) * (size_t)U2 * dr);
    CKS(cudaMemcpyAsync(dSrc.p, src.data(), sizeof(int) * U2, cudaMemcpyHostToDevice, s.st));
    CKS(cudaMemcpyAsync(dBit.p, bits.data(), sizeof(int) * U2, cudaMemcpyHostToDevice, s.st));
    CKS(cudaMemcpyAsync(dScale.p, scale.data(), sizeof(double) * U2, cudaMemcpyHostToDevice, s.st));
    long long blocks = ((long long)U2 * dr + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    gather_env_kernel<<<(unsigned)std::max(1LL, blocks), 256, 0, s.st>>>(
        (const cplx*)dT.p, 2LL * dr, dr, (const int*)dSrc.p, (const int*)dBit.p, (const double*)dScale.p, U2,
        (cplx*)dE2.p, dr);
    ++s.launches;
    CKS(cudaStreamSynchronize(s.st));
    CKS(cudaGetLastError());
    std::swap(dE, dE2);
    prefix.swap(nprefix);
    U = U2;
  }
}

// Statistics replay (sampler.cpp:91-138) of one chunk of shots: shot-major,
// site-minor, on the host trie that persists across chunks and calls.
void replay_stats(mpsim_gpu_sampler& sp, uint64_t shots, const std::vector<int>& node_of,
                  const std::vector<std::string>& prefix) {
  const int n = sp.n;
  // map (depth, node) -> trie node, built lazily per shot
  for (uint64_t sh = 0; sh < shots; ++sh) {
    int tnode = 0;
    for (int site = 0; site < n; ++site) {
      if (site == 0) {
        if (sp.root_known) ++sp.hits;
        else sp.root_known = true;
      } else if (sp.trie.entry[(size_t)tnode]) {
        if (sp.trie.known[(size_t)tnode]) ++sp.hits;
        else sp.trie.known[(size_t)tnode] = 1;
      }
      // bit of this shot at this site: the node at depth site+1 tells it
      const std::string& pre = prefix[(size_t)node_of[sh]];
      const int b = pre[(size_t)site] - '0';
      tnode = sp.trie.step(tnode, b);
      if (sp.trie.entry[(size_t)tnode]) continue;  // env reused from the cache
      if (sp.cap == 0 || sp.cache_size < sp.cap) {
        sp.trie.entry[(size_t)tnode] = 1;
        ++sp.cache_size;
      }
    }
  }
}

void run_sample(mpsim_gpu_sampler& sp, uint64_t shots, uint64_t seed) {
  NvtxRange nv("mpsim: sample");
  State& s = *sp.st;
  const int n = sp.n;
  DeviceGuard g(s.device);
  // Shots go in chunks so host variates (chunk x n doubles) and device
  // environments (distinct prefixes x 2 chi) stay bounded for any shot count;
  // the variates come from one engine that carries over between chunks, in the
  // reference order (shot-major, one per site, sampler.cpp:84/115).
  const uint64_t chunk = std::max<uint64_t>(1024, (256ull << 20) / (32ull * (uint64_t)s.chi));
  std::mt19937_64 eng(seed);
  std::map<std::string, uint64_t> counts;
  std::vector<double> u;
  std::vector<int> node_of;
  std::vector<std::string> prefix;
  DeviceBuf dE;
  const cplx one = make_double2(1.0, 0.0);
  for (uint64_t c0 = 0; c0 < shots; c0 += chunk) {
    const uint64_t cs = std::min(chunk, shots - c0);
    u.resize((size_t)cs * n);
    for (size_t i = 0; i < u.size(); ++i) u[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
    node_of.assign(cs, 0);  // shot -> node at the current depth
    prefix.assign(1, std::string());  // node -> prefix
    int U = 1;
    dE.ensure(sizeof(cplx) * s.chi);
    CKS(cudaMemcpyAsync(dE.p, &one, sizeof(cplx), cudaMemcpyHostToDevice, s.st));
    sample_walk(s, 0, n, cs, [&](uint64_t sh, int site) { return u[sh * n + site]; }, U, dE, node_of, prefix);
    // counts, lexicographic (std::map order, sampler.cpp:140)
    std::vector<uint64_t> cnt((size_t)U, 0);
    for (uint64_t sh = 0; sh < cs; ++sh) ++cnt[(size_t)node_of[sh]];
    for (int k = 0; k < U; ++k) counts[prefix[(size_t)k]] += cnt[(size_t)k];
    if (sp.memoize) replay_stats(sp, cs, node_of, prefix);
  }
  sp.result.assign(counts.begin(), counts.end());
}

}  // namespace

extern "C" {

int mpsim_gpu_sampler_create(const mpsim_gpu_state* s, int32_t memoize, uint64_t cap, mpsim_gpu_sampler** out) {
  return sguard([&] {
    if (!s || !out) fail(MPSIM_EINVAL, "null argument");
    double nrm = 0.0;
    if (mpsim_gpu_norm(s, &nrm) != MPSIM_OK) fail(MPSIM_ECUDA, mpsim_gpu_last_error());
    if (std::abs(nrm - 1.0) > 1e-8)  // sampler.cpp:36-40
      fail(MPSIM_ENUMERIC, "sampling requires a normalized state, norm is " + std::to_string(nrm));
    mpsim_gpu_state* copy = nullptr;
    if (mpsim_gpu_state_copy(s, &copy) != MPSIM_OK) fail(MPSIM_ECUDA, mpsim_gpu_last_error());
    auto* sp = new mpsim_gpu_sampler();
    sp->st = reinterpret_cast<State*>(copy);
    sp->n = sp->st->n;
    sp->memoize = memoize != 0;
    sp->cap = cap;
    try {
      move_center_impl(*sp->st, sp->n - 1);  // left_canonicalize (sampler.cpp:46)
      move_center_impl(*sp->st, 0);          // right_canonicalize (sampler.cpp:47)
    } catch (...) {
      delete sp;
      throw;
    }
    *out = sp;
  });
}

}  // extern "C"

namespace {

// env_dev: env_in / env_out live on the state's device (the sharded sampler's
// hand-off buffers, NCCL send/recv'd without a host round trip), else host.
int sample_segment_impl(const mpsim_gpu_state* s, int32_t i0, int32_t i1, uint64_t shots, const double* u,
                        int32_t u_in, const double* env_in, const int32_t* node_in, int32_t* u_out, double* env_out,
                        int32_t* node_out, char* bits_out, bool env_dev) {
  return sguard([&] {
    if (!s || !u || !u_out || !node_out || !bits_out) fail(MPSIM_EINVAL, "null argument");
    State& st = const_cast<State&>(*reinterpret_cast<const State*>(s));
    if (i0 < 0 || i1 > st.n || i0 >= i1) fail(MPSIM_EINVAL, "site range out of bounds");
    if (shots == 0) fail(MPSIM_EINVAL, "shots must be positive");
    DeviceGuard g(st.device);
    const int w = i1 - i0;
    int U = env_in ? u_in : 1;
    if (U < 1) fail(MPSIM_EINVAL, "need at least one input environment");
    if (!env_in && st.sdl[i0] != 1) fail(MPSIM_EINVAL, "open left bond needs input environments");
    DeviceBuf dE;
    const long long dl0 = st.sdl[i0];
    dE.ensure(sizeof(cplx) * (size_t)U * dl0);
    if (env_in) {
      CKS(cudaMemcpyAsync(dE.p, env_in, sizeof(cplx) * (size_t)U * dl0,
                          env_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st.st));
    } else {
      const cplx one = make_double2(1.0, 0.0);
      CKS(cudaMemcpyAsync(dE.p, &one, sizeof(cplx), cudaMemcpyHostToDevice, st.st));
    }
    std::vector<int> node_of(shots, 0);
    if (env_in && node_in)
      for (uint64_t sh = 0; sh < shots; ++sh) {
        if (node_in[sh] < 0 || node_in[sh] >= U) fail(MPSIM_EINVAL, "node index out of range");
        node_of[sh] = node_in[sh];
      }
    std::vector<std::string> prefix((size_t)U, std::string());
    sample_walk(st, i0, i1, shots, [&](uint64_t sh, int site) { return u[sh * w + (site - i0)]; }, U, dE, node_of,
                prefix);
    const long long dr = st.sdr[i1 - 1];
    if (env_out)
      CKS(cudaMemcpyAsync(env_out, dE.p, sizeof(cplx) * (size_t)U * dr,
                          env_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st.st));
    CKS(cudaStreamSynchronize(st.st));
    *u_out = U;
    for (uint64_t sh = 0; sh < shots; ++sh) {
      node_out[sh] = node_of[sh];
      std::memcpy(bits_out + sh * w, prefix[(size_t)node_of[sh]].data(), (size_t)w);
    }
  });
}

}  // namespace

extern "C" {

int mpsim_gpu_sample_segment(const mpsim_gpu_state* s, int32_t i0, int32_t i1, uint64_t shots, const double* u,
                             int32_t u_in, const double* env_in, const int32_t* node_in, int32_t* u_out,
                             double* env_out, int32_t* node_out, char* bits_out) {
  return sample_segment_impl(s, i0, i1, shots, u, u_in, env_in, node_in, u_out, env_out, node_out, bits_out, false);
}

int mpsim_gpu_sample_segment_dev(const mpsim_gpu_state* s, int32_t i0, int32_t i1, uint64_t shots, const double* u,
                                 int32_t u_in, const double* env_in, const int32_t* node_in, int32_t* u_out,
                                 double* env_out, int32_t* node_out, char* bits_out) {
  return sample_segment_impl(s, i0, i1, shots, u, u_in, env_in, node_in, u_out, env_out, node_out, bits_out, true);
}

int mpsim_uniform_variates(uint64_t seed, uint64_t skip, uint64_t count, double* out) {
  return sguard([&] {
    if (!out && count) fail(MPSIM_EINVAL, "null output");
    std::mt19937_64 eng(seed);
    eng.discard(skip);
    for (uint64_t i = 0; i < count; ++i) out[i] = static_cast<double>(eng() >> 11) * 0x1.0p-53;
  });
}

int mpsim_gpu_sampler_destroy(mpsim_gpu_sampler* sp) {
  return sguard([&] { delete sp; });
}

int mpsim_gpu_sample(mpsim_gpu_sampler* sp, uint64_t shots, uint64_t seed, int32_t* unique) {
  return sguard([&] {
    if (!sp) fail(MPSIM_EINVAL, "null sampler");
    if (shots == 0) fail(MPSIM_EINVAL, "shots must be positive");
    run_sample(*sp, shots, seed);
    if (unique) *unique = (int32_t)sp->result.size();
  });
}

int mpsim_gpu_sampler_result(const mpsim_gpu_sampler* sp, int32_t i, char* bits, uint64_t* count) {
  return sguard([&] {
    if (!sp || i < 0 || (size_t)i >= sp->result.size()) fail(MPSIM_EINVAL, "result index out of range");
    std::memcpy(bits, sp->result[(size_t)i].first.data(), sp->result[(size_t)i].first.size());
    *count = sp->result[(size_t)i].second;
  });
}

int mpsim_gpu_sampler_stats(const mpsim_gpu_sampler* sp, uint64_t* cache_hits, uint64_t* cache_size) {
  return sguard([&] {
    if (!sp) fail(MPSIM_EINVAL, "null sampler");
    if (cache_hits) *cache_hits = sp->hits;
    if (cache_size) *cache_size = sp->cache_size;
  });
}

int mpsim_gpu_sampler_clear_cache(mpsim_gpu_sampler* sp) {  // sampler.cpp:145-148
  return sguard([&] {
    if (!sp) fail(MPSIM_EINVAL, "null sampler");
    sp->trie.reset();
    sp->root_known = false;
    sp->cache_size = 0;
  });
}

}  // extern "C"
