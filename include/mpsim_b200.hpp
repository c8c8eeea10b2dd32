// mpsim_b200.hpp — header-only C++ facade of the B200 engine with the
// reference simulator's API (namespace mpsim; /root/reference/proj/include/
// mpsim/{tensor,mps,gate_apply,executor,sampler,errors}.hpp). A caller of the
// reference switches the include path and links libmpsim_gpu.so; names,
// argument meaning and exception types are kept:
//   std::invalid_argument  <- MPSIM_EINVAL (mpsim::ConfigError from the front end)
//   mpsim::ParseError      <- MPSIM_EPARSE (line / column kept)
//   mpsim::NumericError    <- MPSIM_ENUMERIC
//   std::logic_error       <- MPSIM_ELOGIC
//   std::runtime_error     <- MPSIM_ECUDA
// Differences, by design: the state lives in HBM, so MpsState::site(i)
// returns a host copy (write back with set_site) instead of a mutable
// reference (mps.hpp:45-46); execute_parallel's `workers` only selects the
// batched launch path (every layer is one launch sequence).
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <limits>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "mpsim_gpu.h"

namespace mpsim {

using Index = std::int64_t;
using Complex = std::complex<double>;
inline constexpr Index kUnbounded = std::numeric_limits<Index>::max();  // tensor.hpp:44

class NumericError : public std::runtime_error {  // errors.hpp:45-48
 public:
  using std::runtime_error::runtime_error;
};

class ParseError : public std::runtime_error {  // errors.hpp:22-37
 public:
  ParseError(int line, int column, const std::string& what) : std::runtime_error(what), line_(line), column_(column) {}
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

class ConfigError : public std::runtime_error {  // errors.hpp:39-43
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == MPSIM_OK) return;
  if (rc == MPSIM_EPARSE) {
    int32_t line = 0, col = 0;
    mpsim_last_parse_location(&line, &col);
    throw ParseError(line, col, mpsim_gpu_last_error());
  }
  const std::string msg = mpsim_gpu_last_error();
  switch (rc) {
    case MPSIM_EINVAL: throw std::invalid_argument(msg);
    case MPSIM_ENUMERIC: throw NumericError(msg);
    case MPSIM_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
// The front end's input errors are ConfigError (runner.cpp:42-62, :141-190).
inline void check_config(int rc) {
  if (rc == MPSIM_EINVAL) throw ConfigError(mpsim_gpu_last_error());
  check(rc);
}
}  // namespace detail

// Minimal dense row-major tensor (tensor.hpp:66-152) for gates and site copies.
class CTensor {
 public:
  CTensor() : data_(1) {}
  explicit CTensor(std::vector<Index> shape) : shape_(std::move(shape)) { data_.assign(count(), Complex{}); }
  CTensor(std::vector<Index> shape, std::vector<Complex> data) : shape_(std::move(shape)), data_(std::move(data)) {
    if (static_cast<Index>(data_.size()) != count()) throw std::invalid_argument("tensor data length mismatch");
  }
  int rank() const { return static_cast<int>(shape_.size()); }
  const std::vector<Index>& shape() const { return shape_; }
  Index extent(int a) const { return shape_.at(static_cast<size_t>(a)); }
  Index size() const { return static_cast<Index>(data_.size()); }
  Complex* data() { return data_.data(); }
  const Complex* data() const { return data_.data(); }
  Complex& operator[](Index i) { return data_[static_cast<size_t>(i)]; }
  const Complex& operator[](Index i) const { return data_[static_cast<size_t>(i)]; }

 private:
  Index count() const {
    Index n = 1;
    for (Index e : shape_) {
      if (e <= 0) throw std::invalid_argument("tensor extents must be positive");
      n *= e;
    }
    return n;
  }
  std::vector<Index> shape_;
  std::vector<Complex> data_;
};

struct TruncationPolicy {  // gate_apply.hpp:35-38
  Index max_bond = kUnbounded;
  double cutoff = 0.0;
};

struct ApplyReport {  // gate_apply.hpp:40-44
  double discarded_weight = 0.0;
  Index new_bond = 1;
  int svd_count = 0;
};

enum class NonlocalMethod { Swap, BondProp };  // gate_apply.hpp:71

struct FusedGate {  // circuit.hpp:71-81
  int q0 = 0;
  int q1 = -1;
  bool flipped = false;
  CTensor matrix;
  bool two_qubit() const { return q1 >= 0; }
  bool local() const { return !two_qubit() || q1 == q0 + 1; }
};

struct LayerPlan {  // circuit.hpp:85-95
  std::vector<std::vector<FusedGate>> layers;
};

struct ExecStats {  // executor.hpp:44-57 (per-layer timing replaced by device time)
  Index peak_bond = 1;
  double total_discarded_weight = 0.0;
  int layers = 0;
  double device_ms = 0.0;
};

class MpsState {  // mps.hpp:33-75
 public:
  explicit MpsState(int n_qubits, Index chi_hint = 16, int device = 0) {
    detail::check(mpsim_gpu_state_create(n_qubits, chi_hint, device, &h_));
  }
  MpsState(const MpsState& o) { detail::check(mpsim_gpu_state_copy(o.h_, &h_)); }
  MpsState& operator=(const MpsState& o) {
    if (this != &o) {
      mpsim_gpu_state* n = nullptr;
      detail::check(mpsim_gpu_state_copy(o.h_, &n));
      mpsim_gpu_state_destroy(h_);
      h_ = n;
    }
    return *this;
  }
  MpsState(MpsState&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  MpsState& operator=(MpsState&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  ~MpsState() {
    if (h_) mpsim_gpu_state_destroy(h_);
  }

  int num_qubits() const {
    int32_t n = 0;
    detail::check(mpsim_gpu_num_qubits(h_, &n));
    return n;
  }
  std::vector<Index> bond_dims() const {
    std::vector<Index> b(static_cast<size_t>(num_qubits()) + 1);
    detail::check(mpsim_gpu_bond_dims(h_, b.data()));
    return b;
  }
  Index bond_dim(int i) const { return bond_dims().at(static_cast<size_t>(i)); }
  void set_bond_dim(int i, Index d) { detail::check(mpsim_gpu_set_bond_dim(h_, i, d)); }
  Index max_bond_dim() const {
    Index m = 0;
    for (Index b : bond_dims()) m = b > m ? b : m;
    return m;
  }
  std::optional<int> ortho_center() const {
    int32_t c = -1;
    detail::check(mpsim_gpu_ortho_center(h_, &c));
    return c < 0 ? std::nullopt : std::optional<int>(c);
  }
  void set_ortho_center(std::optional<int> c) { detail::check(mpsim_gpu_set_ortho_center(h_, c.value_or(-1))); }
  void validate() const { detail::check(mpsim_gpu_validate(h_)); }
  Index total_elements() const {
    const auto b = bond_dims();
    Index t = 0;
    for (size_t i = 0; i + 1 < b.size(); ++i) t += b[i] * 2 * b[i + 1];
    return t;
  }
  // Host copy of site i, shape (Dl, 2, Dr).
  CTensor site(int i) const {
    int64_t dl = 0, dr = 0;
    detail::check(mpsim_gpu_get_site(h_, i, &dl, &dr, nullptr));
    CTensor t({dl, 2, dr});
    detail::check(mpsim_gpu_get_site(h_, i, &dl, &dr, reinterpret_cast<double*>(t.data())));
    return t;
  }
  void set_site(int i, const CTensor& t) {
    if (t.rank() != 3 || t.extent(1) != 2) throw std::invalid_argument("site must be (left, 2, right)");
    detail::check(mpsim_gpu_set_site(h_, i, t.extent(0), t.extent(2), reinterpret_cast<const double*>(t.data())));
  }
  mpsim_gpu_state* handle() const { return h_; }

 private:
  mpsim_gpu_state* h_ = nullptr;
};

inline ApplyReport to_report(const mpsim_report& r) { return ApplyReport{r.discarded_weight, r.new_bond, r.svd_count}; }

inline ApplyReport apply_1q(MpsState& s, const CTensor& u, int q) {  // gate_apply.cpp:99-110
  if (u.rank() != 2 || u.extent(0) != 2 || u.extent(1) != 2) throw std::invalid_argument("gate matrix must be 2x2");
  mpsim_report r{};
  detail::check(mpsim_gpu_apply_1q(s.handle(), reinterpret_cast<const double*>(u.data()), q, &r));
  return to_report(r);
}

inline ApplyReport apply_2q(MpsState& s, const CTensor& u, int q0, int q1, const TruncationPolicy& p, int method) {
  if (u.rank() != 2 || u.extent(0) != 4 || u.extent(1) != 4) throw std::invalid_argument("gate matrix must be 4x4");
  mpsim_policy pol{p.max_bond, p.cutoff};
  mpsim_report r{};
  detail::check(mpsim_gpu_apply_2q(s.handle(), reinterpret_cast<const double*>(u.data()), q0, q1, method, &pol, &r));
  return to_report(r);
}

inline ApplyReport apply_2q_local(MpsState& s, const CTensor& u, int q, const TruncationPolicy& p) {
  if (q < 0 || q + 1 >= s.num_qubits()) throw std::invalid_argument("adjacent pair out of range");
  return apply_2q(s, u, q, q + 1, p, MPSIM_NONLOCAL_SWAP);  // gate_apply.cpp:112-147
}
inline ApplyReport apply_2q_swap(MpsState& s, const CTensor& u, int q0, int q1, const TruncationPolicy& p) {
  return apply_2q(s, u, q0, q1, p, MPSIM_NONLOCAL_SWAP);  // gate_apply.cpp:149-179
}
inline ApplyReport apply_2q_bondprop(MpsState& s, const CTensor& u, int q0, int q1, const TruncationPolicy& p) {
  return apply_2q(s, u, q0, q1, p, MPSIM_NONLOCAL_BONDPROP);  // gate_apply.cpp:181-255
}
inline ApplyReport apply_gate(MpsState& s, const FusedGate& g, const TruncationPolicy& p,
                              NonlocalMethod m = NonlocalMethod::Swap) {  // gate_apply.cpp:257-268
  if (!g.two_qubit()) return apply_1q(s, g.matrix, g.q0);
  return apply_2q(s, g.matrix, g.q0, g.q1, p, m == NonlocalMethod::Swap ? MPSIM_NONLOCAL_SWAP : MPSIM_NONLOCAL_BONDPROP);
}

inline std::vector<mpsim_gate> to_abi(const std::vector<FusedGate>& gates) {
  std::vector<mpsim_gate> out(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) {
    const FusedGate& g = gates[i];
    out[i].q0 = g.q0;
    out[i].q1 = g.two_qubit() ? g.q1 : -1;
    const double* d = reinterpret_cast<const double*>(g.matrix.data());
    for (Index k = 0; k < 2 * g.matrix.size() && k < 32; ++k) out[i].u[k] = d[k];
  }
  return out;
}

// execute_serial (executor.cpp:73-97): layered batched launches, same result.
inline ExecStats execute_serial(MpsState& s, const std::vector<FusedGate>& gates, const TruncationPolicy& p,
                                NonlocalMethod m = NonlocalMethod::Swap) {
  const auto abi = to_abi(gates);
  mpsim_policy pol{p.max_bond, p.cutoff};
  mpsim_exec_stats st{};
  detail::check(mpsim_gpu_execute(s.handle(), abi.data(), static_cast<int32_t>(abi.size()), &pol,
                                  m == NonlocalMethod::Swap ? MPSIM_NONLOCAL_SWAP : MPSIM_NONLOCAL_BONDPROP, &st,
                                  nullptr));
  return ExecStats{st.peak_bond, st.total_discarded_weight, st.layers, st.device_ms};
}

// execute_parallel (executor.cpp:99-232): each layer is one batched launch sequence.
inline ExecStats execute_parallel(MpsState& s, const LayerPlan& plan, const TruncationPolicy& p, int workers) {
  if (workers < 1) throw std::invalid_argument("worker count must be >= 1");
  std::vector<FusedGate> flat;
  for (const auto& layer : plan.layers)
    for (const FusedGate& g : layer) {
      if (!g.local()) throw std::invalid_argument("parallel execution requires a local-gate plan");
      flat.push_back(g);
    }
  return execute_serial(s, flat, p, NonlocalMethod::Swap);
}

inline void move_center(MpsState& s, int c) { detail::check(mpsim_gpu_move_center(s.handle(), c)); }
inline void left_canonicalize(MpsState& s) { move_center(s, s.num_qubits() - 1); }
inline void right_canonicalize(MpsState& s) { move_center(s, 0); }

inline double norm(const MpsState& s) {
  double v = 0.0;
  detail::check(mpsim_gpu_norm(s.handle(), &v));
  return v;
}
inline Complex amplitude(const MpsState& s, std::string_view bits) {
  if (static_cast<int>(bits.size()) != s.num_qubits()) throw std::invalid_argument("bit string length mismatch");
  double out[2];
  detail::check(mpsim_gpu_amplitudes(s.handle(), bits.data(), 1, out));
  return {out[0], out[1]};
}
inline Complex overlap(const MpsState& a, const MpsState& b) {
  double out[2];
  detail::check(mpsim_gpu_overlap(a.handle(), b.handle(), out));
  return {out[0], out[1]};
}
inline std::vector<Complex> to_statevector(const MpsState& s, int max_qubits = 20) {
  const int n = s.num_qubits();
  if (n > max_qubits) throw std::invalid_argument("statevector export capped");
  std::vector<Complex> v(size_t{1} << n);
  detail::check(mpsim_gpu_to_statevector(s.handle(), max_qubits, reinterpret_cast<double*>(v.data())));
  return v;
}

struct ShotResult {  // sampler.hpp:39-43
  std::map<std::string, std::uint64_t> counts;
  std::uint64_t shots = 0;
  std::uint64_t seed = 0;
};
struct SamplerOptions {
  bool memoize = true;
  std::size_t max_cache_entries = 0;
};

class Sampler {  // sampler.hpp:50-86
 public:
  explicit Sampler(const MpsState& s, SamplerOptions o = {}) : n_(s.num_qubits()) {
    detail::check(mpsim_gpu_sampler_create(s.handle(), o.memoize ? 1 : 0, o.max_cache_entries, &h_));
  }
  Sampler(const Sampler&) = delete;
  Sampler& operator=(const Sampler&) = delete;
  ~Sampler() {
    if (h_) mpsim_gpu_sampler_destroy(h_);
  }
  ShotResult sample(std::uint64_t shots, std::uint64_t seed) {
    int32_t unique = 0;
    detail::check(mpsim_gpu_sample(h_, shots, seed, &unique));
    ShotResult r;
    r.shots = shots;
    r.seed = seed;
    std::string bits(static_cast<size_t>(n_), '0');
    for (int i = 0; i < unique; ++i) {
      std::uint64_t c = 0;
      detail::check(mpsim_gpu_sampler_result(h_, i, bits.data(), &c));
      r.counts[bits] = c;
    }
    return r;
  }
  void clear_cache() { detail::check(mpsim_gpu_sampler_clear_cache(h_)); }
  std::size_t cache_size() const {
    uint64_t hits = 0, size = 0;
    detail::check(mpsim_gpu_sampler_stats(h_, &hits, &size));
    return size;
  }
  std::uint64_t cache_hits() const {
    uint64_t hits = 0, size = 0;
    detail::check(mpsim_gpu_sampler_stats(h_, &hits, &size));
    return hits;
  }

 private:
  int n_;
  mpsim_gpu_sampler* h_ = nullptr;
};

inline ShotResult sample(const MpsState& s, std::uint64_t shots, std::uint64_t seed, SamplerOptions o = {}) {
  Sampler sp(s, o);
  return sp.sample(shots, seed);
}

// ---- multi-GPU chains (no reference counterpart: the reference is one
// process; this replaces execute_parallel's worker pool across GPUs). One
// process per GPU; rank 0 draws the NCCL id (nccl_unique_id) and the caller
// hands it to the other ranks out of band, as with ncclCommInitRank. Every
// rank issues the same calls in the same order; results are those of one GPU
// bit for bit.
using NcclId = std::array<unsigned char, 128>;
inline NcclId nccl_unique_id() {
  NcclId id{};
  detail::check(mpsim_gpu_nccl_unique_id(id.data()));
  return id;
}

class ShardedChain {
 public:
  ShardedChain(int n_qubits, Index chi, int rank, int world, const NcclId* id = nullptr, int device = 0)
      : n_(n_qubits) {
    detail::check(mpsim_gpu_shard_create(n_qubits, chi, rank, world, id ? id->data() : nullptr, device, &h_));
    detail::check(mpsim_gpu_shard_info(h_, &lo_, &hi_, nullptr));
  }
  ShardedChain(const ShardedChain&) = delete;
  ShardedChain& operator=(const ShardedChain&) = delete;
  ~ShardedChain() {
    if (h_) mpsim_gpu_shard_destroy(h_);
  }
  int lo() const { return lo_; }  // owned sites [lo, hi)
  int hi() const { return hi_; }
  int num_qubits() const { return n_; }
  void set_site(int i, const CTensor& t) {
    if (t.rank() != 3 || t.extent(1) != 2) throw std::invalid_argument("site must be (left, 2, right)");
    detail::check(mpsim_gpu_shard_set_site(h_, i, t.extent(0), t.extent(2), reinterpret_cast<const double*>(t.data())));
  }
  CTensor site(int i) const {
    int64_t dl = 0, dr = 0;
    detail::check(mpsim_gpu_shard_get_site(h_, i, &dl, &dr, nullptr));
    CTensor t({dl, 2, dr});
    detail::check(mpsim_gpu_shard_get_site(h_, i, &dl, &dr, reinterpret_cast<double*>(t.data())));
    return t;
  }
  std::vector<Index> owned_bond_dims() const {  // bonds lo .. hi
    std::vector<Index> b(static_cast<size_t>(hi_ - lo_) + 1);
    detail::check(mpsim_gpu_shard_bond_dims(h_, b.data()));
    return b;
  }
  // one layer of disjoint local gates (global indices), every rank the same layer
  ExecStats apply_layer(const std::vector<FusedGate>& layer, const TruncationPolicy& p) {
    const auto g = detail_gates(layer);
    const mpsim_policy pol{p.max_bond, p.cutoff};
    mpsim_exec_stats st{};
    detail::check(mpsim_gpu_shard_apply_layer(h_, g.data(), static_cast<int32_t>(g.size()), &pol, &st));
    return ExecStats{st.peak_bond, st.total_discarded_weight, st.layers, st.device_ms};
  }
  // execute_parallel over the chain (non-local gates SWAP-lowered, fusion.cpp:137-190)
  ExecStats execute(const std::vector<FusedGate>& gates, const TruncationPolicy& p) {
    const auto g = detail_gates(gates);
    const mpsim_policy pol{p.max_bond, p.cutoff};
    mpsim_exec_stats st{};
    detail::check(mpsim_gpu_shard_execute(h_, g.data(), static_cast<int32_t>(g.size()), &pol, &st));
    return ExecStats{st.peak_bond, st.total_discarded_weight, st.layers, st.device_ms};
  }
  Complex amplitude(std::string_view bits) {
    if (bits.size() != static_cast<size_t>(n_)) throw std::invalid_argument("bit string length must equal qubit count");
    double out[2];
    detail::check(mpsim_gpu_shard_amplitudes(h_, bits.data(), 1, out));
    return {out[0], out[1]};
  }
  double norm() {
    double v = 0.0;
    detail::check(mpsim_gpu_shard_norm(h_, &v));
    return v;
  }
  Complex expect_1q(const CTensor& op, int q) {
    double out[2];
    detail::check(mpsim_gpu_shard_expect_1q(h_, reinterpret_cast<const double*>(op.data()), q, out));
    return {out[0], out[1]};
  }
  void move_center(int c) { detail::check(mpsim_gpu_shard_move_center(h_, c)); }
  ShotResult sample(std::uint64_t shots, std::uint64_t seed, std::uint64_t chunk = 4096) {
    int32_t unique = 0;
    detail::check(mpsim_gpu_shard_sample(h_, shots, seed, chunk, &unique));
    ShotResult r;
    r.shots = shots;
    r.seed = seed;
    std::string bits(static_cast<size_t>(n_), '0');
    for (int i = 0; i < unique; ++i) {
      std::uint64_t c = 0;
      detail::check(mpsim_gpu_shard_sample_result(h_, i, bits.data(), &c));
      r.counts[bits] = c;
    }
    return r;
  }
  double max_over_ranks(double x) {
    detail::check(mpsim_gpu_shard_allreduce(h_, &x, 1, MPSIM_REDUCE_MAX));
    return x;
  }
  void barrier() { detail::check(mpsim_gpu_shard_barrier(h_)); }
  mpsim_gpu_shard* handle() const { return h_; }

 private:
  static std::vector<mpsim_gate> detail_gates(const std::vector<FusedGate>& gates);
  int n_;
  int32_t lo_ = 0, hi_ = 0;
  mpsim_gpu_shard* h_ = nullptr;
};
inline std::vector<mpsim_gate> ShardedChain::detail_gates(const std::vector<FusedGate>& gates) {
  return to_abi(gates);
}

// ---- host front end (circuit.hpp, runner.hpp, generators.hpp) -------------
// Differences, by design: parse_qasm + fuse_circuit are one call (fuse_qasm)
// over the library's own parser; run_circuit returns the JSON record text of
// run_output_to_json (docs/run_output.schema.json) instead of a RunOutput
// struct plus nlohmann::json.

// parse_qasm + inject_sidecar + fuse_circuit (qasm_parser.cpp, runner.cpp:168-190, fusion.cpp:79-135)
inline std::vector<FusedGate> fuse_qasm(const std::string& qasm, const std::string& sidecar_json = {},
                                        int* n_qubits = nullptr) {
  int32_t n = 0, count = 0;
  mpsim_gate* g = nullptr;
  int32_t* fl = nullptr;
  detail::check_config(mpsim_fuse_qasm(qasm.c_str(), sidecar_json.empty() ? nullptr : sidecar_json.c_str(), &n, &g,
                                       &fl, &count));
  std::vector<FusedGate> out(static_cast<size_t>(count));
  for (int32_t i = 0; i < count; ++i) {
    FusedGate& f = out[static_cast<size_t>(i)];
    f.q0 = g[i].q0;
    f.q1 = g[i].q1;
    f.flipped = fl[i] != 0;
    const Index dim = f.q1 >= 0 ? 4 : 2;
    std::vector<Complex> m(static_cast<size_t>(dim * dim));
    for (Index e = 0; e < dim * dim; ++e) m[static_cast<size_t>(e)] = Complex(g[i].u[2 * e], g[i].u[2 * e + 1]);
    f.matrix = CTensor({dim, dim}, std::move(m));
  }
  mpsim_free(g);
  mpsim_free(fl);
  if (n_qubits) *n_qubits = n;
  return out;
}

// layerize(decompose_nonlocal(gates, n)) (fusion.cpp:137-190)
inline LayerPlan plan_layers(const std::vector<FusedGate>& gates, int n_qubits) {
  const auto abi = to_abi(gates);
  mpsim_gate* g = nullptr;
  int32_t* lo = nullptr;
  int32_t count = 0, nl = 0;
  detail::check(mpsim_plan_layers(abi.data(), static_cast<int32_t>(abi.size()), n_qubits, &g, &lo, &count, &nl));
  LayerPlan plan;
  plan.layers.resize(static_cast<size_t>(nl));
  for (int32_t i = 0; i < count; ++i) {
    FusedGate f;
    f.q0 = g[i].q0;
    f.q1 = g[i].q1;
    const Index dim = f.q1 >= 0 ? 4 : 2;
    std::vector<Complex> m(static_cast<size_t>(dim * dim));
    for (Index e = 0; e < dim * dim; ++e) m[static_cast<size_t>(e)] = Complex(g[i].u[2 * e], g[i].u[2 * e + 1]);
    f.matrix = CTensor({dim, dim}, std::move(m));
    plan.layers[static_cast<size_t>(lo[i])].push_back(std::move(f));
  }
  mpsim_free(g);
  mpsim_free(lo);
  return plan;
}

namespace detail {
inline std::string take(char* p) {
  std::string s = p ? p : "";
  mpsim_free(p);
  return s;
}
}  // namespace detail

inline std::string ghz_qasm(int n_qubits, bool measure = false) {  // generators.cpp:52-71
  char* q = nullptr;
  detail::check_config(mpsim_gen_ghz_qasm(n_qubits, measure ? 1 : 0, &q));
  return detail::take(q);
}

enum class Entangler { Cx, Haar };  // generators.hpp:40
struct BrickworkOptions {           // generators.hpp:42-48
  int n_qubits = 0;
  int depth = 0;
  std::uint64_t seed = 1;
  bool measure = false;
  Entangler entangler = Entangler::Cx;
};
struct GeneratedCircuit {  // generators.hpp:59-62 (sidecar as u4-sidecar-v1 JSON text; empty for cx)
  std::string qasm;
  std::string sidecar_json;
};
inline GeneratedCircuit brickwork_qasm(const BrickworkOptions& o) {  // generators.cpp:95-145
  char *q = nullptr, *sc = nullptr;
  detail::check_config(mpsim_gen_brickwork_qasm(o.n_qubits, o.depth, o.seed, o.measure ? 1 : 0,
                                                o.entangler == Entangler::Haar ? 1 : 0, &q, &sc));
  return GeneratedCircuit{detail::take(q), detail::take(sc)};
}

enum class Backend { MpsSerial, MpsParallel, Statevector };  // runner.hpp:38

struct RunConfig {  // runner.hpp:46-62
  std::string qasm_path, qasm_text, sidecar_path, sidecar_json, input_label;
  Backend backend = Backend::MpsSerial;
  NonlocalMethod nonlocal = NonlocalMethod::Swap;
  Index max_bond = 0;  // 0 = unbounded
  double cutoff = 0.0;
  std::uint64_t shots = 0, seed = 1;
  int workers = 1;
  bool memoize = true;
  std::size_t cache_cap = 0;
  int statevector_cap = 20;
  int device = 0;
};

// run_circuit + run_output_to_json (runner.cpp:219-328): the JSON record text
inline std::string run_circuit_json(const RunConfig& c) {
  mpsim_run_config k;
  mpsim_run_config_defaults(&k);
  auto cs = [](const std::string& s) { return s.empty() ? nullptr : s.c_str(); };
  k.qasm_path = cs(c.qasm_path);
  k.qasm_text = cs(c.qasm_text);
  k.sidecar_path = cs(c.sidecar_path);
  k.sidecar_json = cs(c.sidecar_json);
  k.input_label = cs(c.input_label);
  k.backend = static_cast<int32_t>(c.backend);
  k.nonlocal = c.nonlocal == NonlocalMethod::Swap ? MPSIM_NONLOCAL_SWAP : MPSIM_NONLOCAL_BONDPROP;
  k.max_bond = c.max_bond;
  k.cutoff = c.cutoff;
  k.shots = c.shots;
  k.seed = c.seed;
  k.workers = c.workers;
  k.memoize = c.memoize ? 1 : 0;
  k.cache_cap = c.cache_cap;
  k.statevector_cap = c.statevector_cap;
  k.device = c.device;
  char* json = nullptr;
  detail::check_config(mpsim_gpu_run_circuit(&k, &json));
  return detail::take(json);
}

// exit_code_for_error (runner.cpp:330-341)
inline int exit_code_for_error(const std::exception& e) {
  if (dynamic_cast<const ParseError*>(&e)) return 2;
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const NumericError*>(&e)) return 3;
  return 1;
}

}  // namespace mpsim
