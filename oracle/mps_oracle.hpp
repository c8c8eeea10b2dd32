// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU oracle: a from-scratch, Eigen-free restatement of the reference mpsim
// MPS gate-application path (arXiv 2601.04422 TN-Sim, /root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it, and only as the checker or the timed
// CPU baseline. The product (paper_2601_04422_b200/) never links it.
//
// Third-party arithmetic boundary: the reference calls Eigen3 (>= 3.3,
// un-vendored, absent from /root/reference and from this image) for GEMM
// (tensor.hpp:326-329), BDCSVD (svd.hpp:95) and HouseholderQR (mps.cpp:59,
// generators.cpp:81). This restatement replaces them with LAPACK zgesdd
// (divide-and-conquer SVD, the same algorithm family as BDCSVD), zgeqrf +
// zungqr (Householder QR) and zgemm from the OpenBLAS that ships with scipy
// in this image. Results agree with Eigen to rounding, not bit-for-bit:
// parity is pinned at the property/known-answer level of the reference's own
// tests (see tests/test_oracle_*.py) plus the independent dense statevector
// restatement below.
#pragma once

#include <atomic>
#include <array>
#include <complex>
#include <cstdint>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace oracle {

using Index = std::int64_t;
using cplx = std::complex<double>;
inline constexpr Index kUnbounded = INT64_MAX;

struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Row-major dense matrix helper (rows x cols), last index fastest, as in
// tensor.hpp:17-18.
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<cplx> a;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), a(static_cast<size_t>(r * c)) {}
  cplx& operator()(Index r, Index c) { return a[static_cast<size_t>(r * cols + c)]; }
  const cplx& operator()(Index r, Index c) const { return a[static_cast<size_t>(r * cols + c)]; }
};

// C = op(A) * op(B) through zgemm; both row-major.
Mat matmul(const Mat& A, const Mat& B, bool conjA = false, bool conjB = false);

// svd.hpp:37-43
struct SvdResult {
  Mat u;                   // m x k
  std::vector<double> s;   // k, descending
  Mat vdag;                // k x n
  double discarded_weight = 0.0;
};

// svd.hpp:48-74 — the truncation rule, restated verbatim in semantics.
Index truncation_rank(const std::vector<double>& s, Index max_rank, double cutoff,
                      double* discarded_weight);

// svd.hpp:79-110
SvdResult svd(const Mat& m, Index max_rank = kUnbounded, double cutoff = 0.0);
extern std::atomic<int> g_svd_backend;  // 0 zgesdd, 1 zgesvj (oracle pinning)

// One MPS site (Dl, 2, Dr), flat index (l*2+p)*Dr + r (tensor.hpp:139-148).
struct Site {
  Index dl = 1, dr = 1;
  std::vector<cplx> a;
  cplx& at(Index l, Index p, Index r) { return a[static_cast<size_t>((l * 2 + p) * dr + r)]; }
  const cplx& at(Index l, Index p, Index r) const { return a[static_cast<size_t>((l * 2 + p) * dr + r)]; }
};

// mps.hpp:33-75
struct MpsState {
  std::vector<Site> sites;
  std::vector<Index> bonds;  // n+1
  int center = -1;           // -1 = unknown
  explicit MpsState(int n);
  int n() const { return static_cast<int>(sites.size()); }
  Index max_bond() const;
  void validate() const;
};

// gate_apply.hpp:35-44
struct Policy {
  Index max_bond = kUnbounded;
  double cutoff = 0.0;
};
struct Report {
  double w = 0.0;
  Index new_bond = 1;
  int svd_count = 0;
};

Report apply_1q(MpsState& s, const Mat& u, int q);                          // gate_apply.cpp:99-110
Report apply_2q_local(MpsState& s, const Mat& u, int q, const Policy& p);   // gate_apply.cpp:112-147
Report apply_2q_swap(MpsState& s, const Mat& u, int q0, int q1, const Policy& p);      // :149-179
Report apply_2q_bondprop(MpsState& s, const Mat& u, int q0, int q1, const Policy& p);  // :181-255

void move_center(MpsState& s, int c);  // mps.cpp:177-187
double norm(const MpsState& s);        // mps.cpp:189-202
cplx amplitude(const MpsState& s, const std::string& bits);  // mps.cpp:204-221
cplx overlap(const MpsState& a, const MpsState& b);          // mps.cpp:223-239
std::vector<cplx> to_statevector(const MpsState& s, int max_qubits = 20);  // mps.cpp:241-256

// Circuit IR (circuit.hpp).
enum class GateKind { H, X, Y, Z, S, Sdg, T, Tdg, Rx, Ry, Rz, U1, U2, U3, Cx, Cz, Swap, U4 };
struct PrimOp {
  GateKind kind = GateKind::H;
  int q0 = 0, q1 = -1;
  std::vector<double> params;
  Mat matrix;  // U4 only
  bool two() const { return q1 >= 0; }
};
struct Circuit {
  int n = 0;
  std::vector<PrimOp> ops;
};
struct FusedGate {
  int q0 = 0, q1 = -1;
  bool flipped = false;
  Mat m;
  bool two() const { return q1 >= 0; }
  bool local() const { return !two() || q1 == q0 + 1; }
  int lo() const { return q0; }
  int hi() const { return two() ? q1 : q0; }
};

int param_count(GateKind k);
Mat gate_matrix_1q(GateKind k, const std::vector<double>& params);  // gates.cpp:119-172
Mat gate_matrix(const PrimOp& op);                                   // gates.cpp:174-208
std::vector<FusedGate> fuse_circuit(const Circuit& c);               // fusion.cpp:79-135
std::vector<FusedGate> decompose_nonlocal(const std::vector<FusedGate>& g, int n);  // fusion.cpp:137-161
std::vector<std::vector<FusedGate>> layerize(const std::vector<FusedGate>& g);      // fusion.cpp:163-190

// Generators (generators.cpp, tests/support/test_util.cpp).
double uniform_unit(std::mt19937_64& e);
double normal_unit(std::mt19937_64& e);
Mat haar_unitary(Index dim, std::uint64_t seed);                                 // generators.cpp:73-93
Circuit ghz_circuit(int n);                                                       // generators.cpp:52-71
Circuit brickwork_circuit(int n, int depth, std::uint64_t seed, bool haar);       // generators.cpp:95-145 (+ runner.cpp:193-217 sidecar injection)
Circuit random_circuit(int n, int gates, std::uint64_t seed, bool nonlocal);     // test_util.cpp:36-75
MpsState random_mps(int n, Index chi, std::uint64_t seed);                        // test_util.cpp:77-119

// Executor (executor.cpp).
struct ExecStats {
  Index peak_bond = 1;
  double total_w = 0.0;
  std::vector<Report> reports;  // per gate, in plan order
  std::uint64_t wall_ns = 0;
};
ExecStats execute_serial(MpsState& s, const std::vector<FusedGate>& g, const Policy& p,
                         bool bondprop);                                              // executor.cpp:73-97
ExecStats execute_parallel(MpsState& s, const std::vector<std::vector<FusedGate>>& layers,
                           const Policy& p, int workers);                             // executor.cpp:99-232

// Sampler (sampler.cpp).
struct Sampler {
  int n = 0;
  std::vector<std::array<Mat, 2>> slices;
  bool memoize = true;
  size_t cap = 0;
  struct Entry {
    std::vector<cplx> env;
    double p0 = -1.0;
  };
  std::unordered_map<std::string, Entry> cache;
  double root_p0 = -1.0;
  std::uint64_t hits = 0;
  Sampler(const MpsState& s, bool memo, size_t cap);
  std::map<std::string, std::uint64_t> sample(std::uint64_t shots, std::uint64_t seed);
  double prob0(const std::vector<cplx>& env, int site) const;
};

// Dense statevector oracle (statevector.cpp).
std::vector<cplx> sv_run(int n, const std::vector<FusedGate>& gates);
std::vector<cplx> sv_run_circuit(const Circuit& c);

}  // namespace oracle
