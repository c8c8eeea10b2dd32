// TEST INFRASTRUCTURE — NOT PRODUCT CODE. See mps_oracle.hpp for the scope
// and the Eigen -> LAPACK substitution. Each function cites the reference
// file:line it restates (paths relative to /root/reference/proj).
#include "mps_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <exception>
#include <mutex>
#include <thread>

extern "C" {
void scipy_zgesdd_(const char* jobz, const int* m, const int* n, oracle::cplx* a, const int* lda,
                   double* s, oracle::cplx* u, const int* ldu, oracle::cplx* vt, const int* ldvt,
                   oracle::cplx* work, const int* lwork, double* rwork, int* iwork, int* info,
                   size_t jobz_len);
void scipy_zgesvd_(const char* jobu, const char* jobvt, const int* m, const int* n, oracle::cplx* a,
                   const int* lda, double* s, oracle::cplx* u, const int* ldu, oracle::cplx* vt,
                   const int* ldvt, oracle::cplx* work, const int* lwork, double* rwork, int* info,
                   size_t, size_t);
void scipy_zgeqrf_(const int* m, const int* n, oracle::cplx* a, const int* lda, oracle::cplx* tau,
                   oracle::cplx* work, const int* lwork, int* info);
void scipy_zungqr_(const int* m, const int* n, const int* k, oracle::cplx* a, const int* lda,
                   const oracle::cplx* tau, oracle::cplx* work, const int* lwork, int* info);
void scipy_cblas_zgemm(int order, int ta, int tb, int m, int n, int k, const void* alpha,
                       const void* a, int lda, const void* b, int ldb, const void* beta, void* c,
                       int ldc);
void scipy_openblas_set_num_threads(int);
void scipy_zgesvj_(const char* joba, const char* jobu, const char* jobv, const int* m, const int* n,
                   oracle::cplx* a, const int* lda, double* sva, const int* mv, oracle::cplx* v, const int* ldv,
                   oracle::cplx* cwork, const int* lwork, double* rwork, const int* lrwork, int* info, size_t,
                   size_t, size_t);
}

namespace oracle {

namespace {

constexpr int kRowMajor = 101, kNoTrans = 111, kConjTrans = 113;

struct BlasInit {
  // One thread per LAPACK call: parallelism comes from the executor's workers,
  // as in the reference (executor.cpp:213-220, single-threaded Eigen per gate).
  BlasInit() { scipy_openblas_set_num_threads(1); }
};
BlasInit g_blas_init;

// Column-major copy for LAPACK.
std::vector<cplx> to_colmajor(const Mat& m) {
  std::vector<cplx> c(m.a.size());
  for (Index r = 0; r < m.rows; ++r)
    for (Index k = 0; k < m.cols; ++k) c[static_cast<size_t>(k * m.rows + r)] = m(r, k);
  return c;
}

Mat transpose_conj(const Mat& m) {
  Mat t(m.cols, m.rows);
  for (Index r = 0; r < m.rows; ++r)
    for (Index c = 0; c < m.cols; ++c) t(c, r) = std::conj(m(r, c));
  return t;
}

Mat site_left(const Site& s) {  // (2Dl x Dr) view copy, mps.cpp:37-39
  Mat m(s.dl * 2, s.dr);
  m.a = s.a;
  return m;
}
Mat site_right(const Site& s) {  // (Dl x 2Dr), mps.cpp:41-43
  Mat m(s.dl, 2 * s.dr);
  m.a = s.a;
  return m;
}
Mat phys_slice(const Site& s, int p) {  // (Dl x Dr) at fixed p, mps.cpp:30-35
  Mat m(s.dl, s.dr);
  for (Index l = 0; l < s.dl; ++l)
    for (Index r = 0; r < s.dr; ++r) m(l, r) = s.at(l, p, r);
  return m;
}
Site site_from(const Mat& m, Index dl, Index dr) {
  Site s;
  s.dl = dl;
  s.dr = dr;
  s.a = m.a;
  return s;
}

void check_policy(const Policy& p) {  // gate_apply.cpp:26-33
  if (p.max_bond < 1) throw std::invalid_argument("truncation policy needs max_bond >= 1");
  if (p.cutoff < 0.0 || p.cutoff >= 1.0)
    throw std::invalid_argument("truncation cutoff must lie in [0, 1)");
}
void check_matrix(const Mat& u, Index dim) {  // gate_apply.cpp:35-40
  if (u.rows != dim || u.cols != dim)
    throw std::invalid_argument("gate matrix must be " + std::to_string(dim) + "x" +
                                std::to_string(dim));
}
void renormalize_kept(SvdResult& d) {  // gate_apply.cpp:44-51
  if (d.discarded_weight > 0.0) {
    const double scale = 1.0 / std::sqrt(1.0 - d.discarded_weight);
    for (double& s : d.s) s *= scale;
  }
}
Mat scale_rows(const std::vector<double>& s, const Mat& vdag) {  // gate_apply.cpp:54-64
  Mat out(vdag.rows, vdag.cols);
  for (Index i = 0; i < vdag.rows; ++i)
    for (Index j = 0; j < vdag.cols; ++j) out(i, j) = s[static_cast<size_t>(i)] * vdag(i, j);
  return out;
}
void update_center(MpsState& s, int lo, int hi) {  // gate_apply.cpp:70-77
  if (s.center < 0) return;
  s.center = (s.center >= lo && s.center <= hi) ? hi : -1;
}
Mat swap_matrix() {  // gate_apply.cpp:79-84
  Mat m(4, 4);
  m(0, 0) = m(1, 2) = m(2, 1) = m(3, 3) = 1.0;
  return m;
}
Mat swap_conjugate4(const Mat& m) {  // gate_apply.cpp:86-95, gates.cpp:37-46
  auto rev = [](Index x) { return ((x & 1) << 1) | (x >> 1); };
  Mat out(4, 4);
  for (Index r = 0; r < 4; ++r)
    for (Index c = 0; c < 4; ++c) out(r, c) = m(rev(r), rev(c));
  return out;
}

// Householder thin QR (mps.cpp:57-65): q (rows x k), r (k x cols), k = min.
void thin_qr(const Mat& m, Mat& q, Mat& r) {
  const int rows = static_cast<int>(m.rows), cols = static_cast<int>(m.cols);
  const int k = std::min(rows, cols);
  std::vector<cplx> a = to_colmajor(m);
  std::vector<cplx> tau(static_cast<size_t>(std::max(1, k)));
  int info = 0, lwork = -1;
  cplx wq;
  scipy_zgeqrf_(&rows, &cols, a.data(), &rows, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq.real()));
  std::vector<cplx> work(static_cast<size_t>(lwork));
  scipy_zgeqrf_(&rows, &cols, a.data(), &rows, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw NumericError("zgeqrf failed");
  r = Mat(k, cols);
  for (int i = 0; i < k; ++i)
    for (int j = i; j < cols; ++j) r(i, j) = a[static_cast<size_t>(j * rows + i)];
  lwork = -1;
  scipy_zungqr_(&rows, &k, &k, a.data(), &rows, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq.real()));
  work.assign(static_cast<size_t>(lwork), cplx{});
  scipy_zungqr_(&rows, &k, &k, a.data(), &rows, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw NumericError("zungqr failed");
  q = Mat(rows, k);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < k; ++j) q(i, j) = a[static_cast<size_t>(j * rows + i)];
}

}  // namespace

Mat matmul(const Mat& A, const Mat& B, bool conjA, bool conjB) {
  const Index m = conjA ? A.cols : A.rows;
  const Index k = conjA ? A.rows : A.cols;
  const Index kb = conjB ? B.cols : B.rows;
  const Index n = conjB ? B.rows : B.cols;
  if (k != kb) throw std::invalid_argument("matmul: inner dimension mismatch");
  Mat C(m, n);
  if (m == 0 || n == 0) return C;
  if (k == 0) return C;
  const cplx one(1.0, 0.0), zero(0.0, 0.0);
  scipy_cblas_zgemm(kRowMajor, conjA ? kConjTrans : kNoTrans, conjB ? kConjTrans : kNoTrans,
                    static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), &one, A.a.data(),
                    static_cast<int>(A.cols), B.a.data(), static_cast<int>(B.cols), &zero, C.a.data(),
                    static_cast<int>(n));
  return C;
}

// svd.hpp:48-74
Index truncation_rank(const std::vector<double>& s, Index max_rank, double cutoff,
                      double* discarded_weight) {
  const Index full = static_cast<Index>(s.size());
  double total = 0.0;
  for (Index i = 0; i < full; ++i) total += s[i] * s[i];
  Index keep = full;
  if (total > 0.0) {
    double tail = 0.0;
    while (keep > 1 && tail + s[keep - 1] * s[keep - 1] <= cutoff * total) {
      tail += s[keep - 1] * s[keep - 1];
      --keep;
    }
  } else {
    keep = 1;
  }
  keep = std::min(keep, std::max<Index>(1, max_rank));
  if (discarded_weight != nullptr) {
    double dropped = 0.0;
    for (Index i = keep; i < full; ++i) dropped += s[i] * s[i];
    *discarded_weight = total > 0.0 ? dropped / total : 0.0;
  }
  return keep;
}

// Second, independent SVD for pinning the oracle (tests/golden/make_golden.py):
// LAPACK zgesvj, one-sided Jacobi (de Rijk pivoting, Drmac-Veselic) — an
// algorithm family unrelated to zgesdd's bidiagonal divide and conquer.
// zgesvj needs rows >= cols; wider matrices go through their adjoint.
std::atomic<int> g_svd_backend{0};

namespace {
SvdResult svd_jacobi(const Mat& m, Index max_rank, double cutoff) {
  const bool tr = m.rows < m.cols;
  const int rows = static_cast<int>(tr ? m.cols : m.rows), cols = static_cast<int>(tr ? m.rows : m.cols);
  std::vector<cplx> a(static_cast<size_t>(rows) * cols);  // column-major rows x cols
  for (Index i = 0; i < m.rows; ++i)
    for (Index j = 0; j < m.cols; ++j) {
      if (tr) a[static_cast<size_t>(i * rows + j)] = std::conj(m(i, j));
      else a[static_cast<size_t>(j * rows + i)] = m(i, j);
    }
  std::vector<double> sva(static_cast<size_t>(cols));
  std::vector<cplx> v(static_cast<size_t>(cols) * cols);
  const int lwork = rows + cols, lrwork = std::max(6, cols);
  std::vector<cplx> cwork(static_cast<size_t>(lwork));
  std::vector<double> rwork(static_cast<size_t>(lrwork));
  int info = 0, mv = 0;
  const char ja = 'G', ju = 'U', jv = 'V';
  scipy_zgesvj_(&ja, &ju, &jv, &rows, &cols, a.data(), &rows, sva.data(), &mv, v.data(), &cols, cwork.data(),
                &lwork, rwork.data(), &lrwork, &info, 1, 1, 1);
  if (info != 0)
    throw NumericError("zgesvj did not converge for (" + std::to_string(rows) + "," + std::to_string(cols) +
                       ") matrix");
  const double scale = rwork[0];
  std::vector<double> s(static_cast<size_t>(cols));
  for (int i = 0; i < cols; ++i) s[static_cast<size_t>(i)] = sva[static_cast<size_t>(i)] * scale;
  SvdResult r;
  const Index keep = truncation_rank(s, max_rank, cutoff, &r.discarded_weight);
  // A = Ua S V^H (column-major Ua in a); for the adjoint case m = V S Ua^H.
  r.u = Mat(m.rows, keep);
  r.vdag = Mat(keep, m.cols);
  for (Index j = 0; j < keep; ++j) {
    for (Index i = 0; i < m.rows; ++i)
      r.u(i, j) = tr ? v[static_cast<size_t>(j * cols + i)] : a[static_cast<size_t>(j * rows + i)];
    for (Index i = 0; i < m.cols; ++i)
      r.vdag(j, i) = tr ? std::conj(a[static_cast<size_t>(j * rows + i)])
                        : std::conj(v[static_cast<size_t>(j * cols + i)]);
  }
  r.s.assign(s.begin(), s.begin() + keep);
  return r;
}
}  // namespace

// svd.hpp:79-110, with Eigen::BDCSVD replaced by LAPACK zgesdd (thin U, V).
SvdResult svd(const Mat& m, Index max_rank, double cutoff) {
  if (max_rank < 1) throw std::invalid_argument("svd max_rank must be >= 1");
  if (cutoff < 0.0 || cutoff >= 1.0) throw std::invalid_argument("svd cutoff must lie in [0, 1)");
  const int backend = g_svd_backend.load(std::memory_order_relaxed);
  if (backend == 1) return svd_jacobi(m, max_rank, cutoff);
  const int rows = static_cast<int>(m.rows), cols = static_cast<int>(m.cols);
  const int mn = std::min(rows, cols), mx = std::max(rows, cols);
  std::vector<cplx> a = to_colmajor(m);
  std::vector<double> s(static_cast<size_t>(mn));
  std::vector<cplx> u(static_cast<size_t>(rows) * mn), vt(static_cast<size_t>(mn) * cols);
  const size_t lrwork = std::max<size_t>(static_cast<size_t>(5) * mn * mn + 5 * mn,
                                         static_cast<size_t>(2) * mx * mn + 2 * mn * mn + mn) + 16;
  std::vector<double> rwork(lrwork);
  std::vector<int> iwork(static_cast<size_t>(8) * mn + 8);
  int info = 0, lwork = -1;
  cplx wq;
  const char jobz = 'S';
  std::vector<cplx> a_copy = a;
  std::vector<cplx> work;
  if (backend == 2) {
    info = 1;  // zgesvd (bidiagonal QR iteration) below, the spread check of make_golden.py
  } else {
    scipy_zgesdd_(&jobz, &rows, &cols, a.data(), &rows, s.data(), u.data(), &rows, vt.data(), &mn, &wq,
                  &lwork, rwork.data(), iwork.data(), &info, 1);
    lwork = std::max(1, static_cast<int>(wq.real()));
    work.resize(static_cast<size_t>(lwork));
    scipy_zgesdd_(&jobz, &rows, &cols, a.data(), &rows, s.data(), u.data(), &rows, vt.data(), &mn,
                  work.data(), &lwork, rwork.data(), iwork.data(), &info, 1);
  }
  if (info > 0) {
    // Divide-and-conquer did not converge: retry with QR-iteration zgesvd
    // before reporting failure (svd.hpp:96-99 throws NumericError).
    a = a_copy;
    const char js = 'S';
    lwork = -1;
    std::vector<double> rw(static_cast<size_t>(5) * mn + 16);
    scipy_zgesvd_(&js, &js, &rows, &cols, a.data(), &rows, s.data(), u.data(), &rows, vt.data(), &mn,
                  &wq, &lwork, rw.data(), &info, 1, 1);
    lwork = std::max(1, static_cast<int>(wq.real()));
    work.assign(static_cast<size_t>(lwork), cplx{});
    scipy_zgesvd_(&js, &js, &rows, &cols, a.data(), &rows, s.data(), u.data(), &rows, vt.data(), &mn,
                  work.data(), &lwork, rw.data(), &info, 1, 1);
  }
  if (info != 0)
    throw NumericError("singular value decomposition did not converge for (" +
                       std::to_string(rows) + "," + std::to_string(cols) + ") matrix");
  SvdResult r;
  const Index keep = truncation_rank(s, max_rank, cutoff, &r.discarded_weight);
  r.u = Mat(rows, keep);
  for (Index i = 0; i < rows; ++i)
    for (Index j = 0; j < keep; ++j) r.u(i, j) = u[static_cast<size_t>(j * rows + i)];
  r.vdag = Mat(keep, cols);
  for (Index i = 0; i < keep; ++i)
    for (Index j = 0; j < cols; ++j) r.vdag(i, j) = vt[static_cast<size_t>(j * mn + i)];
  r.s.assign(s.begin(), s.begin() + keep);
  return r;
}

// mps.cpp:99-110
MpsState::MpsState(int n) {
  if (n < 1) throw std::invalid_argument("state needs at least one qubit");
  sites.resize(static_cast<size_t>(n));
  for (auto& s : sites) {
    s.dl = s.dr = 1;
    s.a.assign(2, cplx{});
    s.a[0] = 1.0;
  }
  bonds.assign(static_cast<size_t>(n) + 1, 1);
}

Index MpsState::max_bond() const { return *std::max_element(bonds.begin(), bonds.end()); }

// mps.cpp:150-169
void MpsState::validate() const {
  const int nn = n();
  if (bonds.size() != static_cast<size_t>(nn) + 1) throw std::logic_error("bond bookkeeping has wrong length");
  if (bonds.front() != 1 || bonds.back() != 1) throw std::logic_error("boundary bonds must have dimension 1");
  for (int i = 0; i < nn; ++i) {
    const Site& t = sites[static_cast<size_t>(i)];
    if (static_cast<Index>(t.a.size()) != t.dl * 2 * t.dr)
      throw std::logic_error("site " + std::to_string(i) + " is not a (left, 2, right) tensor");
    if (t.dl != bonds[static_cast<size_t>(i)] || t.dr != bonds[static_cast<size_t>(i) + 1])
      throw std::logic_error("site " + std::to_string(i) + " disagrees with recorded bond dimensions");
  }
}

// gate_apply.cpp:99-110: A'[l,p',r] = sum_p u[p',p] A[l,p,r].
Report apply_1q(MpsState& s, const Mat& u, int q) {
  check_matrix(u, 2);
  if (q < 0 || q >= s.n()) throw std::invalid_argument("qubit " + std::to_string(q) + " out of range");
  Site& t = s.sites[static_cast<size_t>(q)];
  for (Index l = 0; l < t.dl; ++l)
    for (Index r = 0; r < t.dr; ++r) {
      const cplx a0 = t.at(l, 0, r), a1 = t.at(l, 1, r);
      t.at(l, 0, r) = u(0, 0) * a0 + u(0, 1) * a1;
      t.at(l, 1, r) = u(1, 0) * a0 + u(1, 1) * a1;
    }
  Report rep;
  rep.new_bond = std::max(s.bonds[static_cast<size_t>(q)], s.bonds[static_cast<size_t>(q) + 1]);
  return rep;
}

// gate_apply.cpp:112-147
Report apply_2q_local(MpsState& s, const Mat& u, int q, const Policy& p) {
  check_matrix(u, 4);
  check_policy(p);
  if (q < 0 || q + 1 >= s.n())
    throw std::invalid_argument("adjacent pair (" + std::to_string(q) + "," + std::to_string(q + 1) +
                                ") out of range");
  Site& A = s.sites[static_cast<size_t>(q)];
  Site& B = s.sites[static_cast<size_t>(q) + 1];
  const Index dl = A.dl, dr = B.dr;
  // merged[(l,p0),(p1,r)] = A[(l,p0), m] * B[m, (p1,r)]  (gate_apply.cpp:126)
  const Mat merged = matmul(site_left(A), site_right(B));
  // theta[(l,p0'),(p1',r)] = sum_{p0,p1} u[2p0'+p1', 2p0+p1] merged  (:127-129)
  Mat theta(dl * 2, 2 * dr);
  for (Index l = 0; l < dl; ++l)
    for (Index r = 0; r < dr; ++r) {
      cplx x[4];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) x[a * 2 + b] = merged(l * 2 + a, b * dr + r);
      for (int o = 0; o < 4; ++o) {
        cplx acc{};
        for (int i = 0; i < 4; ++i) acc += x[i] * u(o, i);
        theta(l * 2 + (o >> 1), (o & 1) * dr + r) = acc;
      }
    }
  SvdResult d = svd(theta, p.max_bond, p.cutoff);  // :130-132
  renormalize_kept(d);                              // :133
  const Index k = static_cast<Index>(d.s.size());
  A = site_from(d.u, dl, k);                                   // :136
  B = site_from(scale_rows(d.s, d.vdag), k, dr);               // :137-138
  s.bonds[static_cast<size_t>(q) + 1] = k;                     // :139
  update_center(s, q, q + 1);                                  // :140
  Report rep;
  rep.w = d.discarded_weight;
  rep.new_bond = k;
  rep.svd_count = 1;
  return rep;
}

// gate_apply.cpp:149-179
Report apply_2q_swap(MpsState& s, const Mat& u, int q0, int q1, const Policy& p) {
  if (q0 == q1) throw std::invalid_argument("two-qubit gate needs two distinct qubits");
  Mat m = u;
  if (q0 > q1) {
    std::swap(q0, q1);
    m = swap_conjugate4(m);
  }
  if (q1 == q0 + 1) return apply_2q_local(s, m, q0, p);
  const Mat sw = swap_matrix();
  Report total;
  auto absorb = [&total](const Report& r) {
    total.w += r.w;
    total.new_bond = std::max(total.new_bond, r.new_bond);
    total.svd_count += r.svd_count;
  };
  for (int i = q0; i < q1 - 1; ++i) absorb(apply_2q_local(s, sw, i, p));
  absorb(apply_2q_local(s, m, q1 - 1, p));
  for (int i = q1 - 2; i >= q0; --i) absorb(apply_2q_local(s, sw, i, p));
  return total;
}

// gate_apply.cpp:181-255
Report apply_2q_bondprop(MpsState& s, const Mat& u, int q0, int q1, const Policy& p) {
  check_matrix(u, 4);
  check_policy(p);
  if (q0 == q1) throw std::invalid_argument("two-qubit gate needs two distinct qubits");
  Mat m = u;
  if (q0 > q1) {
    std::swap(q0, q1);
    m = swap_conjugate4(m);
  }
  if (q0 < 0 || q1 >= s.n())
    throw std::invalid_argument("qubit pair (" + std::to_string(q0) + "," + std::to_string(q1) +
                                ") out of range");
  // split[(p0',p0),(p1',p1)] = u[2p0'+p1', 2p0+p1]  (:200-202)
  Mat split(4, 4);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int c = 0; c < 2; ++c)
        for (int e = 0; e < 2; ++e) split(a * 2 + c, b * 2 + e) = m(a * 2 + b, c * 2 + e);
  SvdResult g = svd(split);  // :203, unbounded, cutoff 0
  const Index prop = static_cast<Index>(g.s.size());
  const Mat& left = g.u;                            // [(p0',p0), kappa]
  const Mat right = scale_rows(g.s, g.vdag);        // [kappa, (p1',p1)]
  Report rep;

  // Open (:210-225): ordered[(l,p0'),(kappa,b)] = sum_p site[l,p,b] left[(p0',p),kappa]
  Site& S0 = s.sites[static_cast<size_t>(q0)];
  const Index dl0 = S0.dl, b0 = S0.dr;
  Mat ordered(dl0 * 2, prop * b0);
  for (Index l = 0; l < dl0; ++l)
    for (int po = 0; po < 2; ++po)
      for (Index kk = 0; kk < prop; ++kk)
        for (Index b = 0; b < b0; ++b) {
          cplx acc{};
          for (int pi = 0; pi < 2; ++pi) acc += S0.at(l, pi, b) * left(po * 2 + pi, kk);
          ordered(l * 2 + po, kk * b0 + b) = acc;
        }
  SvdResult d = svd(ordered, p.max_bond, p.cutoff);
  renormalize_kept(d);
  Index k = static_cast<Index>(d.s.size());
  S0 = site_from(d.u, dl0, k);
  s.bonds[static_cast<size_t>(q0) + 1] = k;
  rep.w += d.discarded_weight;
  rep.new_bond = std::max(rep.new_bond, k);
  ++rep.svd_count;
  Mat carrier = scale_rows(d.s, d.vdag);  // [k, (kappa, b)]
  Index bprev = b0;

  // Push (:227-246)
  for (int site = q0 + 1; site < q1; ++site) {
    Site& T = s.sites[static_cast<size_t>(site)];
    const Index br = T.dr;
    // pulled[k,kappa,p,r] = sum_b carrier[k,kappa,b] T[b,p,r]; arranged [(k,p),(kappa,r)]
    Mat cm(k * prop, bprev);
    cm.a = carrier.a;
    const Mat pulled = matmul(cm, site_right(T));  // [(k,kappa),(p,r)]
    Mat arranged(k * 2, prop * br);
    for (Index a = 0; a < k; ++a)
      for (Index kk = 0; kk < prop; ++kk)
        for (int pp = 0; pp < 2; ++pp)
          for (Index r = 0; r < br; ++r) arranged(a * 2 + pp, kk * br + r) = pulled(a * prop + kk, pp * br + r);
    SvdResult st = svd(arranged, p.max_bond, p.cutoff);
    renormalize_kept(st);
    const Index k2 = static_cast<Index>(st.s.size());
    T = site_from(st.u, k, k2);
    s.bonds[static_cast<size_t>(site) + 1] = k2;
    rep.w += st.discarded_weight;
    rep.new_bond = std::max(rep.new_bond, k2);
    ++rep.svd_count;
    carrier = scale_rows(st.s, st.vdag);
    k = k2;
    bprev = br;
  }

  // Close (:248-253): site[k,p1',r] = sum_{kappa,p1,b} carrier[k,kappa,b] T[b,p1,r] right[kappa,(p1',p1)]
  Site& T = s.sites[static_cast<size_t>(q1)];
  const Index dr1 = T.dr;
  Mat cm(k * prop, bprev);
  cm.a = carrier.a;
  const Mat target = matmul(cm, site_right(T));  // [(k,kappa),(p1,r)]
  Site out;
  out.dl = k;
  out.dr = dr1;
  out.a.assign(static_cast<size_t>(k * 2 * dr1), cplx{});
  for (Index a = 0; a < k; ++a)
    for (int po = 0; po < 2; ++po)
      for (Index r = 0; r < dr1; ++r) {
        cplx acc{};
        for (Index kk = 0; kk < prop; ++kk)
          for (int pi = 0; pi < 2; ++pi) acc += target(a * prop + kk, pi * dr1 + r) * right(kk, po * 2 + pi);
        out.at(a, po, r) = acc;
      }
  T = std::move(out);
  update_center(s, q0, q1);
  return rep;
}

// mps.cpp:69-80
static void sweep_left_of(MpsState& s, int center) {
  for (int i = 0; i < center; ++i) {
    Mat q, r;
    thin_qr(site_left(s.sites[static_cast<size_t>(i)]), q, r);
    const Index dl = s.sites[static_cast<size_t>(i)].dl;
    const Index k = q.cols;
    s.sites[static_cast<size_t>(i)] = site_from(q, dl, k);
    Site& nx = s.sites[static_cast<size_t>(i) + 1];
    const Mat next = matmul(r, site_right(nx));
    nx = site_from(next, k, nx.dr);
    s.bonds[static_cast<size_t>(i) + 1] = k;
  }
}

// mps.cpp:84-95
static void sweep_right_of(MpsState& s, int center) {
  for (int i = s.n() - 1; i > center; --i) {
    Mat q, r;
    thin_qr(transpose_conj(site_right(s.sites[static_cast<size_t>(i)])), q, r);
    const Index dr = s.sites[static_cast<size_t>(i)].dr;
    const Index k = q.cols;
    s.sites[static_cast<size_t>(i)] = site_from(transpose_conj(q), k, dr);
    Site& pv = s.sites[static_cast<size_t>(i) - 1];
    const Mat prev = matmul(site_left(pv), r, false, true);
    pv = site_from(prev, pv.dl, k);
    s.bonds[static_cast<size_t>(i)] = k;
  }
}

// mps.cpp:177-187
void move_center(MpsState& s, int c) {
  if (c < 0 || c >= s.n()) throw std::invalid_argument("center out of range");
  sweep_left_of(s, c);
  sweep_right_of(s, c);
  double nrm2 = 0.0;
  for (const cplx& v : s.sites[static_cast<size_t>(c)].a) nrm2 += std::norm(v);
  if (std::sqrt(nrm2) < 1e-14) throw NumericError("cannot canonicalize a zero-norm state");
  s.center = c;
}

// mps.cpp:189-202
double norm(const MpsState& s) {
  Mat env(1, 1);
  env(0, 0) = 1.0;
  for (const Site& t : s.sites) {
    Mat next(t.dr, t.dr);
    for (int p = 0; p < 2; ++p) {
      const Mat sl = phys_slice(t, p);
      const Mat x = matmul(matmul(sl, env, true, false), sl);
      for (size_t e = 0; e < next.a.size(); ++e) next.a[e] += x.a[e];
    }
    env = std::move(next);
  }
  return std::sqrt(std::max(0.0, env(0, 0).real()));
}

// mps.cpp:204-221
cplx amplitude(const MpsState& s, const std::string& bits) {
  if (static_cast<int>(bits.size()) != s.n())
    throw std::invalid_argument("bit string length " + std::to_string(bits.size()) +
                                " does not match qubit count " + std::to_string(s.n()));
  Mat env(1, 1);
  env(0, 0) = 1.0;
  for (int i = 0; i < s.n(); ++i) {
    const char c = bits[static_cast<size_t>(i)];
    if (c != '0' && c != '1') throw std::invalid_argument("bit string must contain only 0 and 1");
    env = matmul(env, phys_slice(s.sites[static_cast<size_t>(i)], c - '0'));
  }
  return env(0, 0);
}

// mps.cpp:223-239
cplx overlap(const MpsState& a, const MpsState& b) {
  if (a.n() != b.n()) throw std::invalid_argument("overlap requires equal qubit counts");
  Mat env(1, 1);
  env(0, 0) = 1.0;
  for (int i = 0; i < a.n(); ++i) {
    const Site& ta = a.sites[static_cast<size_t>(i)];
    const Site& tb = b.sites[static_cast<size_t>(i)];
    Mat next(ta.dr, tb.dr);
    for (int p = 0; p < 2; ++p) {
      const Mat x = matmul(matmul(phys_slice(ta, p), env, true, false), phys_slice(tb, p));
      for (size_t e = 0; e < next.a.size(); ++e) next.a[e] += x.a[e];
    }
    env = std::move(next);
  }
  return env(0, 0);
}

// mps.cpp:241-256
std::vector<cplx> to_statevector(const MpsState& s, int max_qubits) {
  if (s.n() > max_qubits)
    throw std::invalid_argument("statevector export capped at " + std::to_string(max_qubits) +
                                " qubits, got " + std::to_string(s.n()));
  Mat acc(1, 1);
  acc(0, 0) = 1.0;
  for (const Site& t : s.sites) {
    const Mat grown = matmul(acc, site_right(t));
    acc = Mat(grown.rows * 2, t.dr);
    acc.a = grown.a;
  }
  return acc.a;
}

// ---------------------------------------------------------------- circuits

int param_count(GateKind k) {  // gates.cpp:68-82
  switch (k) {
    case GateKind::Rx: case GateKind::Ry: case GateKind::Rz: case GateKind::U1: return 1;
    case GateKind::U2: return 2;
    case GateKind::U3: return 3;
    default: return 0;
  }
}

static Mat mat2(cplx a, cplx b, cplx c, cplx d) {
  Mat m(2, 2);
  m.a = {a, b, c, d};
  return m;
}

// gates.cpp:119-172
Mat gate_matrix_1q(GateKind kind, const std::vector<double>& params) {
  const cplx I(0.0, 1.0);
  const double h2 = 1.0 / std::sqrt(2.0);
  switch (kind) {
    case GateKind::H: return mat2(h2, h2, h2, -h2);
    case GateKind::X: return mat2(0, 1, 1, 0);
    case GateKind::Y: return mat2(0, -I, I, 0);
    case GateKind::Z: return mat2(1, 0, 0, -1);
    case GateKind::S: return mat2(1, 0, 0, I);
    case GateKind::Sdg: return mat2(1, 0, 0, -I);
    case GateKind::T: return mat2(1, 0, 0, std::exp(I * (M_PI / 4.0)));
    case GateKind::Tdg: return mat2(1, 0, 0, std::exp(-I * (M_PI / 4.0)));
    case GateKind::Rx: {
      const double h = params.at(0) / 2.0;
      return mat2(std::cos(h), -I * std::sin(h), -I * std::sin(h), std::cos(h));
    }
    case GateKind::Ry: {
      const double h = params.at(0) / 2.0;
      return mat2(std::cos(h), -std::sin(h), std::sin(h), std::cos(h));
    }
    case GateKind::Rz: {
      const double h = params.at(0) / 2.0;
      return mat2(std::exp(-I * h), 0, 0, std::exp(I * h));
    }
    case GateKind::U1: return mat2(1, 0, 0, std::exp(I * params.at(0)));
    case GateKind::U2: {
      const double phi = params.at(0), lam = params.at(1);
      return mat2(h2, -std::exp(I * lam) * h2, std::exp(I * phi) * h2, std::exp(I * (phi + lam)) * h2);
    }
    case GateKind::U3: {
      const double half = params.at(0) / 2.0, phi = params.at(1), lam = params.at(2);
      return mat2(std::cos(half), -std::exp(I * lam) * std::sin(half), std::exp(I * phi) * std::sin(half),
                  std::exp(I * (phi + lam)) * std::cos(half));
    }
    default: throw std::invalid_argument("not a one-qubit gate");
  }
}

// gates.cpp:174-208
Mat gate_matrix(const PrimOp& op) {
  if (!op.two()) return gate_matrix_1q(op.kind, op.params);
  Mat m(4, 4);
  switch (op.kind) {
    case GateKind::Cx: m(0, 0) = m(1, 1) = m(2, 3) = m(3, 2) = 1.0; break;
    case GateKind::Cz: m(0, 0) = m(1, 1) = m(2, 2) = 1.0; m(3, 3) = -1.0; break;
    case GateKind::Swap: m(0, 0) = m(1, 2) = m(2, 1) = m(3, 3) = 1.0; break;
    case GateKind::U4: m = op.matrix; break;
    default: throw std::invalid_argument("not a two-qubit gate");
  }
  return op.q0 < op.q1 ? m : swap_conjugate4(m);
}

namespace {

bool touches(const FusedGate& g, int q) { return g.q0 == q || (g.two() && g.q1 == q); }
bool shares_qubit(const FusedGate& a, const FusedGate& b) {
  return touches(a, b.q0) || (b.two() && touches(a, b.q1));
}

// fusion.cpp:38-52
Mat embed_1q(const Mat& g, bool at_low) {
  Mat out(4, 4);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int c = 0; c < 2; ++c)
        for (int d = 0; d < 2; ++d)
          out((a << 1) | b, (c << 1) | d) =
              at_low ? g(a, c) * cplx(b == d ? 1.0 : 0.0) : g(b, d) * cplx(a == c ? 1.0 : 0.0);
  return out;
}

FusedGate make_block(const PrimOp& op) {  // fusion.cpp:54-67
  FusedGate g;
  if (op.two()) {
    g.q0 = std::min(op.q0, op.q1);
    g.q1 = std::max(op.q0, op.q1);
    g.flipped = op.q0 > op.q1;
    g.m = gate_matrix(op);
  } else {
    g.q0 = op.q0;
    g.q1 = -1;
    g.m = gate_matrix_1q(op.kind, op.params);
  }
  return g;
}

FusedGate swap_block(int q) {  // fusion.cpp:69-75
  PrimOp op;
  op.kind = GateKind::Swap;
  op.q0 = q;
  op.q1 = q + 1;
  return make_block(op);
}

}  // namespace

// fusion.cpp:79-135
std::vector<FusedGate> fuse_circuit(const Circuit& c) {
  std::vector<FusedGate> blocks;
  for (const PrimOp& op : c.ops) {
    FusedGate cur = make_block(op);
    for (;;) {
      int j = -1;
      for (int k = static_cast<int>(blocks.size()) - 1; k >= 0; --k)
        if (shares_qubit(blocks[static_cast<size_t>(k)], cur)) {
          j = k;
          break;
        }
      if (j < 0) {
        blocks.push_back(std::move(cur));
        break;
      }
      FusedGate& prev = blocks[static_cast<size_t>(j)];
      if (prev.q0 == cur.q0 && prev.q1 == cur.q1) {
        cur.m = matmul(cur.m, prev.m);
        blocks.erase(blocks.begin() + j);
        continue;
      }
      if (!prev.two() && cur.two()) {
        cur.m = matmul(cur.m, embed_1q(prev.m, prev.q0 == cur.q0));
        blocks.erase(blocks.begin() + j);
        continue;
      }
      if (!cur.two() && prev.two()) {
        const int other = prev.q0 == cur.q0 ? prev.q1 : prev.q0;
        bool quiet = true;
        for (size_t k = static_cast<size_t>(j) + 1; k < blocks.size(); ++k)
          quiet = quiet && !touches(blocks[k], other);
        if (quiet) {
          prev.m = matmul(embed_1q(cur.m, cur.q0 == prev.q0), prev.m);
          break;
        }
        blocks.push_back(std::move(cur));
        break;
      }
      blocks.push_back(std::move(cur));
      break;
    }
  }
  return blocks;
}

// fusion.cpp:137-161
std::vector<FusedGate> decompose_nonlocal(const std::vector<FusedGate>& gates, int n) {
  std::vector<FusedGate> out;
  for (const FusedGate& g : gates) {
    if (g.two() && (g.q0 < 0 || g.q1 >= n)) throw std::invalid_argument("gate qubits out of range");
    if (g.local()) {
      out.push_back(g);
      continue;
    }
    for (int i = g.q0; i < g.q1 - 1; ++i) out.push_back(swap_block(i));
    FusedGate local = g;
    local.q0 = g.q1 - 1;
    out.push_back(std::move(local));
    for (int i = g.q1 - 2; i >= g.q0; --i) out.push_back(swap_block(i));
  }
  return out;
}

// fusion.cpp:163-190
std::vector<std::vector<FusedGate>> layerize(const std::vector<FusedGate>& gates) {
  int n = 0;
  for (const FusedGate& g : gates) {
    if (!g.local()) throw std::invalid_argument("layerize requires local gates");
    n = std::max(n, g.hi() + 1);
  }
  std::vector<std::vector<FusedGate>> plan;
  std::vector<int> last(static_cast<size_t>(n), -1);
  for (const FusedGate& g : gates) {
    int layer = 0;
    for (int q = g.lo(); q <= g.hi(); ++q) layer = std::max(layer, last[static_cast<size_t>(q)] + 1);
    if (static_cast<size_t>(layer) >= plan.size()) plan.resize(static_cast<size_t>(layer) + 1);
    plan[static_cast<size_t>(layer)].push_back(g);
    for (int q = g.lo(); q <= g.hi(); ++q) last[static_cast<size_t>(q)] = layer;
  }
  return plan;
}

// ---------------------------------------------------------------- generators

double uniform_unit(std::mt19937_64& e) {  // generators.cpp:31-33
  return static_cast<double>(e() >> 11) * 0x1.0p-53;
}

double normal_unit(std::mt19937_64& e) {  // generators.cpp:35-42
  double u1 = uniform_unit(e);
  while (u1 <= 0.0) u1 = uniform_unit(e);
  const double u2 = uniform_unit(e);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// generators.cpp:73-93: QR of a complex Gaussian matrix with the R-diagonal
// phase fix; the fixed Q is unique, so LAPACK's Householder conventions give
// the same matrix as Eigen's to rounding.
Mat haar_unitary(Index dim, std::uint64_t seed) {
  std::mt19937_64 e(seed);
  Mat g(dim, dim);
  for (Index r = 0; r < dim; ++r)
    for (Index c = 0; c < dim; ++c) {
      // The reference writes Complex(normal_unit(engine), normal_unit(engine));
      // g++ (the reference's toolchain here) evaluates constructor arguments
      // right to left, so the imaginary part is drawn first.
      const double im = normal_unit(e);
      const double re = normal_unit(e);
      g(r, c) = cplx(re, im);
    }
  Mat q, r;
  thin_qr(g, q, r);
  for (Index j = 0; j < dim; ++j) {
    const cplx d = r(j, j);
    const double mag = std::abs(d);
    if (mag > 0.0)
      for (Index i = 0; i < dim; ++i) q(i, j) *= d / mag;
  }
  return q;
}

Circuit ghz_circuit(int n) {  // generators.cpp:52-71
  Circuit c;
  c.n = n;
  PrimOp h;
  h.kind = GateKind::H;
  h.q0 = 0;
  c.ops.push_back(h);
  for (int i = 0; i + 1 < n; ++i) {
    PrimOp cx;
    cx.kind = GateKind::Cx;
    cx.q0 = i;
    cx.q1 = i + 1;
    c.ops.push_back(cx);
  }
  return c;
}

// generators.cpp:95-145; with the Haar entangler the sidecar gates are
// injected at their op_index (runner.cpp:193-217), which reproduces the
// emission order, so the op list is built directly in that order. The
// QASM text prints angles with %.17g (generators.cpp:44-48), which
// round-trips doubles exactly.
Circuit brickwork_circuit(int n, int depth, std::uint64_t seed, bool haar) {
  if (n < 2) throw std::invalid_argument("brickwork generator needs at least 2 qubits");
  if (depth < 1) throw std::invalid_argument("brickwork generator needs depth >= 1");
  std::mt19937_64 e(seed);
  Circuit c;
  c.n = n;
  for (int unit = 0; unit < depth; ++unit) {
    for (int q = 0; q < n; ++q) {
      PrimOp op;
      op.kind = GateKind::U3;
      op.q0 = q;
      const double theta = uniform_unit(e) * 2.0 * M_PI;
      const double phi = uniform_unit(e) * 2.0 * M_PI;
      const double lam = uniform_unit(e) * 2.0 * M_PI;
      op.params = {theta, phi, lam};
      c.ops.push_back(op);
    }
    for (int p = unit % 2; p + 1 < n; p += 2) {
      PrimOp op;
      op.q0 = p;
      op.q1 = p + 1;
      if (!haar) {
        op.kind = GateKind::Cx;
      } else {
        op.kind = GateKind::U4;
        op.matrix = haar_unitary(4, e());
      }
      c.ops.push_back(op);
    }
  }
  return c;
}

// tests/support/test_util.cpp:36-75
Circuit random_circuit(int n, int gates, std::uint64_t seed, bool nonlocal) {
  std::mt19937_64 e(seed);
  auto pick = [&e](int bound) { return static_cast<int>(e() % static_cast<std::uint64_t>(bound)); };
  static const GateKind one[] = {GateKind::H,  GateKind::X,  GateKind::Y,  GateKind::Z,  GateKind::S,
                                 GateKind::Sdg, GateKind::T, GateKind::Tdg, GateKind::Rx, GateKind::Ry,
                                 GateKind::Rz, GateKind::U1, GateKind::U2, GateKind::U3};
  static const GateKind two[] = {GateKind::Cx, GateKind::Cz, GateKind::Swap};
  Circuit c;
  c.n = n;
  for (int i = 0; i < gates; ++i) {
    PrimOp op;
    const bool tw = n > 1 && pick(100) < 40;
    if (tw) {
      op.kind = two[pick(3)];
      op.q0 = pick(n);
      do {
        op.q1 = nonlocal ? pick(n) : std::min(n - 1, std::max(0, op.q0 + (pick(2) ? 1 : -1)));
      } while (op.q1 == op.q0);
    } else {
      op.kind = one[pick(14)];
      op.q0 = pick(n);
    }
    for (int p = 0; p < param_count(op.kind); ++p) op.params.push_back(uniform_unit(e) * 2.0 * M_PI);
    c.ops.push_back(std::move(op));
  }
  return c;
}

// tests/support/test_util.cpp:77-119
MpsState random_mps(int n, Index chi, std::uint64_t seed) {
  std::mt19937_64 e(seed);
  auto gaussian = [&e]() {
    double u1 = uniform_unit(e);
    while (u1 <= 0.0) u1 = uniform_unit(e);
    const double u2 = uniform_unit(e);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  };
  MpsState s(n);
  std::vector<Index> bonds(static_cast<size_t>(n) + 1, 1);
  for (int i = 1; i < n; ++i) {
    const Index lc = Index{1} << std::min(i, 30);
    const Index rc = Index{1} << std::min(n - i, 30);
    bonds[static_cast<size_t>(i)] = std::min({chi, lc, rc});
  }
  for (int i = 0; i < n; ++i) {
    Site t;
    t.dl = bonds[static_cast<size_t>(i)];
    t.dr = bonds[static_cast<size_t>(i) + 1];
    t.a.resize(static_cast<size_t>(t.dl * 2 * t.dr));
    for (auto& v : t.a) {
      // Complex(gaussian(), gaussian()) under g++: imaginary part drawn first.
      const double im = gaussian();
      const double re = gaussian();
      v = cplx(re, im);
    }
    s.sites[static_cast<size_t>(i)] = std::move(t);
  }
  s.bonds = bonds;
  s.center = -1;
  const double nrm = norm(s);
  if (nrm <= 0.0) throw std::runtime_error("random state degenerated");
  for (auto& v : s.sites[0].a) v /= nrm;
  return s;
}

// ---------------------------------------------------------------- executor

static Report apply_fused(MpsState& s, const FusedGate& g, const Policy& p, bool bondprop) {
  // gate_apply.cpp:257-268
  if (!g.two()) return apply_1q(s, g.m, g.q0);
  if (g.local()) return apply_2q_local(s, g.m, g.q0, p);
  return bondprop ? apply_2q_bondprop(s, g.m, g.q0, g.q1, p) : apply_2q_swap(s, g.m, g.q0, g.q1, p);
}

using Clock = std::chrono::steady_clock;

// executor.cpp:73-97
ExecStats execute_serial(MpsState& s, const std::vector<FusedGate>& gates, const Policy& p,
                         bool bondprop) {
  const auto t0 = Clock::now();
  ExecStats st;
  st.peak_bond = s.max_bond();
  for (const FusedGate& g : gates) {
    const Report r = apply_fused(s, g, p, bondprop);
    st.reports.push_back(r);
    st.total_w += r.w;
    st.peak_bond = std::max(st.peak_bond, s.max_bond());
  }
  s.validate();
  st.wall_ns = static_cast<std::uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
  return st;
}

// executor.cpp:99-232: per layer, `workers` threads claim gate indices from
// an atomic counter; a barrier completion merges the layer and re-arms.
ExecStats execute_parallel(MpsState& s, const std::vector<std::vector<FusedGate>>& layers,
                           const Policy& p, int workers) {
  if (workers < 1) throw std::invalid_argument("worker count must be >= 1");
  for (const auto& layer : layers)
    for (const FusedGate& g : layer) {
      if (!g.local()) throw std::invalid_argument("parallel execution requires a local-gate plan");
      if (g.hi() >= s.n()) throw std::invalid_argument("gate qubits out of range");
    }
  const auto t0 = Clock::now();
  ExecStats st;
  st.peak_bond = s.max_bond();
  size_t total = 0;
  std::vector<size_t> offset;
  for (const auto& l : layers) {
    offset.push_back(total);
    total += l.size();
  }
  st.reports.resize(total);
  if (layers.empty()) return st;
  std::atomic<size_t> counter{0};
  std::atomic<bool> failed{false};
  std::exception_ptr first;
  std::mutex mu;
  size_t cursor = 0;
  auto complete = [&]() noexcept {
    try {
      if (!failed.load()) s.validate();
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!first) first = std::current_exception();
      failed.store(true);
    }
    st.peak_bond = std::max(st.peak_bond, s.max_bond());
    counter.store(0);
    ++cursor;
  };
  std::barrier sync(workers, complete);
  auto body = [&]() {
    for (size_t li = 0; li < layers.size(); ++li) {
      const auto& layer = layers[li];
      while (!failed.load(std::memory_order_acquire)) {
        const size_t idx = counter.fetch_add(1);
        if (idx >= layer.size()) break;
        try {
          st.reports[offset[li] + idx] = apply_fused(s, layer[idx], p, false);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!first) first = std::current_exception();
          failed.store(true, std::memory_order_release);
        }
      }
      sync.arrive_and_wait();
    }
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) pool.emplace_back(body);
  for (auto& t : pool) t.join();
  if (failed.load()) {
    try {
      std::rethrow_exception(first);
    } catch (const std::exception& e) {
      throw NumericError(std::string("parallel execution aborted: ") + e.what());
    }
  }
  for (const Report& r : st.reports) st.total_w += r.w;
  st.wall_ns = static_cast<std::uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
  return st;
}

// ---------------------------------------------------------------- sampler

// sampler.cpp:35-66
Sampler::Sampler(const MpsState& state, bool memo, size_t cap_) : memoize(memo), cap(cap_) {
  const double nrm = norm(state);
  if (std::abs(nrm - 1.0) > 1e-8)
    throw NumericError("sampling requires a normalized state, norm is " + std::to_string(nrm));
  MpsState prepared = state;
  move_center(prepared, prepared.n() - 1);  // left_canonicalize
  move_center(prepared, 0);                 // right_canonicalize
  n = prepared.n();
  for (int i = 0; i < n; ++i) {
    const Site& t = prepared.sites[static_cast<size_t>(i)];
    slices.push_back({phys_slice(t, 0), phys_slice(t, 1)});
  }
}

static std::vector<cplx> rowvec_times(const std::vector<cplx>& env, const Mat& m) {
  std::vector<cplx> out(static_cast<size_t>(m.cols));
  for (Index c = 0; c < m.cols; ++c) {
    cplx acc{};
    for (Index r = 0; r < m.rows; ++r) acc += env[static_cast<size_t>(r)] * m(r, c);
    out[static_cast<size_t>(c)] = acc;
  }
  return out;
}
static double sq_norm(const std::vector<cplx>& v) {
  double s = 0.0;
  for (const cplx& x : v) s += std::norm(x);
  return s;
}

// sampler.cpp:68-78
double Sampler::prob0(const std::vector<cplx>& env, int site) const {
  const auto& sl = slices[static_cast<size_t>(site)];
  const double raw0 = sq_norm(rowvec_times(env, sl[0]));
  const double raw1 = sq_norm(rowvec_times(env, sl[1]));
  const double total = raw0 + raw1;
  if (total < 1e-12)
    throw NumericError("degenerate state: total probability vanished at site " + std::to_string(site));
  return raw0 / total;
}

// sampler.cpp:80-143
std::map<std::string, std::uint64_t> Sampler::sample(std::uint64_t shots, std::uint64_t seed) {
  if (shots == 0) throw std::invalid_argument("shots must be positive");
  std::mt19937_64 e(seed);
  std::map<std::string, std::uint64_t> counts;
  std::string prefix;
  for (std::uint64_t shot = 0; shot < shots; ++shot) {
    prefix.clear();
    std::vector<cplx> env(1, cplx(1.0, 0.0));
    for (int site = 0; site < n; ++site) {
      double* memo = nullptr;
      if (memoize) {
        if (site == 0) {
          memo = &root_p0;
        } else if (auto it = cache.find(prefix); it != cache.end()) {
          memo = &it->second.p0;
        }
      }
      double p0;
      if (memo != nullptr && *memo >= 0.0) {
        p0 = *memo;
        ++hits;
      } else {
        p0 = prob0(env, site);
        if (memo != nullptr) *memo = p0;
      }
      const double u = uniform_unit(e);
      const int bit = u < p0 ? 0 : 1;
      prefix.push_back(static_cast<char>('0' + bit));
      if (memoize) {
        if (auto it = cache.find(prefix); it != cache.end()) {
          env = it->second.env;
          continue;
        }
      }
      std::vector<cplx> next = rowvec_times(env, slices[static_cast<size_t>(site)][static_cast<size_t>(bit)]);
      const double raw = sq_norm(next);
      if (raw < 1e-12 * 1e-12) throw NumericError("degenerate state: chosen branch has no weight");
      const double inv = std::sqrt(raw);
      for (auto& x : next) x /= inv;
      env = std::move(next);
      if (memoize && (cap == 0 || cache.size() < cap)) cache.emplace(prefix, Entry{env, -1.0});
    }
    ++counts[prefix];
  }
  return counts;
}

// ---------------------------------------------------------------- statevector

namespace {
struct Dense {
  int n;
  std::vector<cplx> a;
  explicit Dense(int nq) : n(nq), a(size_t{1} << nq) { a[0] = 1.0; }
  void apply_1q(const Mat& u, int q) {  // statevector.cpp:35-52
    const size_t stride = size_t{1} << (n - 1 - q);
    for (size_t block = 0; block < a.size(); block += 2 * stride)
      for (size_t i = block; i < block + stride; ++i) {
        const cplx a0 = a[i], a1 = a[i + stride];
        a[i] = u(0, 0) * a0 + u(0, 1) * a1;
        a[i + stride] = u(1, 0) * a0 + u(1, 1) * a1;
      }
  }
  void apply_2q(const Mat& u, int q0, int q1) {  // statevector.cpp:54-81
    const size_t s0 = size_t{1} << (n - 1 - q0), s1 = size_t{1} << (n - 1 - q1);
    for (size_t i = 0; i < a.size(); ++i) {
      if ((i & s0) || (i & s1)) continue;
      const cplx x[4] = {a[i], a[i + s1], a[i + s0], a[i + s0 + s1]};
      for (int r = 0; r < 4; ++r) {
        cplx acc{};
        for (int c = 0; c < 4; ++c) acc += u(r, c) * x[c];
        a[i + ((r & 2) ? s0 : 0) + ((r & 1) ? s1 : 0)] = acc;
      }
    }
  }
};
}  // namespace

std::vector<cplx> sv_run(int n, const std::vector<FusedGate>& gates) {  // statevector.cpp:104-115
  if (n > 24) throw std::invalid_argument("statevector capped");
  Dense d(n);
  for (const FusedGate& g : gates) {
    if (g.two()) d.apply_2q(g.m, g.q0, g.q1);
    else d.apply_1q(g.m, g.q0);
  }
  return d.a;
}

std::vector<cplx> sv_run_circuit(const Circuit& c) {  // statevector.cpp:91-102
  if (c.n > 24) throw std::invalid_argument("statevector capped");
  Dense d(c.n);
  for (const PrimOp& op : c.ops) {
    if (op.two()) d.apply_2q(gate_matrix(op), std::min(op.q0, op.q1), std::max(op.q0, op.q1));
    else d.apply_1q(gate_matrix_1q(op.kind, op.params), op.q0);
  }
  return d.a;
}

}  // namespace oracle
