// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
// extern "C" surface of the CPU oracle for the Python test harness (ctypes).
// Complex arrays are interleaved (re, im) doubles, row-major.
#include <cstring>
#include <string>

#include "mps_oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid argument, 3 numeric, 4 logic/other (runner.cpp:330-341 style).
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

Mat mat_from(const double* u, int dim) {
  Mat m(dim, dim);
  for (int i = 0; i < dim * dim; ++i) m.a[static_cast<size_t>(i)] = cplx(u[2 * i], u[2 * i + 1]);
  return m;
}

void put(double* out, const std::vector<cplx>& v) {
  std::memcpy(out, v.data(), v.size() * sizeof(cplx));
}

void put_report(const Report& r, double* w, Index* k, int* svd) {
  if (w) *w = r.w;
  if (k) *k = r.new_bond;
  if (svd) *svd = r.svd_count;
}

using GateList = std::vector<FusedGate>;

struct SamplerBox {
  Sampler s;
  std::map<std::string, std::uint64_t> last;
  std::vector<std::pair<std::string, std::uint64_t>> flat;
};

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- state
void* orc_state_new(int n) {
  MpsState* s = nullptr;
  guard([&] { s = new MpsState(n); });
  return s;
}
void* orc_state_random(int n, Index chi, std::uint64_t seed) {
  MpsState* s = nullptr;
  guard([&] { s = new MpsState(random_mps(n, chi, seed)); });
  return s;
}
void* orc_state_copy(void* h) { return new MpsState(*static_cast<MpsState*>(h)); }
void orc_state_free(void* h) { delete static_cast<MpsState*>(h); }
int orc_state_n(void* h) { return static_cast<MpsState*>(h)->n(); }
void orc_state_bonds(void* h, Index* out) {
  const auto& b = static_cast<MpsState*>(h)->bonds;
  std::memcpy(out, b.data(), b.size() * sizeof(Index));
}
int orc_state_center(void* h) { return static_cast<MpsState*>(h)->center; }
void orc_state_set_center(void* h, int c) { static_cast<MpsState*>(h)->center = c; }
int orc_state_validate(void* h) {
  return guard([&] { static_cast<MpsState*>(h)->validate(); });
}
int orc_get_site(void* h, int i, Index* dl, Index* dr, double* out) {
  return guard([&] {
    const Site& t = static_cast<MpsState*>(h)->sites.at(static_cast<size_t>(i));
    *dl = t.dl;
    *dr = t.dr;
    if (out) put(out, t.a);
  });
}
// Replaces site i (like tests writing state.site(i) and set_bond_dim).
int orc_set_site(void* h, int i, Index dl, Index dr, const double* data) {
  return guard([&] {
    MpsState& s = *static_cast<MpsState*>(h);
    Site& t = s.sites.at(static_cast<size_t>(i));
    t.dl = dl;
    t.dr = dr;
    t.a.resize(static_cast<size_t>(dl * 2 * dr));
    std::memcpy(t.a.data(), data, t.a.size() * sizeof(cplx));
    s.bonds[static_cast<size_t>(i)] = dl;
    s.bonds[static_cast<size_t>(i) + 1] = dr;
  });
}

// ---- gates
int orc_apply_1q(void* h, const double* u, int q, double* w, Index* k, int* svd) {
  return guard([&] { put_report(apply_1q(*static_cast<MpsState*>(h), mat_from(u, 2), q), w, k, svd); });
}
// method: 0 local (q1 must be q0+1), 1 swap chain, 2 bond propagation
int orc_apply_2q(void* h, const double* u, int q0, int q1, int method, Index max_bond, double cutoff,
                 double* w, Index* k, int* svd) {
  return guard([&] {
    MpsState& s = *static_cast<MpsState*>(h);
    Policy p{max_bond, cutoff};
    const Mat m = mat_from(u, 4);
    Report r;
    if (method == 0) {
      if (q1 != q0 + 1) throw std::invalid_argument("local method needs q1 == q0 + 1");
      r = apply_2q_local(s, m, q0, p);
    } else if (method == 1) {
      r = apply_2q_swap(s, m, q0, q1, p);
    } else {
      r = apply_2q_bondprop(s, m, q0, q1, p);
    }
    put_report(r, w, k, svd);
  });
}

// ---- queries
int orc_move_center(void* h, int c) {
  return guard([&] { move_center(*static_cast<MpsState*>(h), c); });
}
int orc_norm(void* h, double* out) {
  return guard([&] { *out = norm(*static_cast<MpsState*>(h)); });
}
int orc_amplitude(void* h, const char* bits, double* out) {
  return guard([&] {
    const cplx a = amplitude(*static_cast<MpsState*>(h), bits);
    out[0] = a.real();
    out[1] = a.imag();
  });
}
int orc_overlap(void* a, void* b, double* out) {
  return guard([&] {
    const cplx v = overlap(*static_cast<MpsState*>(a), *static_cast<MpsState*>(b));
    out[0] = v.real();
    out[1] = v.imag();
  });
}
int orc_to_statevector(void* h, int max_qubits, double* out) {
  return guard([&] { put(out, to_statevector(*static_cast<MpsState*>(h), max_qubits)); });
}

// ---- svd (svd.hpp contract), for the truncation-rule tests
int orc_svd(int rows, int cols, const double* data, Index max_rank, double cutoff, Index* k, double* s,
            double* u, double* vdag, double* w) {
  return guard([&] {
    Mat m(rows, cols);
    std::memcpy(m.a.data(), data, m.a.size() * sizeof(cplx));
    SvdResult r = svd(m, max_rank, cutoff);
    *k = static_cast<Index>(r.s.size());
    std::memcpy(s, r.s.data(), r.s.size() * sizeof(double));
    if (u) put(u, r.u.a);
    if (vdag) put(vdag, r.vdag.a);
    *w = r.discarded_weight;
  });
}
// 0: zgesdd (default, BDCSVD's family), 1: zgesvj (independent cross-check),
// 2: zgesvd (bidiagonal QR iteration)
int orc_set_svd_backend(int b) {
  oracle::g_svd_backend.store(b == 1 || b == 2 ? b : 0);
  return 0;
}

Index orc_truncation_rank(const double* s, Index n, Index max_rank, double cutoff, double* w) {
  std::vector<double> v(s, s + n);
  return truncation_rank(v, max_rank, cutoff, w);
}

void orc_haar(int dim, std::uint64_t seed, double* out) { put(out, haar_unitary(dim, seed).a); }

// ---- circuits / gate lists
void* orc_circuit_new(int n) {
  auto* c = new Circuit();
  c->n = n;
  return c;
}
void orc_circuit_free(void* c) { delete static_cast<Circuit*>(c); }
// kind = GateKind ordinal; matrix only for U4 (16 interleaved complex)
int orc_circuit_add(void* c, int kind, int q0, int q1, const double* params, int np, const double* matrix) {
  return guard([&] {
    PrimOp op;
    op.kind = static_cast<GateKind>(kind);
    op.q0 = q0;
    op.q1 = q1;
    op.params.assign(params, params + np);
    if (op.kind == GateKind::U4) op.matrix = mat_from(matrix, 4);
    static_cast<Circuit*>(c)->ops.push_back(std::move(op));
  });
}
void* orc_circuit_brickwork(int n, int depth, std::uint64_t seed, int haar) {
  Circuit* c = nullptr;
  guard([&] { c = new Circuit(brickwork_circuit(n, depth, seed, haar != 0)); });
  return c;
}
void* orc_circuit_ghz(int n) { return new Circuit(ghz_circuit(n)); }
void* orc_circuit_random(int n, int gates, std::uint64_t seed, int nonlocal) {
  return new Circuit(random_circuit(n, gates, seed, nonlocal != 0));
}
int orc_circuit_size(void* c) { return static_cast<int>(static_cast<Circuit*>(c)->ops.size()); }
int orc_circuit_n(void* c) { return static_cast<Circuit*>(c)->n; }
// op i: kind, q0, q1, params (up to 3), matrix (16 complex, U4 or the canonical matrix)
int orc_circuit_get(void* c, int i, int* kind, int* q0, int* q1, double* params, int* np) {
  return guard([&] {
    const PrimOp& op = static_cast<Circuit*>(c)->ops.at(static_cast<size_t>(i));
    *kind = static_cast<int>(op.kind);
    *q0 = op.q0;
    *q1 = op.q1;
    *np = static_cast<int>(op.params.size());
    for (size_t j = 0; j < op.params.size(); ++j) params[j] = op.params[j];
  });
}
int orc_gate_matrix(int kind, int q0, int q1, const double* params, int np, const double* u4, double* out) {
  return guard([&] {
    PrimOp op;
    op.kind = static_cast<GateKind>(kind);
    op.q0 = q0;
    op.q1 = q1;
    op.params.assign(params, params + np);
    if (op.kind == GateKind::U4) op.matrix = mat_from(u4, 4);
    put(out, gate_matrix(op).a);
  });
}

void* orc_gates_new() { return new GateList(); }
void orc_gates_free(void* g) { delete static_cast<GateList*>(g); }
int orc_gates_size(void* g) { return static_cast<int>(static_cast<GateList*>(g)->size()); }
int orc_gates_add(void* g, int q0, int q1, const double* m) {
  return guard([&] {
    FusedGate fg;
    fg.q0 = q0;
    fg.q1 = q1;
    fg.m = mat_from(m, q1 >= 0 ? 4 : 2);
    static_cast<GateList*>(g)->push_back(std::move(fg));
  });
}
int orc_gates_get(void* g, int i, int* q0, int* q1, int* flipped, double* m) {
  return guard([&] {
    const FusedGate& fg = static_cast<GateList*>(g)->at(static_cast<size_t>(i));
    *q0 = fg.q0;
    *q1 = fg.q1;
    *flipped = fg.flipped ? 1 : 0;
    put(m, fg.m.a);
  });
}
void* orc_fuse(void* c) {
  GateList* g = nullptr;
  guard([&] { g = new GateList(fuse_circuit(*static_cast<Circuit*>(c))); });
  return g;
}
void* orc_decompose(void* g, int n) {
  GateList* out = nullptr;
  guard([&] { out = new GateList(decompose_nonlocal(*static_cast<GateList*>(g), n)); });
  return out;
}
// Fills layer_of[i] with the layer of gate i (layerize order); returns #layers or -1.
int orc_layerize(void* g, int* layer_of) {
  int nl = -1;
  guard([&] {
    const GateList& gl = *static_cast<GateList*>(g);
    int n = 0;
    for (const auto& x : gl) n = std::max(n, x.hi() + 1);
    std::vector<int> last(static_cast<size_t>(n), -1);
    const auto plan = layerize(gl);  // validates locality
    for (size_t i = 0; i < gl.size(); ++i) {
      int layer = 0;
      for (int q = gl[i].lo(); q <= gl[i].hi(); ++q) layer = std::max(layer, last[static_cast<size_t>(q)] + 1);
      for (int q = gl[i].lo(); q <= gl[i].hi(); ++q) last[static_cast<size_t>(q)] = layer;
      layer_of[i] = layer;
    }
    nl = static_cast<int>(plan.size());
  });
  return nl;
}

// ---- execution
int orc_execute_serial(void* h, void* g, Index max_bond, double cutoff, int bondprop, double* total_w,
                       Index* peak, double* gate_w, Index* gate_k, std::uint64_t* wall_ns) {
  return guard([&] {
    ExecStats st = execute_serial(*static_cast<MpsState*>(h), *static_cast<GateList*>(g),
                                  Policy{max_bond, cutoff}, bondprop != 0);
    *total_w = st.total_w;
    *peak = st.peak_bond;
    for (size_t i = 0; i < st.reports.size(); ++i) {
      if (gate_w) gate_w[i] = st.reports[i].w;
      if (gate_k) gate_k[i] = st.reports[i].new_bond;
    }
    if (wall_ns) *wall_ns = st.wall_ns;
  });
}
// Layerizes the (local) gate list and runs it with `workers` threads. Reports
// are returned in layer-plan order.
int orc_execute_parallel(void* h, void* g, Index max_bond, double cutoff, int workers, double* total_w,
                         Index* peak, double* gate_w, Index* gate_k, std::uint64_t* wall_ns) {
  return guard([&] {
    const auto plan = layerize(*static_cast<GateList*>(g));
    ExecStats st = execute_parallel(*static_cast<MpsState*>(h), plan, Policy{max_bond, cutoff}, workers);
    *total_w = st.total_w;
    *peak = st.peak_bond;
    for (size_t i = 0; i < st.reports.size(); ++i) {
      if (gate_w) gate_w[i] = st.reports[i].w;
      if (gate_k) gate_k[i] = st.reports[i].new_bond;
    }
    if (wall_ns) *wall_ns = st.wall_ns;
  });
}

int orc_sv_run(int n, void* g, double* out) {
  return guard([&] { put(out, sv_run(n, *static_cast<GateList*>(g))); });
}
int orc_sv_run_circuit(void* c, double* out) {
  return guard([&] { put(out, sv_run_circuit(*static_cast<Circuit*>(c))); });
}

// ---- sampler
void* orc_sampler_new(void* h, int memo, std::uint64_t cap) {
  SamplerBox* b = nullptr;
  guard([&] { b = new SamplerBox{Sampler(*static_cast<MpsState*>(h), memo != 0, cap), {}, {}}; });
  return b;
}
void orc_sampler_free(void* s) { delete static_cast<SamplerBox*>(s); }
int orc_sample(void* s, std::uint64_t shots, std::uint64_t seed, int* unique) {
  return guard([&] {
    auto* b = static_cast<SamplerBox*>(s);
    b->last = b->s.sample(shots, seed);
    b->flat.assign(b->last.begin(), b->last.end());
    *unique = static_cast<int>(b->flat.size());
  });
}
void orc_sample_get(void* s, int i, char* bits, std::uint64_t* count) {
  auto* b = static_cast<SamplerBox*>(s);
  const auto& e = b->flat.at(static_cast<size_t>(i));
  std::memcpy(bits, e.first.data(), e.first.size());
  *count = e.second;
}
std::uint64_t orc_sampler_hits(void* s) { return static_cast<SamplerBox*>(s)->s.hits; }
std::uint64_t orc_sampler_cache_size(void* s) { return static_cast<SamplerBox*>(s)->s.cache.size(); }
void orc_sampler_clear(void* s) {
  auto* b = static_cast<SamplerBox*>(s);
  b->s.cache.clear();
  b->s.root_p0 = -1.0;
}

}  // extern "C"
