// C++ drop-in check: the reference-style API (include/mpsim_b200.hpp) driving
// the B200 engine, mirroring test_gate_apply.cpp / test_mps.cpp known answers.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "mpsim_b200.hpp"

using namespace mpsim;

#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      std::exit(1);                                                  \
    }                                                                \
  } while (0)

// Host-only front end: parse/fuse/plan/generate (no device touched).
static void host_checks() {
  int n = 0;
  const auto g = fuse_qasm("OPENQASM 2.0;\nqreg q[3];\nh q[0];\ncx q[2],q[0];\n", {}, &n);
  CHECK(n == 3 && g.size() == 1 && g[0].q0 == 0 && g[0].q1 == 2 && g[0].flipped);
  const LayerPlan plan = plan_layers(g, 3);
  CHECK(plan.layers.size() == 3 && plan.layers[1][0].q0 == 1);
  bool threw = false;
  try {
    fuse_qasm("OPENQASM 2.0; qreg q[2];\nccx q[0],q[1];");
  } catch (const ParseError& e) {
    threw = e.line() == 2 && exit_code_for_error(e) == 2;
  }
  CHECK(threw);
  BrickworkOptions o;
  o.n_qubits = 6;
  o.depth = 3;
  o.seed = 5;
  o.entangler = Entangler::Haar;
  const GeneratedCircuit gc = brickwork_qasm(o);
  CHECK(!gc.sidecar_json.empty());
  const auto fused = fuse_qasm(gc.qasm, gc.sidecar_json);
  CHECK(fused.size() == 8);  // 3 + 2 + 3 entanglers; every u3 is absorbed
  threw = false;
  try {
    RunConfig bad;
    bad.qasm_text = ghz_qasm(4);
    bad.backend = Backend::MpsParallel;
    bad.nonlocal = NonlocalMethod::BondProp;
    run_circuit_json(bad);
  } catch (const ConfigError& e) {
    threw = exit_code_for_error(e) == 1;
  }
  CHECK(threw);
}

int main(int argc, char** argv) {
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "--host-only") {
    std::printf("facade host ok\n");
    return 0;
  }
  const double hs = 1.0 / std::sqrt(2.0);
  const CTensor h({2, 2}, {hs, hs, hs, -hs});
  const CTensor cx({4, 4}, {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0});
  // GHZ bonds exactly 2 (test_gate_apply.cpp:283-295)
  for (int n : {4, 16, 64}) {
    MpsState s(n);
    apply_1q(s, h, 0);
    for (int i = 0; i + 1 < n; ++i) apply_2q_local(s, cx, i, TruncationPolicy{});
    for (int i = 1; i < n; ++i) CHECK(s.bond_dim(i) == 2);
    CHECK(std::abs(amplitude(s, std::string(n, '1')) - Complex(hs, 0)) <= 1e-12);
  }
  // CX|00> trims to bond 1 (test_gate_apply.cpp:110-117)
  {
    MpsState s(2);
    const ApplyReport r = apply_2q_local(s, cx, 0, TruncationPolicy{});
    CHECK(r.new_bond == 1 && r.discarded_weight == 0.0);
  }
  // bad inputs raise std::invalid_argument (test_gate_apply.cpp:173-183)
  {
    MpsState s(3);
    bool threw = false;
    try {
      TruncationPolicy bad;
      bad.cutoff = 1.5;
      apply_2q_local(s, cx, 0, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // swap routing over distance (test_gate_apply.cpp:194-210)
  {
    MpsState s(4);
    apply_1q(s, h, 0);
    const ApplyReport r = apply_2q_swap(s, cx, 0, 3, TruncationPolicy{});
    CHECK(r.svd_count == 5);
    const auto sv = to_statevector(s);
    CHECK(std::abs(sv[0] - Complex(hs, 0)) <= 1e-12 && std::abs(sv[9] - Complex(hs, 0)) <= 1e-12);
    s.validate();
  }
  // executor over a fused list with a capped policy
  {
    MpsState s(8);
    std::vector<FusedGate> gates;
    for (int layer = 0; layer < 6; ++layer)
      for (int q = layer % 2; q + 1 < 8; q += 2) {
        FusedGate g;
        g.q0 = q;
        g.q1 = q + 1;
        const double c = std::cos(0.3 + q), sn = std::sin(0.3 + q);
        g.matrix = CTensor({4, 4}, {c, 0, 0, Complex(0, -sn), 0, c, Complex(0, -sn), 0, 0, Complex(0, -sn), c, 0,
                                    Complex(0, -sn), 0, 0, c});
        gates.push_back(g);
      }
    TruncationPolicy p;
    p.max_bond = 4;
    p.cutoff = 1e-12;
    const ExecStats st = execute_serial(s, gates, p);
    CHECK(st.peak_bond <= 4 && st.layers == 6);
    CHECK(std::abs(norm(s) - 1.0) < 1e-6 || st.total_discarded_weight > 0.0);
  }
  // run_circuit: GHZ counts on the corner strings (test_runner.cpp:37-51)
  {
    RunConfig c;
    c.qasm_text = ghz_qasm(4);
    c.shots = 1000;
    c.seed = 5;
    const std::string j = run_circuit_json(c);
    CHECK(j.find("\"peak_bond\":2") != std::string::npos);
    CHECK(j.find("\"0000\":") != std::string::npos && j.find("\"1111\":") != std::string::npos);
  }
  std::printf("facade ok\n");
  return 0;
}
