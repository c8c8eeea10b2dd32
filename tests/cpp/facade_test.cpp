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

int main() {
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
  std::printf("facade ok\n");
  return 0;
}
