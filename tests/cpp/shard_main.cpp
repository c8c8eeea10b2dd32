// Multi-GPU shard layer through the C++ facade (include/mpsim_b200.hpp), the
// way a C++ host of the reference would drive it: one process per GPU, the
// NCCL id handed over through a file. Every rank runs brick layers and a
// circuit with non-local gates on a sharded chain; rank 0 reruns the same
// work on one GPU (MpsState) and checks bonds, amplitudes, norm, <Z_q> and
// sample counts bit for bit.
//   shard_main RANK WORLD ID_FILE [DEVICE]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <thread>

#include "mpsim_b200.hpp"

using namespace mpsim;

static CTensor haar4(std::mt19937_64& e) {
  std::normal_distribution<double> nd;
  std::vector<Complex> z(16);
  for (auto& x : z) x = Complex(nd(e), nd(e));
  // Gram-Schmidt on the columns
  std::vector<Complex> q(16);
  for (int c = 0; c < 4; ++c) {
    std::vector<Complex> v(4);
    for (int r = 0; r < 4; ++r) v[r] = z[r * 4 + c];
    for (int p = 0; p < c; ++p) {
      Complex d = 0;
      for (int r = 0; r < 4; ++r) d += std::conj(q[r * 4 + p]) * v[r];
      for (int r = 0; r < 4; ++r) v[r] -= d * q[r * 4 + p];
    }
    double nrm = 0;
    for (auto& x : v) nrm += std::norm(x);
    for (int r = 0; r < 4; ++r) q[r * 4 + c] = v[r] / std::sqrt(nrm);
  }
  CTensor t({4, 4});
  for (int i = 0; i < 16; ++i) t.data()[i] = q[i];
  return t;
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const int rank = std::atoi(argv[1]), world = std::atoi(argv[2]);
  const std::string idf = argv[3];
  const int device = argc > 4 ? std::atoi(argv[4]) : rank;
  NcclId id{};
  if (world > 1) {
    if (rank == 0) {
      id = nccl_unique_id();
      std::ofstream(idf + ".tmp", std::ios::binary).write(reinterpret_cast<const char*>(id.data()), 128);
      std::rename((idf + ".tmp").c_str(), idf.c_str());
    } else {
      for (int i = 0; i < 6000; ++i) {
        std::ifstream f(idf, std::ios::binary);
        if (f && f.read(reinterpret_cast<char*>(id.data()), 128)) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(50));
      }
    }
  }
  const int n = 24;
  const Index chi = 32;
  std::mt19937_64 e(77);
  std::vector<std::vector<FusedGate>> layers;
  for (int L = 0; L < 6; ++L) {
    std::vector<FusedGate> layer;
    for (int q = L % 2; q + 1 < n; q += 2) layer.push_back(FusedGate{q, q + 1, false, haar4(e)});
    layers.push_back(layer);
  }
  CTensor cx({4, 4});
  for (int i = 0; i < 16; ++i) cx.data()[i] = 0;
  cx.data()[0] = cx.data()[5] = cx.data()[11] = cx.data()[14] = 1;
  std::vector<FusedGate> nonlocal;
  for (int q = 0; q + 3 < n; q += 5) nonlocal.push_back(FusedGate{q, q + 3, false, cx});
  for (int q = 1; q + 1 < n; q += 2) nonlocal.push_back(FusedGate{q, q + 1, false, haar4(e)});
  TruncationPolicy p;
  p.max_bond = chi;
  p.cutoff = 1e-12;
  ShardedChain ch(n, chi, rank, world, world > 1 ? &id : nullptr, device);
  for (auto& l : layers) ch.apply_layer(l, p);
  ch.execute(nonlocal, p);
  std::vector<std::string> bits;
  std::mt19937_64 b(9);
  for (int k = 0; k < 8; ++k) {
    std::string s(n, '0');
    for (auto& c : s) c = (b() & 1) ? '1' : '0';
    bits.push_back(s);
  }
  std::vector<Complex> amps;
  for (auto& s : bits) amps.push_back(ch.amplitude(s));
  const double nrm = ch.norm();
  CTensor pz({2, 2});
  pz.data()[0] = 1;
  pz.data()[1] = pz.data()[2] = 0;
  pz.data()[3] = -1;
  const Complex z5 = ch.expect_1q(pz, 5);
  const int c = n / 2;
  ch.move_center(c);
  const double nc = ch.norm();
  if (ch.lo() <= c && c < ch.hi()) {
    CTensor t = ch.site(c);
    for (Index i = 0; i < t.size(); ++i) t.data()[i] /= nc;
    ch.set_site(c, t);
  }
  ShotResult sr = ch.sample(2000, 5, 512);
  const auto owned = ch.owned_bond_dims();
  ch.barrier();
  if (rank == 0) {
    MpsState ref(n, chi, device);
    for (auto& l : layers) execute_parallel(ref, LayerPlan{{l}}, p, 1);
    execute_serial(ref, nonlocal, p);
    bool ok = std::abs(nrm - norm(ref)) == 0.0;
    for (size_t k = 0; k < bits.size(); ++k) ok = ok && amps[k] == amplitude(ref, bits[k]);
    ok = ok && owned[0] == ref.bond_dims()[static_cast<size_t>(ch.lo())];
    move_center(ref, c);
    CTensor t = ref.site(c);
    const double rn = norm(ref);
    for (Index i = 0; i < t.size(); ++i) t.data()[i] /= rn;
    ref.set_site(c, t);
    ShotResult rs = sample(ref, 2000, 5);
    const bool ok_s = rs.counts == sr.counts;
    std::printf("shard world=%d n=%d chi=%lld amplitudes/norm %s, <Z5> %.12f, sample counts %s\n", world, n,
                (long long)chi, ok ? "bit-identical" : "DIFFER", z5.real(), ok_s ? "equal" : "DIFFER");
    if (!(ok && ok_s)) return 1;
    std::printf("shard ok\n");
  }
  return 0;
}
