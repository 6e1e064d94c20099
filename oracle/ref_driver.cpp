// ref_driver: runs the UNMODIFIED reference (qforge headers under
// /root/reference/proj/include, built with third_party/eigen_lite) to
//   (1) emit golden vectors for tests/golden/ (`ref_driver golden <dir>`), and
//   (2) time the reference CPU simulator through its public API for bench.py's
//       cpu_baseline / --impl reference leg (`ref_driver bench ...`).
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product links or calls this.
#include <omp.h>

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "circuits.hpp"
#include "qforge/bench.hpp"
#include "qforge/fusion.hpp"
#include "qforge/pathsum.hpp"
#include "qforge/simulator.hpp"
#include "qforge/variational.hpp"
#include "test_util.hpp"  // oracle::random_circuit (reference tests)

using namespace qforge;

namespace {

std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}
std::string g17(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// Circuit text format (parsed by tests/golden_io.py):
//   P <qubits> <cbits>
//   G <kind> <dagger> <nt> t.. <nc> c.. <np> p(hex).. <nm> m(hex re, im)..
//   M <qubit> <cbit>
void write_program(const std::string& path, const Program& p) {
  std::ofstream f(path);
  f << "P " << p.qubit_count << " " << p.cbit_count << "\n";
  for (const auto& ins : p.body) {
    if (auto* g = std::get_if<GateOp>(&ins)) {
      const Gate& x = g->gate;
      f << "G " << static_cast<int>(x.kind) << " " << (x.dagger ? 1 : 0) << " " << x.targets.size();
      for (auto t : x.targets) f << " " << t;
      f << " " << x.controls.size();
      for (auto c : x.controls) f << " " << c;
      f << " " << x.params.size();
      for (auto v : x.params) f << " " << hexd(v);
      if (x.custom) {
        const auto& m = *x.custom;
        f << " " << m.rows() * m.cols();
        for (Eigen::Index r = 0; r < m.rows(); ++r)
          for (Eigen::Index c = 0; c < m.cols(); ++c)
            f << " " << hexd(m(r, c).real()) << " " << hexd(m(r, c).imag());
      } else {
        f << " 0";
      }
      f << "\n";
    } else if (auto* m = std::get_if<MeasureOp>(&ins)) {
      f << "M " << m->qubit << " " << m->cbit << "\n";
    } else {
      throw std::runtime_error("write_program: only flat gate/measure programs");
    }
  }
}

void write_amps(const std::string& path, const StateVector& sv) {
  std::ofstream f(path, std::ios::binary);
  auto a = sv.amplitudes();
  f.write(reinterpret_cast<const char*>(a.data()), static_cast<std::streamsize>(a.size() * sizeof(cdouble)));
}

struct Manifest {
  std::vector<std::string> entries;
  void add(const std::string& json) { entries.push_back(json); }
  void write(const std::string& path) {
    std::ofstream f(path);
    f << "[\n";
    for (std::size_t i = 0; i < entries.size(); ++i) f << "  " << entries[i] << (i + 1 < entries.size() ? ",\n" : "\n");
    f << "]\n";
  }
};

std::string qlist(const std::vector<std::uint32_t>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}
std::string dlist(const std::vector<double>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + g17(v[i]);
  return s + "]";
}

// Final state + reductions of a gate-only program, through run() (simulator.hpp:142).
void state_case(Manifest& man, const std::string& dir, const std::string& name, const Program& p,
                bool fusion = false) {
  SimOptions o;
  o.fusion_enabled = fusion;
  RunResult rr = run(p, o, 0);
  const StateVector& sv = *rr.final_state;
  write_program(dir + "/" + name + ".circ", p);
  write_amps(dir + "/" + name + ".amps", sv);
  std::vector<double> p1;
  for (std::uint32_t q = 0; q < p.qubit_count; ++q) p1.push_back(sv.probability_of_one(q));
  std::vector<std::uint32_t> sub;
  for (std::uint32_t q = 0; q < p.qubit_count; q += 2) sub.push_back(q);
  std::reverse(sub.begin(), sub.end());
  const auto marg = sv.probabilities(sub);
  man.add("{\"name\":\"" + name + "\",\"type\":\"state\",\"n\":" + std::to_string(p.qubit_count) +
          ",\"fusion\":" + (fusion ? "true" : "false") + ",\"checksum\":" + g17(probability_checksum(sv)) +
          ",\"norm2\":" + g17(sv.norm_squared()) + ",\"prob_one\":" + dlist(p1) +
          ",\"marginal_qubits\":" + qlist(sub) + ",\"marginal\":" + dlist(marg) + "}");
}

Program random_custom_circuit(std::uint32_t n, std::uint32_t gates, std::uint64_t seed) {
  // Mixed circuit with dense custom blocks k = 1..5 (random unitaries via QR),
  // extra controls and dagger, plus named gates from the reference corpus.
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gau;
  Program p = oracle::random_circuit(n, gates / 2, seed + 1000, true);
  Program out(n, 0);
  std::size_t next = 0;
  for (std::uint32_t i = 0; i < gates; ++i) {
    if (i % 2 == 0 && next < p.body.size()) {
      out.body.push_back(p.body[next++]);
      continue;
    }
    const std::uint32_t k = 1 + static_cast<std::uint32_t>(rng() % std::min<std::uint32_t>(5, n));
    std::vector<std::uint32_t> perm(n);
    for (std::uint32_t q = 0; q < n; ++q) perm[q] = q;
    for (std::uint32_t q = n; q > 1; --q) std::swap(perm[q - 1], perm[rng() % q]);
    const Eigen::Index dim = Eigen::Index(1) << k;
    CMatrix m(dim, dim);
    for (Eigen::Index r = 0; r < dim; ++r)
      for (Eigen::Index c = 0; c < dim; ++c) m(r, c) = cdouble(gau(rng), gau(rng));
    Eigen::HouseholderQR<CMatrix> qr(m);
    CMatrix u = qr.householderQ();
    std::vector<std::uint32_t> t(perm.begin(), perm.begin() + k);
    Gate g = make_custom_gate(t, u);
    if (k < n && rng() % 3 == 0) g.controls = {perm[k]};
    if (rng() % 4 == 0) g.dagger = true;
    out.add(std::move(g));
  }
  return out;
}

std::string counts_json(const std::map<std::string, std::uint64_t>& c) {
  std::string s = "{";
  bool first = true;
  for (auto& [k, v] : c) {
    s += (first ? "\"" : ",\"") + k + "\":" + std::to_string(v);
    first = false;
  }
  return s + "}";
}

void sample_case(Manifest& man, const std::string& dir, const std::string& name, const Program& p,
                 std::uint64_t seed, std::uint64_t shots) {
  SimOptions o;
  o.seed = seed;
  RunResult rr = run(p, o, shots);
  write_program(dir + "/" + name + ".circ", p);
  man.add("{\"name\":\"" + name + "\",\"type\":\"sample\",\"n\":" + std::to_string(p.qubit_count) +
          ",\"seed\":" + std::to_string(seed) + ",\"shots\":" + std::to_string(shots) +
          ",\"counts\":" + counts_json(rr.counts) + "}");
}

int golden(const std::string& dir) {
  Manifest man;
  // -- RNG stream (rng.hpp:9-46)
  {
    std::string s = "{\"name\":\"rng\",\"type\":\"rng\",\"streams\":[";
    const std::uint64_t seeds[] = {0, 7, 42, 424242, 0xdeadbeefcafeULL};
    for (std::size_t i = 0; i < 5; ++i) {
      Rng r(seeds[i]);
      s += std::string(i ? "," : "") + "{\"seed\":" + std::to_string(seeds[i]) + ",\"next\":[";
      for (int k = 0; k < 8; ++k) s += (k ? ",\"" : "\"") + std::to_string(r.next()) + "\"";
      Rng u(seeds[i]);
      std::vector<double> us;
      for (int k = 0; k < 8; ++k) us.push_back(u.uniform());
      Rng d = Rng::derive(seeds[i], 3);
      s += "],\"uniform\":" + dlist(us) + ",\"derive3\":\"" + std::to_string(d.next()) +
           "\",\"splitmix\":\"" + std::to_string(splitmix64(seeds[i])) + "\",\"below10\":\"" +
           std::to_string(Rng(seeds[i]).below(10)) + "\"}";
    }
    man.add(s + "]}");
  }
  // -- random layered circuits (bench.hpp:72-94)
  const std::uint32_t rc[][3] = {{4, 3, 7}, {5, 4, 7}, {8, 6, 42}, {10, 5, 424242}, {12, 4, 1}, {14, 3, 424242}};
  for (auto& c : rc) {
    state_case(man, dir, "random_" + std::to_string(c[0]) + "_" + std::to_string(c[1]) + "_" + std::to_string(c[2]),
               gen_random_circuit(c[0], c[1], c[2]));
  }
  state_case(man, dir, "random_10_5_424242_fused", gen_random_circuit(10, 5, 424242), true);
  // -- mixed named-gate corpus with controls and dagger (tests/test_util.hpp:213-257)
  for (std::uint64_t seed = 1; seed <= 6; ++seed) {
    const std::uint32_t n = 4 + static_cast<std::uint32_t>(seed % 4);
    state_case(man, dir, "mixed_" + std::to_string(seed), oracle::random_circuit(n, 60, 900 + seed, true));
  }
  // acceptance criterion 2 corpus (acceptance_test.cpp:81-85)
  for (std::size_t i = 0; i < 12; ++i) {
    const std::uint32_t n = 2 + static_cast<std::uint32_t>(i % 4);
    const std::uint32_t gates = 5 + static_cast<std::uint32_t>((i * 7) % 16);
    state_case(man, dir, "equiv_" + std::to_string(i), oracle::random_circuit(n, gates, 40000 + i, true));
  }
  // -- dense custom blocks k = 1..5 with controls / dagger
  for (std::uint64_t seed = 1; seed <= 4; ++seed) {
    const std::uint32_t n = 6 + static_cast<std::uint32_t>(seed);
    state_case(man, dir, "custom_" + std::to_string(seed), random_custom_circuit(n, 24, 700 + seed));
  }
  // -- fuse_circuit output (fusion.hpp:108-133) for the planner's reference mode
  for (std::uint64_t seed = 1; seed <= 3; ++seed) {
    Program p = oracle::random_circuit(6, 40, 300 + seed, true);
    for (std::uint32_t k = 2; k <= 5; ++k) {
      Program f = fuse_circuit(p, k);
      const std::string nm = "fuse_" + std::to_string(seed) + "_k" + std::to_string(k);
      write_program(dir + "/" + nm + ".in.circ", p);
      write_program(dir + "/" + nm + ".circ", f);
      man.add("{\"name\":\"" + nm + "\",\"type\":\"fuse\",\"k\":" + std::to_string(k) + ",\"blocks\":" +
              std::to_string(f.gate_count()) + "}");
    }
  }
  {
    Program p = gen_random_circuit(8, 4, 11);
    Program f = fuse_circuit(p, 3);
    write_program(dir + "/fuse_random_8_4_11_k3.in.circ", p);
    write_program(dir + "/fuse_random_8_4_11_k3.circ", f);
    man.add("{\"name\":\"fuse_random_8_4_11_k3\",\"type\":\"fuse\",\"k\":3,\"blocks\":" +
            std::to_string(f.gate_count()) + "}");
  }
  // -- GHZ / QFT / HEA generators (oracle/circuits.hpp)
  state_case(man, dir, "ghz_6", oraclegen::gen_ghz(6));
  state_case(man, dir, "qft_6_13", oraclegen::gen_qft(6, 13));
  state_case(man, dir, "qft_10_717", oraclegen::gen_qft(10, 717));
  state_case(man, dir, "hea_8_3_5", oraclegen::gen_hea(8, 3, 5));
  // -- expectation values (variational.hpp:19-54)
  for (std::uint32_t n : {4u, 8u}) {
    Program p = oraclegen::gen_hea(n, 3, 17 + n);
    PauliOperator h = oraclegen::hea_hamiltonian(n);
    const double e = expectation(p, h);
    write_program(dir + "/expect_hea_" + std::to_string(n) + ".circ", p);
    man.add("{\"name\":\"expect_hea_" + std::to_string(n) + "\",\"type\":\"expectation\",\"n\":" + std::to_string(n) +
            ",\"hamiltonian\":\"" + h.to_string() + "\",\"value\":" + g17(e) + "}");
  }
  // -- sampling (simulator.hpp:164-178)
  {
    Program bell(2, 2);
    bell.add(GateKind::H, {0});
    bell.add(GateKind::CNOT, {0, 1});
    bell.measure(0, 0);
    bell.measure(1, 1);
    sample_case(man, dir, "sample_bell", bell, 7, 4000);
    Program x(2, 2);
    x.add(GateKind::X, {0});
    x.measure(0, 0);
    x.measure(1, 1);
    sample_case(man, dir, "sample_key", x, 0, 10);
    for (std::uint64_t seed = 0; seed < 3; ++seed) {
      Program p = gen_random_circuit(10, 3, 50 + seed);
      p.cbit_count = 10;
      for (std::uint32_t q = 0; q < 10; ++q) p.measure(q, q);
      sample_case(man, dir, "sample_random10_" + std::to_string(seed), p, seed, 100000);
    }
    // partial, permuted measurement into a wider register
    Program p = oraclegen::gen_hea(9, 2, 3);
    p.cbit_count = 6;
    p.measure(8, 0);
    p.measure(0, 5);
    p.measure(4, 2);
    p.measure(2, 3);
    sample_case(man, dir, "sample_partial", p, 99, 50000);
    Program q = oraclegen::gen_qft(12, 1234);
    q.cbit_count = 12;
    for (std::uint32_t k = 0; k < 12; ++k) q.measure(k, k);
    sample_case(man, dir, "sample_qft12", q, 5, 200000);
  }
  // -- measurement collapse (statevector.hpp:219-247)
  {
    Program p = gen_random_circuit(6, 3, 21);
    std::string s = "{\"name\":\"collapse\",\"type\":\"collapse\",\"n\":6,\"circuit\":\"collapse.circ\",\"steps\":[";
    write_program(dir + "/collapse.circ", p);
    StateVector sv = *run(p).final_state;
    const double us[] = {0.1, 0.9, 0.5, 0.3, 0.77, 0.01};
    const std::uint32_t qs[] = {0, 5, 2, 3, 1, 4};
    for (int i = 0; i < 6; ++i) {
      int o = sv.measure_collapse(qs[i], us[i]);
      s += std::string(i ? "," : "") + "{\"q\":" + std::to_string(qs[i]) + ",\"u\":" + g17(us[i]) +
           ",\"outcome\":" + std::to_string(o) + ",\"norm2\":" + g17(sv.norm_squared()) + "}";
      if (i == 2) write_amps(dir + "/collapse_mid.amps", sv);
    }
    man.add(s + "]}");
  }
  // -- config 1 digests: GHZ(20) and QFT(20) full state + probabilities
  for (int which = 0; which < 2; ++which) {
    Program p = which == 0 ? oraclegen::gen_ghz(20) : oraclegen::gen_qft(20, 0x5a5a5);
    const std::string nm = which == 0 ? "ghz_20" : "qft_20";
    StateVector sv = *run(p).final_state;
    Rng r(1);
    std::vector<std::uint32_t> idx;
    std::vector<double> re, im;
    for (int k = 0; k < 4096; ++k) {
      std::uint64_t i = r.below(1u << 20);
      idx.push_back(static_cast<std::uint32_t>(i));
      re.push_back(sv.amplitude(i).real());
      im.push_back(sv.amplitude(i).imag());
    }
    auto probs = sv.probabilities();
    std::vector<double> first(probs.begin(), probs.begin() + 256);
    std::vector<std::uint32_t> sub = {19, 7, 0};
    write_program(dir + "/" + nm + ".circ", p);
    man.add("{\"name\":\"" + nm + "\",\"type\":\"digest\",\"n\":20,\"checksum\":" + g17(probability_checksum(sv)) +
            ",\"norm2\":" + g17(sv.norm_squared()) + ",\"idx\":" + qlist(idx) + ",\"re\":" + dlist(re) +
            ",\"im\":" + dlist(im) + ",\"probs_head\":" + dlist(first) + ",\"marginal_qubits\":" + qlist(sub) +
            ",\"marginal\":" + dlist(sv.probabilities(sub)) + "}");
  }
  // -- bench harness (bench.hpp:166-195)
  {
    BenchSpec spec;
    spec.qubits = 8;
    spec.layers = 6;
    spec.seed = 42;
    BenchResult a = run_bench(spec);
    spec.fusion = false;
    spec.peephole = false;
    BenchResult b = run_bench(spec);
    man.add("{\"name\":\"bench_8_6_42\",\"type\":\"bench\",\"checksum_opt\":" + g17(a.checksum) +
            ",\"checksum_raw\":" + g17(b.checksum) + ",\"gates_before\":" + std::to_string(a.gates_before) +
            ",\"gates_after\":" + std::to_string(a.gates_after) + "}");
  }
  man.write(dir + "/manifest.json");
  return 0;
}

// Digest of a 24-qubit sampling sweep too large to store as counts: FNV-1a of
// the per-shot basis indices (uint64, in draw order) plus the expectation.
int golden_big(const std::string& dir) {
  Manifest man;
  Program p = oraclegen::gen_hea(24, 10, 2024);
  PauliOperator h = oraclegen::hea_hamiltonian(24);
  const double e = expectation(p, h);
  write_program(dir + "/hea_24_10_2024.circ", p);
  StateVector sv = *run(p).final_state;
  std::string seeds = "[";
  BasisSampler sampler(sv);
  for (std::uint64_t seed = 0; seed < 10; ++seed) {
    Rng r(seed);
    std::uint64_t h64 = 1469598103934665603ULL;
    std::vector<std::uint64_t> hist(256, 0);
    for (int s = 0; s < 1000000; ++s) {
      std::uint64_t b = sampler.sample(r.uniform());
      for (int k = 0; k < 8; ++k) {
        h64 ^= (b >> (8 * k)) & 0xff;
        h64 *= 1099511628211ULL;
      }
      hist[b >> 16]++;
    }
    std::string hs = "[";
    for (int k = 0; k < 256; ++k) hs += (k ? "," : "") + std::to_string(hist[k]);
    seeds += std::string(seed ? "," : "") + "{\"seed\":" + std::to_string(seed) + ",\"fnv\":\"" + std::to_string(h64) +
             "\",\"hist_top8\":" + hs + "]}";
  }
  man.add("{\"name\":\"hea_24\",\"type\":\"sweep\",\"n\":24,\"layers\":10,\"seed\":2024,\"shots\":1000000,\"expectation\":" +
          g17(e) + ",\"checksum\":" + g17(probability_checksum(sv)) + ",\"seeds\":" + seeds + "]}");
  man.write(dir + "/manifest_big.json");
  return 0;
}

// Reference results for the BENCHMARKED configurations at their real size
// (BASELINE configs 2 and 3, bench.py workloads random28 / random30 / qft30):
// the final state of run() (simulator.hpp:142-194, fusion at the default k=3)
// reduced to probability_checksum (bench.hpp:141-148), norm_squared, 8 windows
// of 4096 amplitudes (window 0 at index 0, 7 at Rng(7)-drawn offsets), the
// first 256 probabilities and one 6-qubit marginal (statevector.hpp:190-207).
// Peak host memory ~2 x 16 GiB at 30 qubits (state + RunResult copy).
//   ref_driver golden_huge <dir> [random28|random30|qft30 ...]
int golden_huge(const std::string& dir, const std::vector<std::string>& which) {
  Manifest man;
  for (const std::string& name : which) {
    Program p;
    std::string gen;
    if (name == "random28") {
      p = gen_random_circuit(28, 20, 424242);
      gen = "\"random\",\"args\":[28,20,424242]";
    } else if (name == "random30") {
      p = gen_random_circuit(30, 20, 424242);
      gen = "\"random\",\"args\":[30,20,424242]";
    } else if (name == "qft30") {
      p = oraclegen::gen_qft(30, 0x2AAAAAAAull);
      gen = "\"qft\",\"args\":[30,715827882]";
    } else {
      std::fprintf(stderr, "golden_huge: unknown case %s\n", name.c_str());
      return 2;
    }
    const std::uint32_t n = p.qubit_count;
    const std::size_t dim = std::size_t{1} << n;
    auto t0 = std::chrono::steady_clock::now();
    RunResult rr = run(p);
    auto t1 = std::chrono::steady_clock::now();
    const StateVector& sv = *rr.final_state;
    const double cs = probability_checksum(sv);
    const double nrm = sv.norm_squared();
    constexpr std::size_t W = 4096;
    std::vector<std::uint64_t> starts = {0};
    Rng r(7);
    while (starts.size() < 8) starts.push_back(r.below(dim - W) & ~std::uint64_t{15});
    {
      std::ofstream f(dir + "/" + name + ".win.amps", std::ios::binary);
      for (std::uint64_t s : starts)
        for (std::size_t i = 0; i < W; ++i) {
          const cdouble a = sv.amplitude(s + i);
          f.write(reinterpret_cast<const char*>(&a), sizeof a);
        }
    }
    std::vector<double> head;
    for (std::size_t i = 0; i < 256; ++i) head.push_back(std::norm(sv.amplitude(i)));
    std::vector<std::uint32_t> sub = {n - 1, 17, 13, 5, 1, 0};
    const auto marg = sv.probabilities(sub);
    std::string st = "[";
    for (std::size_t i = 0; i < starts.size(); ++i) st += (i ? "," : "") + std::to_string(starts[i]);
    man.add("{\"name\":\"" + name + "\",\"type\":\"huge\",\"n\":" + std::to_string(n) + ",\"gen\":" + gen +
            ",\"gates\":" + std::to_string(p.body.size()) + ",\"checksum\":" + g17(cs) + ",\"norm2\":" + g17(nrm) +
            ",\"window\":4096,\"starts\":" + st + "],\"amps\":\"" + name + ".win.amps\",\"probs_head\":" +
            dlist(head) + ",\"marginal_qubits\":" + qlist(sub) + ",\"marginal\":" + dlist(marg) +
            ",\"run_seconds\":" + g17(std::chrono::duration<double>(t1 - t0).count()) +
            ",\"threads\":" + std::to_string(omp_get_max_threads()) + "}");
    std::fprintf(stderr, "golden_huge %s: run %.1f s, checksum %.17g\n", name.c_str(),
                 std::chrono::duration<double>(t1 - t0).count(), cs);
    man.write(dir + "/manifest_huge.json");  // rewritten after every case
  }
  return 0;
}

// CPU timing of the reference through run() (simulator.hpp:142): the first
// `layers` layers of gen_random_circuit(n, d, seed) (a bounded sample of the
// workload), `reps` repetitions; prints one JSON line per repetition.
int bench(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: ref_driver bench random <n> <d> <seed> <layers> <fusion0|1> [reps]\n");
    return 2;
  }
  const std::string kind = argv[2];
  const std::uint32_t n = std::stoul(argv[3]), d = std::stoul(argv[4]);
  const std::uint64_t seed = std::stoull(argv[5]);
  const std::uint32_t layers = std::stoul(argv[6]);
  const bool fusion = std::stoi(argv[7]) != 0;
  const int reps = argc > 8 ? std::stoi(argv[8]) : 1;
  Program full = kind == "qft" ? oraclegen::gen_qft(n, seed) : gen_random_circuit(n, d, seed);
  Program p(n, 0);
  const std::size_t per_layer = kind == "qft" ? full.body.size() : (n > 1 ? 2 * n : n);
  const std::size_t take = std::min(full.body.size(), per_layer * layers);
  p.body.assign(full.body.begin(), full.body.begin() + static_cast<std::ptrdiff_t>(take));
  SimOptions o;
  o.fusion_enabled = fusion;
  o.seed = seed;
  for (int r = 0; r < reps; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    RunResult rr = run(p, o, 0);
    auto t1 = std::chrono::steady_clock::now();
    const double cs = probability_checksum(*rr.final_state);
    auto t2 = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(t1 - t0).count();
    const double sec_all = std::chrono::duration<double>(t2 - t0).count();
    std::printf("{\"gates\":%zu,\"seconds\":%.6f,\"seconds_with_checksum\":%.6f,\"threads\":%d,\"checksum\":%.17g}\n",
                p.body.size(), sec, sec_all, omp_get_max_threads(), cs);
    std::fflush(stdout);
  }
  return 0;
}

// Cut planning and partial amplitudes (pathsum.hpp:232-459) of layered random
// circuits: the reference's CutPlan and its partial_amplitude values for a few
// targets, for tests/test_pathsum_gpu.py.  ref_driver golden_cut <dir>
int golden_cut(const std::string& dir) {
  Manifest man;
  const std::uint32_t ns[] = {6, 9, 12, 14, 16, 20};
  for (std::uint32_t n : ns) {
    Program p = gen_random_circuit(n, 2, 7 + n);
    const std::string name = "cut_random_" + std::to_string(n);
    write_program(dir + "/" + name + ".circ", p);
    CutPlan plan = plan_cut(p);
    std::vector<std::string> targets;
    Rng r(n);
    std::vector<std::uint64_t> idx = {0, (std::uint64_t{1} << n) - 1};
    for (int t = 0; t < 4; ++t) idx.push_back(r.below(std::uint64_t{1} << n));
    for (auto i : idx) {
      std::string b(n, '0');
      for (std::uint32_t q = 0; q < n; ++q)
        if ((i >> q) & 1) b[n - 1 - q] = '1';
      targets.push_back(b);
    }
    auto amps = partial_amplitude(p, plan, targets);
    std::vector<std::uint32_t> ca(plan.crossing_gates.begin(), plan.crossing_gates.end());
    std::vector<double> re, im;
    std::string ts = "[";
    for (std::size_t t = 0; t < targets.size(); ++t) {
      ts += std::string(t ? "," : "") + "\"" + targets[t] + "\"";
      re.push_back(amps[targets[t]].real());
      im.push_back(amps[targets[t]].imag());
    }
    man.add("{\"name\":\"" + name + "\",\"type\":\"cut\",\"n\":" + std::to_string(n) + ",\"block_a\":" +
            qlist(plan.block_a) + ",\"block_b\":" + qlist(plan.block_b) + ",\"crossing_gates\":" + qlist(ca) +
            ",\"branch_count\":" + std::to_string(plan.branch_count) + ",\"targets\":" + ts + "],\"re\":" +
            dlist(re) + ",\"im\":" + dlist(im) + "}");
  }
  man.write(dir + "/manifest_cut.json");
  return 0;
}

// Like-for-like CPU timing: the reference's own run() body
// (simulator.hpp:147-159: fuse_circuit, then StateVector::apply_gate per
// block with opts.kernel_options()) on ONE resident state, so a step excludes
// the per-run() 2^n allocation + single-threaded zero fill (statevector.hpp:139)
// and the final-state copy (simulator.hpp:163) -- as bench.py's `value`
// excludes the device allocation.  A step = the next `per_step` gates of the
// circuit (cyclic), fused and applied.  Prints one JSON line for the
// allocation and one per step.
//   ref_driver bench_steps random|qft <n> <d|input> <seed> <per_step> <steps> <fusion0|1>
int bench_steps(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: ref_driver bench_steps random|qft <n> <d|input> <seed> <per_step> <steps> <fusion>\n");
    return 2;
  }
  const std::string kind = argv[2];
  const std::uint32_t n = std::stoul(argv[3]);
  const std::uint64_t a3 = std::stoull(argv[4]), seed = std::stoull(argv[5]);
  const std::size_t per = std::stoull(argv[6]);
  const int steps = std::stoi(argv[7]);
  const bool fusion = std::stoi(argv[8]) != 0;
  Program full = kind == "qft" ? oraclegen::gen_qft(n, a3) : gen_random_circuit(n, static_cast<std::uint32_t>(a3), seed);
  SimOptions o;
  o.fusion_enabled = fusion;
  auto t0 = std::chrono::steady_clock::now();
  StateVector sv(n);
  auto t1 = std::chrono::steady_clock::now();
  std::printf("{\"alloc_seconds\":%.6f,\"threads\":%d}\n", std::chrono::duration<double>(t1 - t0).count(),
              omp_get_max_threads());
  std::fflush(stdout);
  std::size_t next = 0;
  for (int s = 0; s < steps; ++s) {
    Program p(n, 0);
    for (std::size_t k = 0; k < per; ++k, next = (next + 1) % full.body.size()) p.body.push_back(full.body[next]);
    auto a = std::chrono::steady_clock::now();
    Program prepared = fusion ? fuse_circuit(p, o.max_fused_qubits) : p;
    std::size_t passes = 0;
    for (const auto& ins : prepared.body)
      if (auto* g = std::get_if<GateOp>(&ins)) {
        sv.apply_gate(g->gate, o.kernel_options());
        ++passes;
      }
    auto b = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(b - a).count();
    std::printf("{\"gates\":%zu,\"passes\":%zu,\"seconds\":%.6f,\"threads\":%d,\"host_GBps\":%.2f}\n", per, passes,
                sec, omp_get_max_threads(), 32.0 * std::ldexp(1.0, static_cast<int>(n)) * passes / sec / 1e9);
    std::fflush(stdout);
  }
  std::printf("{\"checksum\":%.17g}\n", probability_checksum(sv));
  return 0;
}

// BASELINE.md section 4 CPU baselines, full runs through the public API:
//   config1: GHZ(20) and QFT(20): run() + probabilities(), fusion on and off
//   config2: gen_random_circuit(28, 20, 424242): run(), fusion on and off
//   config5: HEA(24, 10): expectation() and run(p, {seed}, 10^6) for seeds 0..9
// One JSON line per measurement (seconds, gates, gates/s, fused passes, host
// bandwidth 32 * 2^n * passes / t).
//   ref_driver bench_config config1|config2|config5
int bench_config(const std::string& which) {
  auto clock = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  auto passes_of = [](const Program& p, bool fusion) {
    return fusion ? fuse_circuit(p, 3).body.size() : p.body.size();
  };
  auto line = [&](const std::string& name, const Program& p, bool fusion, double sec, const std::string& extra) {
    const std::size_t passes = passes_of(p, fusion);
    std::printf("{\"config\":\"%s\",\"case\":\"%s\",\"n\":%u,\"fusion\":%s,\"gates\":%zu,\"passes\":%zu,"
                "\"seconds\":%.6f,\"gates_per_s\":%.3f,\"host_GBps\":%.2f,\"threads\":%d%s}\n",
                which.c_str(), name.c_str(), p.qubit_count, fusion ? "true" : "false", p.body.size(), passes, sec,
                p.body.size() / sec, 32.0 * std::ldexp(1.0, static_cast<int>(p.qubit_count)) * passes / sec / 1e9,
                omp_get_max_threads(), extra.c_str());
    std::fflush(stdout);
  };
  if (which == "config1") {
    for (int f = 1; f >= 0; --f)
      for (int w = 0; w < 2; ++w) {
        Program p = w == 0 ? oraclegen::gen_ghz(20) : oraclegen::gen_qft(20, 0x5a5a5);
        SimOptions o;
        o.fusion_enabled = f != 0;
        auto a = clock();
        RunResult rr = run(p, o, 0);
        auto probs = rr.final_state->probabilities();
        auto b = clock();
        line(w == 0 ? "ghz20" : "qft20", p, f != 0, secs(a, b),
             ",\"includes\":\"run()+probabilities()\",\"p_last\":" + g17(probs.back()));
      }
    return 0;
  }
  if (which == "config2") {
    Program p = gen_random_circuit(28, 20, 424242);
    for (int f = 1; f >= 0; --f) {
      SimOptions o;
      o.fusion_enabled = f != 0;
      auto a = clock();
      RunResult rr = run(p, o, 0);
      auto b = clock();
      line("random28", p, f != 0, secs(a, b),
           ",\"includes\":\"run()\",\"checksum\":" + g17(probability_checksum(*rr.final_state)));
    }
    return 0;
  }
  if (which == "config5") {
    Program p = oraclegen::gen_hea(24, 10, 2024);
    PauliOperator h = oraclegen::hea_hamiltonian(24);
    auto a = clock();
    const double e = expectation(p, h);
    auto b = clock();
    line("hea24_expectation", p, false, secs(a, b),
         ",\"includes\":\"expectation() (" + std::to_string(h.terms().size()) + " terms)\",\"value\":" + g17(e));
    Program q = p;
    q.cbit_count = 24;
    for (std::uint32_t k = 0; k < 24; ++k) q.measure(k, k);
    for (std::uint64_t seed = 0; seed < 10; ++seed) {
      SimOptions o;
      o.seed = seed;
      auto c = clock();
      RunResult rr = run(q, o, 1000000);
      auto d = clock();
      line("hea24_sample_seed" + std::to_string(seed), p, false, secs(c, d),
           ",\"includes\":\"run(p, {seed}, 1e6 shots) incl. evolution and sampling\",\"keys\":" +
               std::to_string(rr.counts.size()));
    }
    return 0;
  }
  std::fprintf(stderr, "bench_config: unknown %s\n", which.c_str());
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && std::strcmp(argv[1], "bench_steps") == 0) return bench_steps(argc, argv);
  if (argc >= 3 && std::strcmp(argv[1], "golden_cut") == 0) return golden_cut(argv[2]);
  if (argc >= 3 && std::strcmp(argv[1], "bench_config") == 0) return bench_config(argv[2]);
  if (argc >= 3 && std::strcmp(argv[1], "golden") == 0) return golden(argv[2]);
  if (argc >= 3 && std::strcmp(argv[1], "golden_big") == 0) return golden_big(argv[2]);
  if (argc >= 3 && std::strcmp(argv[1], "golden_huge") == 0) {
    std::vector<std::string> which(argv + 3, argv + argc);
    if (which.empty()) which = {"random28", "qft30", "random30"};
    return golden_huge(argv[2], which);
  }
  if (argc >= 2 && std::strcmp(argv[1], "bench") == 0) return bench(argc, argv);
  std::fprintf(stderr, "usage: ref_driver golden <dir> | golden_big <dir> | bench ...\n");
  return 2;
}
