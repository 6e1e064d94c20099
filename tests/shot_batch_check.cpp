// Cross-check of the shot-batched executor (qforge facade, simulator.hpp /
// noise.hpp) against the per-shot executor: identical counts for the same
// seed, final states within 1e-12.  TEST INFRASTRUCTURE: built by
// `make -C paper_2212_14201_b200/csrc droptests`, run by test_dropin_gpu.py.
#include <cstdio>
#include <cstdlib>
#include <qforge/qforge.hpp>

using namespace qforge;

static int failures = 0;

static void compare(const char* name, const RunResult& a, const RunResult& b) {
  if (a.counts != b.counts) {
    std::printf("FAIL %s: counts differ\n", name);
    ++failures;
  }
  const auto x = a.final_state->amplitudes();
  const auto y = b.final_state->amplitudes();
  double d = 0;
  for (std::size_t i = 0; i < x.size(); ++i) d = std::max(d, std::abs(x[i] - y[i]));
  if (d > 1e-12) {
    std::printf("FAIL %s: final states differ by %g\n", name, d);
    ++failures;
  }
  std::printf("%s: %zu keys, max |dpsi| %.3g\n", name, a.counts.size(), d);
}

template <class F>
static void both(const char* name, F run_it) {
  unsetenv("QSB_NO_SHOT_BATCH");
  RunResult batched = run_it();
  setenv("QSB_NO_SHOT_BATCH", "1", 1);
  RunResult per_shot = run_it();
  unsetenv("QSB_NO_SHOT_BATCH");
  compare(name, batched, per_shot);
}

int main() {
  // mid-circuit measurement + reuse + classical assignment
  Program p(5, 4);
  p.add(GateKind::H, {0}).add(GateKind::RY, {1}, {0.7}).add(GateKind::CNOT, {0, 2});
  p.measure(2, 0);
  p.add(GateKind::RX, {2}, {1.1}).add(GateKind::CNOT, {1, 3}).add(GateKind::H, {4});
  p.measure(3, 1);
  p.add(GateKind::U3, {0}, {0.3, 0.2, 0.1}).add(GateKind::CZ, {0, 4});
  p.measure(0, 2);
  p.measure(4, 3);
  SimOptions o;
  o.seed = 99;
  both("mid-circuit", [&] { return run(p, o, 3000); });

  // noise: 1- and 2-qubit channels, restricted rules, readout confusion
  NoiseModel nm;
  nm.add(GateKind::H, make_channel(ChannelFamily::Depolarizing, 0.2));
  nm.add(GateKind::RX, make_channel(ChannelFamily::Damping, 0.3));
  nm.add(GateKind::CNOT, make_decoherence_channel({1.0, 20.0, 15.0}), std::vector<std::uint32_t>{0, 2});
  KrausChannel two;  // 2-qubit channel: identity or a two-qubit phase flip
  CMatrix id = CMatrix::Identity(4, 4), zz = CMatrix::Zero(4, 4);
  for (int i = 0; i < 4; ++i) zz(i, i) = (i == 0 || i == 3) ? 1.0 : -1.0;
  two.ops = {id * cdouble(std::sqrt(0.8), 0), zz * cdouble(std::sqrt(0.2), 0)};
  nm.add(GateKind::CZ, two);
  nm.set_readout(3, {0.05, 0.1});
  nm.set_readout(0, {0.02, 0.0});
  both("noisy", [&] { return run_noisy(p, nm, o, 4000); });

  // control flow in shot batches: divergent branches (gates on subsets of the
  // shots, incl. 2- and 3-qubit operands), nested QIF, repeat-until-success
  // QWHILE, measurement inside branches, classical assignments
  const Program cf = parse_ir(R"(QINIT 5
CREG 5
H q[0]
RY q[1],(0.9)
MEASURE q[0],c[0]
QIF c[0] == 1
  X q[2]
  CNOT q[1],q[3]
  MEASURE q[1],c[1]
  QIF c[1]
    TOFFOLI q[1],q[2],q[4]
  ELSE
    CONTROL q[2]
    RX q[4],(0.4)
    ENDCONTROL
  ENDQIF
ELSE
  RY q[2],(1.3)
  CZ q[0],q[2]
ENDQIF
c[3] = 0
QWHILE c[3] == 0
  H q[3]
  MEASURE q[3],c[3]
  c[4] = c[4] + 1
ENDQWHILE
U3 q[4],(0.3,0.2,0.1)
MEASURE q[2],c[2]
MEASURE q[4],c[1]
)");
  both("control-flow", [&] { return run(cf, o, 3000); });
  SimOptions o2;
  o2.seed = 4242;
  both("control-flow-seed2", [&] { return run(cf, o2, 1500); });
  both("control-flow-noisy", [&] { return run_noisy(cf, nm, o, 2500); });

  std::printf(failures ? "FAILED\n" : "PASSED\n");
  return failures ? 1 : 0;
}
