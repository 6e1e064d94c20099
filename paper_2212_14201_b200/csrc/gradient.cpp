// Parameter gradients of <psi(theta)|H|psi(theta)> by adjoint differentiation.
//
// The reference evaluates gradient() with the parameter-shift rule: two full
// expectation() runs per parameter slot, each building a fresh state and
// copying it once per Pauli term (variational.hpp:33-47, 139-155).  For the
// rotation gates a slot can hold (RX/RY/RZ, ParamCircuit::add_param) the shift
// rule is the exact derivative, so the same numbers come from one forward run
// and one backward sweep over resident states:
//   psi  = U_G ... U_1 |0>                 (tile passes)
//   lam  = H psi                            (one axpy pass per Pauli term)
//   for k = G..1:  if gate k is a slot:  dE/dtheta_k = Im <lam| P_k |psi>
//                  psi <- U_k^dag psi,  lam <- U_k^dag lam
// with R(theta) = exp(-i theta P / 2) up to a global phase (which does not
// change E), P_k the rotation's Pauli.  Cost: 2 per-gate passes per gate plus
// one cross-product read per slot, instead of 2 x (circuit + #terms) passes
// per slot.
#include <cmath>
#include <cstring>

#include "gates.hpp"
#include "kernels.hpp"
#include "plan.hpp"

namespace qsb {

namespace {
struct StateBuf {  // a second resident vector sharing the state's stream
  double2* p = nullptr;
  int dev = 0;
  StateBuf(uint64_t n, int device) : dev(device) {
    DeviceGuard dg(device);
    if (cudaMalloc(&p, n * sizeof(double2)) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw MemoryError("cannot allocate the adjoint state for gradient()");
    }
  }
  ~StateBuf() {
    DeviceGuard dg(dev);
    cudaFree(p);
  }
};
}  // namespace

void gradient_adjoint(State& s, const qs_gate* gates, uint64_t count, const uint64_t* slots, uint64_t nslots,
                      const std::vector<uint64_t>& xm, const std::vector<uint64_t>& zm, const std::vector<int>& ny,
                      const double* coeffs, double* out) {
  const uint32_t n = s.n;
  std::vector<int64_t> slot_of(count, -1);
  for (uint64_t i = 0; i < nslots; ++i) {
    if (slots[i] >= count) throw ValidationError("parameter slot outside the gate list");
    const qs_gate& g = gates[slots[i]];
    if ((g.kind != QS_RX && g.kind != QS_RY && g.kind != QS_RZ) || g.num_controls)
      throw ValidationError("gradient slots must be uncontrolled RX / RY / RZ gates");
    slot_of[slots[i]] = static_cast<int64_t>(i);
  }
  // forward: psi = U |0>
  auto plan = cached_plan(n, gates, count, QS_PLAN_DEFAULT, 3);
  execute_plan_from_basis(s, *plan, 0);
  // lam = H psi
  StateBuf lam(s.size, s.device);
  QSB_CUDA(cudaMemsetAsync(lam.p, 0, s.size * sizeof(double2), s.stream));
  for (size_t t = 0; t < xm.size(); ++t) {
    double fr = coeffs[2 * t], fi = coeffs[2 * t + 1];
    for (int k = 0; k < (ny[t] & 3); ++k) {  // times i^#Y
      const double r2 = -fi, i2 = fr;
      fr = r2;
      fi = i2;
    }
    pauli_axpy(s, lam.p, s.amps, xm[t], zm[t], fr, fi);
  }
  // backward sweep
  State lstate;  // view of lam for the per-gate kernels
  lstate.n = s.n;
  lstate.device = s.device;
  lstate.size = s.size;
  lstate.amps = lam.p;
  lstate.stream = s.stream;
  for (uint64_t k = count; k-- > 0;) {
    const qs_gate& g = gates[k];
    if (slot_of[k] >= 0) {
      const uint32_t q = g.targets[0];
      const uint64_t x = (g.kind == QS_RZ) ? 0 : (1ull << q);
      const uint64_t z = (g.kind == QS_RX) ? 0 : (1ull << q);
      double v[2];  // <lam| P |psi> / i^#Y  (Y = i X Z)
      pauli_cross(s, s.amps, lam.p, s.size, x, z, v);
      double re = v[0], im = v[1];
      if (g.kind == QS_RY) {  // times i
        const double r2 = -im;
        im = re;
        re = r2;
      }
      out[slot_of[k]] = g.dagger ? -im : im;  // R^dag(theta) = R(-theta)
    }
    if (k == 0) break;
    qs_gate inv = g;
    inv.dagger = g.dagger ? 0 : 1;
    const Op op = lower_gate(inv, n, false);
    launch_op(s, op);
    launch_op(lstate, op);
  }
  lstate.amps = nullptr;  // not owned
  s.sync();
}

}  // namespace qsb
