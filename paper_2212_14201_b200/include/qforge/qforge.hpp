// qforge drop-in (B200 backend): umbrella header for the simulation path.
// Link with libqsb.so (paper_2212_14201_b200/libqsb.so); include paths:
//   -I<repo>/include -I<repo>/paper_2212_14201_b200/include [-I<eigen or third_party/eigen_lite>]
#pragma once

#include "qforge/bench.hpp"
#include "qforge/circuit.hpp"
#include "qforge/error.hpp"
#include "qforge/fusion.hpp"
#include "qforge/ir.hpp"
#include "qforge/gates.hpp"
#include "qforge/linalg.hpp"
#include "qforge/noise.hpp"
#include "qforge/pathsum.hpp"
#include "qforge/pauli.hpp"
#include "qforge/rng.hpp"
#include "qforge/simulator.hpp"
#include "qforge/statevector.hpp"
#include "qforge/variational.hpp"
