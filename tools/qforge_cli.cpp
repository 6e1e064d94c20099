// qforge command line (`qforge run|bench`) on the B200
// backend.  Mirrors the reference CLI's run / bench subcommands
// (tools/qforge.cpp:94-134, 180-208): same options, output lines and exit
// codes; written against the public qforge API only, so the same source also
// builds against the reference headers (oracle/Makefile: qforge_cli_ref) and
// the two binaries are compared in tests/test_cli_gpu.py.  The reference's
// compile / draw subcommands and the path backend belong to components outside
// this backend (transpiler, drawing, path-sum) and report exit code 5.
//
// Exit codes: 0 success, 1 usage, 2 file I/O, 3 parse failure, 4 invalid
// input, 5 backend failure.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include <qforge/qforge.hpp>

namespace {

enum Exit { kOk = 0, kUsage = 1, kIo = 2, kParse = 3, kInvalid = 4, kBackend = 5 };

struct Usage {
  std::string what;
};
struct Io {
  std::string what;
};

const char* kHelp =
    "usage: qforge run FILE [--backend statevector|noisy] [--shots N] [--seed S]\n"
    "                       [--workers W] [--opt fusion,peephole|none] [--noise FILE]\n"
    "       qforge bench [--qubits N[,N...]] [--layers L] [--seed S] [--backend B]\n"
    "                    [--opt fusion,peephole|none]\n"
    "Exit codes: 0 success, 1 usage, 2 file I/O, 3 parse failure,\n"
    "4 invalid input, 5 backend failure.\n";

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Io{"cannot open '" + path + "' for reading"};
  std::ostringstream s;
  s << in.rdbuf();
  if (in.bad()) throw Io{"error while reading '" + path + "'"};
  return s.str();
}

std::uint64_t as_u64(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0' || v[0] == '-') throw Usage{"invalid value '" + v + "' for " + flag};
  return x;
}

// --opt: comma list of fusion / peephole, or none
std::pair<bool, bool> opt_flags(const std::string& spec) {
  bool fusion = false, peephole = false;
  if (spec == "none") return {false, false};
  std::stringstream ss(spec);
  for (std::string item; std::getline(ss, item, ',');) {
    if (item == "fusion") fusion = true;
    else if (item == "peephole") peephole = true;
    else if (!item.empty())
      throw qforge::ValidationError("unknown --opt item '" + item + "' (expected fusion, peephole, or none)");
  }
  return {fusion, peephole};
}

// --name value pairs after the subcommand; positional arguments collected
struct Args {
  std::map<std::string, std::string> opts;
  std::vector<std::string> pos;
};
Args parse_args(int argc, char** argv, int from, const std::vector<std::string>& known) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string s = argv[i];
    if (s == "-h" || s == "--help") throw Usage{""};
    if (s.rfind("--", 0) == 0) {
      std::string name = s, value;
      if (const auto eq = s.find('='); eq != std::string::npos) {
        name = s.substr(0, eq);
        value = s.substr(eq + 1);
      } else {
        if (i + 1 >= argc) throw Usage{name + " needs a value"};
        value = argv[++i];
      }
      bool ok = false;
      for (const auto& k : known) ok = ok || k == name;
      if (!ok) throw Usage{"unknown option " + name};
      a.opts[name] = value;
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

int cmd_run(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2, {"--backend", "--shots", "--seed", "--workers", "--opt", "--noise",
                                             "--target", "--budget"});
  if (a.pos.size() != 1) throw Usage{"run needs exactly one circuit file"};
  auto get = [&](const char* k, const char* d) { return a.opts.count(k) ? a.opts.at(k) : std::string(d); };
  const std::string backend = get("--backend", "statevector");
  qforge::Program p = qforge::parse_ir(slurp(a.pos[0]));
  const auto [fusion, peephole] = opt_flags(get("--opt", "none"));
  (void)peephole;  // the peephole pass is a compiler optimisation outside this backend
  qforge::SimOptions o;
  o.seed = as_u64("--seed", get("--seed", "0"));
  o.workers = static_cast<int>(as_u64("--workers", get("--workers", "0")));
  o.fusion_enabled = fusion;
  const std::uint64_t shots = as_u64("--shots", get("--shots", "1024"));
  if (backend == "path") {
    std::fprintf(stderr, "error: the path backend (path-sum amplitudes) is not part of the B200 backend\n");
    return kBackend;
  }
  if (shots == 0) throw qforge::ValidationError("--shots must be at least 1 for backend '" + backend + "'");
  std::map<std::string, std::uint64_t> counts;
  if (backend == "statevector") {
    counts = qforge::run(p, o, shots).counts;
  } else if (backend == "noisy") {
    if (!a.opts.count("--noise")) throw qforge::ValidationError("the noisy backend needs --noise <config file>");
    const qforge::NoiseModel nm = qforge::parse_noise_config(slurp(a.opts.at("--noise")));
    counts = qforge::run_noisy(p, nm, o, shots).counts;
  } else {
    throw qforge::ValidationError("unknown --backend '" + backend + "' (expected statevector, noisy, or path)");
  }
  for (const auto& [bits, n] : counts) std::printf("%s %llu\n", bits.c_str(), static_cast<unsigned long long>(n));
  return kOk;
}

int cmd_bench(int argc, char** argv) {
  const Args a = parse_args(argc, argv, 2, {"--qubits", "--layers", "--seed", "--backend", "--opt"});
  if (!a.pos.empty()) throw Usage{"bench takes no positional arguments"};
  auto get = [&](const char* k, const char* d) { return a.opts.count(k) ? a.opts.at(k) : std::string(d); };
  std::vector<std::uint32_t> qubits;
  std::stringstream ss(get("--qubits", "20"));
  for (std::string item; std::getline(ss, item, ',');)
    qubits.push_back(static_cast<std::uint32_t>(as_u64("--qubits", item)));
  const auto layers = static_cast<std::uint32_t>(as_u64("--layers", get("--layers", "10")));
  const std::uint64_t seed = as_u64("--seed", get("--seed", "0"));
  const auto [fusion, peephole] = opt_flags(get("--opt", "fusion,peephole"));
  const qforge::Backend backend = qforge::backend_from_name(get("--backend", "statevector"));
  std::printf("qubits\tlayers\tbuild_s\tcompile_s\texecute_s\tgates_before\tgates_after\tchecksum\n");
  for (std::uint32_t n : qubits) {
    qforge::BenchSpec spec;
    spec.qubits = n;
    spec.layers = layers;
    spec.seed = seed;
    spec.backend = backend;
    spec.fusion = fusion;
    spec.peephole = peephole;
    const qforge::BenchResult r = qforge::run_bench(spec);
    std::printf("%u\t%u\t%.6f\t%.6f\t%.6f\t%llu\t%llu\t%.17g\n", n, layers, r.build_seconds, r.compile_seconds,
                r.execute_seconds, static_cast<unsigned long long>(r.gates_before),
                static_cast<unsigned long long>(r.gates_after), r.checksum);
  }
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string sub = argc > 1 ? argv[1] : "";
    if (sub == "run") return cmd_run(argc, argv);
    if (sub == "bench") return cmd_bench(argc, argv);
    if (sub == "compile" || sub == "draw") {
      std::fprintf(stderr, "error: '%s' (transpiler / drawing) is not part of the B200 backend\n", sub.c_str());
      return kBackend;
    }
    if (sub == "-h" || sub == "--help") {
      std::fputs(kHelp, stdout);
      return kOk;
    }
    throw Usage{sub.empty() ? "a subcommand is required" : "unknown subcommand '" + sub + "'"};
  } catch (const Usage& u) {
    if (!u.what.empty()) std::fprintf(stderr, "error: %s\n", u.what.c_str());
    std::fputs(kHelp, stderr);
    return u.what.empty() ? kOk : kUsage;
  } catch (const Io& e) {
    std::fprintf(stderr, "error: %s\n", e.what.c_str());
    return kIo;
  } catch (const qforge::ParseError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kParse;
  } catch (const qforge::ValidationError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kInvalid;
  } catch (const qforge::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kBackend;
  }
}
