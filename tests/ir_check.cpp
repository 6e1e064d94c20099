// Test infrastructure: runs parse_ir / emit_ir over a corpus and prints a
// canonical transcript.  Compiled twice from this one source -- against the
// reference headers (oracle/Makefile: oracle/_ref/ir_check_ref) and against
// the drop-in facade (csrc/Makefile facadechecks: build/droptest/ir_check) --
// so the two transcripts must be identical (tests/test_ir_cpu.py).
//
// Corpus format: cases separated by lines "=== <name>"; everything up to the
// next separator is the program text ("\\t" = tab, a trailing "\\r" = CRLF
// line ending, a line "\\EOF" ends the case without a final newline).
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include <qforge/circuit.hpp>
#include <qforge/error.hpp>
#include <qforge/ir.hpp>

namespace {

struct Case {
  std::string name, text;
};

std::vector<Case> load(const std::string& path) {
  std::ifstream f(path);
  std::vector<Case> cases;
  std::string line;
  bool open = false;
  while (std::getline(f, line)) {
    if (line.rfind("=== ", 0) == 0) {
      cases.push_back({line.substr(4), ""});
      open = true;
      continue;
    }
    if (!open) continue;
    std::string& t = cases.back().text;
    for (std::size_t k; (k = line.find("\\t")) != std::string::npos;) line.replace(k, 2, "\t");
    if (line == "\\EOF") {
      if (!t.empty() && t.back() == '\n') t.pop_back();
      open = false;
      continue;
    }
    if (line.size() >= 2 && line.compare(line.size() - 2, 2, "\\r") == 0) {
      t += line.substr(0, line.size() - 2) + "\r\n";
      continue;
    }
    t += line + "\n";
  }
  return cases;
}

std::string transcript(const std::string& text) {
  std::ostringstream o;
  try {
    const qforge::Program p = qforge::parse_ir(text);
    const std::string e = qforge::emit_ir(p);
    o << "OK qubits=" << p.qubit_count << " cbits=" << p.cbit_count << " instructions=" << p.body.size() << "\n" << e;
    // round trip: the emitted text parses back to an equal program and emits identically
    const qforge::Program p2 = qforge::parse_ir(e);
    o << "roundtrip " << ((qforge::emit_ir(p2) == e && p2 == p) ? "ok" : "MISMATCH") << "\n";
  } catch (const qforge::ParseError& err) {
    o << "ParseError kind=" << qforge::parse_error_kind_name(err.kind) << " line=" << err.line
      << " column=" << err.column << "\n" << err.what() << "\n";
  } catch (const std::exception& err) {
    o << "other error: " << err.what() << "\n";
  }
  return o.str();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s corpus.txt | --files a.oir b.oir ...\n", argv[0]);
    return 2;
  }
  if (std::string(argv[1]) == "--files") {
    for (int i = 2; i < argc; ++i) {
      std::ifstream f(argv[i]);
      std::stringstream ss;
      ss << f.rdbuf();
      std::string name = argv[i];
      name = name.substr(name.find_last_of('/') + 1);
      std::cout << "=== " << name << "\n" << transcript(ss.str());
    }
    return 0;
  }
  for (const Case& c : load(argv[1])) std::cout << "=== " << c.name << "\n" << transcript(c.text);
  return 0;
}
