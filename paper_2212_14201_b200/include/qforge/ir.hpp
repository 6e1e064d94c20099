// qforge drop-in (B200 backend): the line-oriented program text format.
//
// Same grammar, diagnostics and round-trip guarantee as the reference's
// ir.hpp (parse_ir / emit_ir, ir.hpp:135-140 and :319-707); written
// independently for this backend.  One instruction per line:
//   QINIT n, CREG n (headers, QINIT first)
//   <MNEMONIC> q[i],q[j],(p1,p2)   gate; CUSTOM takes (re,im,...) row-major
//   DAGGER ... ENDDAGGER           adjoint of the enclosed gates
//   CONTROL q[i] ... ENDCONTROL    one more (leading) control on the enclosed gates
//   MEASURE q[i],c[j]
//   QIF expr / ELSE / ENDQIF,  QWHILE expr / ENDQWHILE,  c[i] = expr
// `#` starts a comment.  Numbers are written with 17 significant digits, so
// emit -> parse is bit-exact.  Errors are ParseError{kind, line, column}.
#pragma once

#include <cctype>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <string_view>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/error.hpp"

namespace qforge {

namespace detail::irtext {

inline bool space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }
inline bool digit(char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; }

inline std::string number(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// ---- writer ---------------------------------------------------------------
inline void write_expr(const ClassicalExpr& e, bool nested, std::string& o) {
  switch (e.kind()) {
    case ClassicalExpr::Kind::Constant: o += std::to_string(e.constant_value()); break;
    case ClassicalExpr::Kind::CBit: o += "c[" + std::to_string(e.cbit_index()) + "]"; break;
    case ClassicalExpr::Kind::Binary:  // operands always bracketed below the top
      if (nested) o += '(';
      write_expr(e.lhs(), true, o);
      o += binop_name(e.op());
      write_expr(e.rhs(), true, o);
      if (nested) o += ')';
      break;
  }
}

inline std::string qref(std::uint32_t q) { return "q[" + std::to_string(q) + "]"; }

inline void write_gate(const Gate& g, std::string& o) {
  for (std::uint32_t c : g.controls) o += "CONTROL " + qref(c) + "\n";
  if (g.dagger) o += "DAGGER\n";
  o += gate_name(g.kind);
  o += ' ';
  for (std::size_t i = 0; i < g.targets.size(); ++i) o += (i ? "," : "") + qref(g.targets[i]);
  std::vector<double> nums;
  if (g.kind == GateKind::Custom) {
    for (Eigen::Index r = 0; r < g.custom->rows(); ++r)
      for (Eigen::Index c = 0; c < g.custom->cols(); ++c) {
        nums.push_back((*g.custom)(r, c).real());
        nums.push_back((*g.custom)(r, c).imag());
      }
  } else {
    nums = g.params;
  }
  if (!nums.empty() || g.kind == GateKind::Custom) {
    o += ",(";
    for (std::size_t i = 0; i < nums.size(); ++i) o += (i ? "," : "") + number(nums[i]);
    o += ')';
  }
  o += '\n';
  if (g.dagger) o += "ENDDAGGER\n";
  for (std::size_t i = 0; i < g.controls.size(); ++i) o += "ENDCONTROL\n";
}

inline void write_body(const std::vector<Instruction>& body, std::string& o) {
  for (const Instruction& ins : body) {
    std::visit(
        [&](const auto& x) {
          using T = std::decay_t<decltype(x)>;
          if constexpr (std::is_same_v<T, GateOp>) {
            write_gate(x.gate, o);
          } else if constexpr (std::is_same_v<T, MeasureOp>) {
            o += "MEASURE " + qref(x.qubit) + ",c[" + std::to_string(x.cbit) + "]\n";
          } else if constexpr (std::is_same_v<T, IfOp>) {
            o += "QIF ";
            write_expr(x.condition, false, o);
            o += '\n';
            write_body(x.then_body->body, o);
            if (x.else_body) {
              o += "ELSE\n";
              write_body(x.else_body->body, o);
            }
            o += "ENDQIF\n";
          } else if constexpr (std::is_same_v<T, WhileOp>) {
            o += "QWHILE ";
            write_expr(x.condition, false, o);
            o += '\n';
            write_body(x.body->body, o);
            o += "ENDQWHILE\n";
          } else {  // AssignOp
            o += "c[" + std::to_string(x.cbit) + "] = ";
            write_expr(x.expr, false, o);
            o += '\n';
          }
        },
        ins);
  }
}

// ---- reader ---------------------------------------------------------------
[[noreturn]] inline void fail(ParseErrorKind k, std::uint32_t line, std::size_t col, const std::string& msg) {
  throw ParseError(k, line, static_cast<std::uint32_t>(col), msg);
}

// Expression over one line's tail, `col0` = 0-based column of its first
// character.  Binding, loosest first: || && ^ (== !=) (< >) (+ -) (* /), all
// left-associative; operands: integers (optionally negative), c[i], (...).
class ExprReader {
 public:
  ExprReader(std::string_view s, std::uint32_t line, std::size_t col0) : s_(s), line_(line), col0_(col0) {}

  ClassicalExpr read() {
    ClassicalExpr e = climb(1);
    blanks();
    if (i_ != s_.size()) error("unexpected trailing text in expression", i_);
    return e;
  }

 private:
  std::string_view s_;
  std::size_t i_ = 0;
  std::uint32_t line_;
  std::size_t col0_;

  [[noreturn]] void error(const std::string& m, std::size_t at) const {
    fail(ParseErrorKind::Syntax, line_, col0_ + at + 1, m);
  }
  void blanks() {
    while (i_ < s_.size() && space(s_[i_])) ++i_;
  }
  // (operator, binding level, width) at the cursor; level 0 = none
  struct Op {
    BinOp op;
    int level;
    std::size_t width;
  };
  Op look() {
    blanks();
    const std::string_view r = s_.substr(i_);
    static constexpr struct {
      const char* text;
      BinOp op;
      int level;
    } table[] = {{"||", BinOp::Or, 1}, {"&&", BinOp::And, 2}, {"==", BinOp::Eq, 4}, {"!=", BinOp::Ne, 4},
                 {"^", BinOp::Xor, 3},  {"<", BinOp::Lt, 5},   {">", BinOp::Gt, 5},   {"+", BinOp::Add, 6},
                 {"-", BinOp::Sub, 6},  {"*", BinOp::Mul, 7},  {"/", BinOp::Div, 7}};
    for (const auto& t : table) {
      const std::string_view tx(t.text);
      if (r.substr(0, tx.size()) == tx) return {t.op, t.level, tx.size()};
    }
    return {BinOp::Add, 0, 0};
  }
  ClassicalExpr climb(int min_level) {
    ClassicalExpr acc = operand();
    for (Op o = look(); o.level && o.level >= min_level; o = look()) {
      i_ += o.width;
      ClassicalExpr rhs = climb(o.level + 1);
      acc = ClassicalExpr::binary(o.op, std::move(acc), std::move(rhs));
    }
    return acc;
  }
  ClassicalExpr operand() {
    blanks();
    if (i_ >= s_.size()) error("expected an operand", i_);
    const char c = s_[i_];
    if (c == '(') {
      ++i_;
      ClassicalExpr e = climb(1);
      blanks();
      if (i_ >= s_.size() || s_[i_] != ')') error("expected ')'", i_);
      ++i_;
      return e;
    }
    if (c == 'c' && i_ + 1 < s_.size() && s_[i_ + 1] == '[') {
      const std::size_t lb = i_ + 1, rb = s_.find(']', lb);
      if (rb == std::string_view::npos) error("expected ']'", lb);
      std::uint32_t idx = 0;
      const std::string_view digits = s_.substr(lb + 1, rb - lb - 1);
      const auto r = std::from_chars(digits.data(), digits.data() + digits.size(), idx);
      if (r.ec != std::errc() || r.ptr != digits.data() + digits.size()) error("expected a classical bit index", lb + 1);
      i_ = rb + 1;
      return ClassicalExpr::cbit(idx);
    }
    if (digit(c) || (c == '-' && i_ + 1 < s_.size() && digit(s_[i_ + 1]))) {
      std::int64_t v = 0;
      const auto r = std::from_chars(s_.data() + i_, s_.data() + s_.size(), v);
      if (r.ec != std::errc()) error("bad integer literal", i_);
      i_ = static_cast<std::size_t>(r.ptr - s_.data());
      return ClassicalExpr::constant(v);
    }
    error("expected an operand", i_);
  }
};

// Comma-separated operands at parenthesis depth 0, trimmed, with their
// 0-based offsets; an empty tail has no operands.
struct Piece {
  std::string text;
  std::size_t at;
};
inline std::vector<Piece> operands(std::string_view r) {
  std::vector<Piece> out;
  int depth = 0;
  std::size_t from = 0;
  for (std::size_t i = 0; i <= r.size(); ++i) {
    const bool cut = i == r.size() || (r[i] == ',' && depth == 0);
    if (!cut) {
      depth += r[i] == '(' ? 1 : (r[i] == ')' ? -1 : 0);
      continue;
    }
    std::size_t a = from, b = i;
    while (a < b && space(r[a])) ++a;
    while (b > a && space(r[b - 1])) --b;
    out.push_back({std::string(r.substr(a, b - a)), a});
    from = i + 1;
  }
  if (out.size() == 1 && out[0].text.empty()) out.clear();
  return out;
}

inline std::uint32_t read_count(std::string_view s, std::uint32_t line, std::size_t col, const char* what) {
  std::uint32_t v = 0;
  const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (r.ec != std::errc() || r.ptr != s.data() + s.size())
    fail(ParseErrorKind::Syntax, line, col + 1, std::string("expected ") + what);
  return v;
}

// "q[i]" / "c[i]" at 0-based column `col`
inline std::uint32_t read_ref(const std::string& s, char reg, std::uint32_t line, std::size_t col) {
  if (s.size() < 4 || s[0] != reg || s[1] != '[' || s.back() != ']')
    fail(ParseErrorKind::Syntax, line, col + 1, std::string("expected ") + reg + "[index], got '" + s + "'");
  return read_count(std::string_view(s).substr(2, s.size() - 3), line, col + 2, "a register index");
}

// An open block while reading.
struct Open {
  enum Kind { Root, Adjoint, Controlled, Then, Else, Loop } kind = Root;
  std::uint32_t line = 0;
  std::uint32_t qubit = 0;  // Controlled
  ClassicalExpr cond = ClassicalExpr::constant(0);
  std::vector<Instruction> body, then_body;
  const char* name() const {
    switch (kind) {
      case Adjoint: return "DAGGER";
      case Controlled: return "CONTROL";
      case Then:
      case Else: return "QIF";
      case Loop: return "QWHILE";
      default: return "?";
    }
  }
};

class Reader {
 public:
  Program read(const std::string& text) {
    std::uint32_t line = 0;
    std::size_t start = 0;
    while (start <= text.size()) {
      std::size_t end = text.find('\n', start);
      if (end == std::string::npos) end = text.size();
      std::string ln = text.substr(start, end - start);
      start = end + 1;
      ++line;
      if (start > text.size() && ln.empty()) break;  // after the final newline
      if (const std::size_t h = ln.find('#'); h != std::string::npos) ln.resize(h);
      while (!ln.empty() && (ln.back() == '\r' || ln.back() == ' ' || ln.back() == '\t')) ln.pop_back();
      std::size_t ind = 0;
      while (ind < ln.size() && space(ln[ind])) ++ind;
      if (ind == ln.size()) continue;
      statement(ln, ind, line);
    }
    last_line_ = line;
    if (stack_.size() > 1)
      fail(ParseErrorKind::UnterminatedBlock, stack_.back().line, 0,
           std::string(stack_.back().name()) + " block is never closed");
    if (!have_q_) fail(ParseErrorKind::Syntax, line ? line : 1, 0, "missing QINIT header");
    Program p(nq_, nc_);
    p.body = std::move(stack_.back().body);
    return p;
  }

 private:
  std::vector<Open> stack_ = std::vector<Open>(1);
  std::uint32_t nq_ = 0, nc_ = 0, last_line_ = 0;
  bool have_q_ = false, have_c_ = false, started_ = false;

  bool in_gate_block() const {
    for (const Open& o : stack_)
      if (o.kind == Open::Adjoint || o.kind == Open::Controlled) return true;
    return false;
  }
  std::vector<Instruction>& sink() { return stack_.back().body; }
  void check_qubit(std::uint32_t q, std::uint32_t line, std::size_t col1) const {
    if (q >= nq_)
      fail(ParseErrorKind::RangeError, line, col1,
           "q[" + std::to_string(q) + "] exceeds QINIT " + std::to_string(nq_));
  }
  void check_cbit(std::uint32_t c, std::uint32_t line, std::size_t col1) const {
    if (c >= nc_)
      fail(ParseErrorKind::RangeError, line, col1,
           "c[" + std::to_string(c) + "] exceeds CREG " + std::to_string(nc_));
  }
  void check_reads(const ClassicalExpr& e, const char* what, std::uint32_t line, std::size_t col1) const {
    if (e.cbits_used() > nc_)
      fail(ParseErrorKind::RangeError, line, col1,
           std::string(what) + " reads c[" + std::to_string(e.cbits_used() - 1) + "] but CREG is " +
               std::to_string(nc_));
  }
  Open pop() {
    Open o = std::move(stack_.back());
    stack_.pop_back();
    return o;
  }

  void statement(const std::string& ln, std::size_t ind, std::uint32_t line) {
    const std::string_view st = std::string_view(ln).substr(ind);
    const std::size_t col1 = ind + 1;
    if (st.substr(0, 2) == "c[") return assignment(st, ind, line);

    std::size_t w = 0;
    while (w < st.size() && !space(st[w])) ++w;
    const std::string word(st.substr(0, w));
    std::string_view tail = st.substr(w);
    while (!tail.empty() && space(tail.front())) tail.remove_prefix(1);
    const std::size_t tcol = ind + (st.size() - tail.size());  // 0-based column of the tail

    if (word == "QINIT") {
      if (have_q_) fail(ParseErrorKind::Syntax, line, col1, "duplicate QINIT");
      if (started_ || have_c_) fail(ParseErrorKind::Syntax, line, col1, "QINIT must be the first statement");
      nq_ = read_count(tail, line, tcol, "a qubit count");
      have_q_ = true;
      return;
    }
    if (word == "CREG") {
      if (!have_q_) fail(ParseErrorKind::Syntax, line, col1, "CREG requires a preceding QINIT");
      if (have_c_) fail(ParseErrorKind::Syntax, line, col1, "duplicate CREG");
      if (started_) fail(ParseErrorKind::Syntax, line, col1, "CREG must precede instructions");
      nc_ = read_count(tail, line, tcol, "a cbit count");
      have_c_ = true;
      return;
    }
    if (!have_q_) fail(ParseErrorKind::Syntax, line, col1, "QINIT must precede instructions");
    started_ = true;
    auto bare = [&]() {
      if (!tail.empty()) fail(ParseErrorKind::Syntax, line, tcol + 1, "unexpected text after " + word);
    };
    auto no_gate_block = [&]() {
      if (in_gate_block()) fail(ParseErrorKind::Syntax, line, col1, word + " not allowed inside DAGGER/CONTROL");
    };

    if (word == "DAGGER") {
      bare();
      Open o;
      o.kind = Open::Adjoint;
      o.line = line;
      stack_.push_back(std::move(o));
    } else if (word == "ENDDAGGER") {
      bare();
      if (stack_.back().kind != Open::Adjoint)
        fail(ParseErrorKind::Syntax, line, col1, "ENDDAGGER without matching DAGGER");
      Open o = pop();
      for (std::size_t k = o.body.size(); k-- > 0;) {  // (g1..gn)^dagger = gn^dagger..g1^dagger
        Gate g = std::get<GateOp>(o.body[k]).gate;
        g.dagger = !g.dagger;
        sink().push_back(GateOp{std::move(g)});
      }
    } else if (word == "CONTROL") {
      const auto ops = operands(tail);
      if (ops.size() != 1) fail(ParseErrorKind::ArityError, line, col1, "CONTROL takes exactly one qubit");
      const std::uint32_t q = read_ref(ops[0].text, 'q', line, tcol + ops[0].at);
      check_qubit(q, line, col1);
      Open o;
      o.kind = Open::Controlled;
      o.line = line;
      o.qubit = q;
      stack_.push_back(std::move(o));
    } else if (word == "ENDCONTROL") {
      bare();
      if (stack_.back().kind != Open::Controlled)
        fail(ParseErrorKind::Syntax, line, col1, "ENDCONTROL without matching CONTROL");
      Open o = pop();
      for (Instruction& ins : o.body) {
        Gate g = std::get<GateOp>(ins).gate;
        g.controls.insert(g.controls.begin(), o.qubit);
        sink().push_back(GateOp{std::move(g)});
      }
    } else if (word == "QIF" || word == "QWHILE") {
      no_gate_block();
      Open o;
      o.kind = word == "QIF" ? Open::Then : Open::Loop;
      o.line = line;
      o.cond = ExprReader(tail, line, tcol).read();
      check_reads(o.cond, "condition", line, col1);
      stack_.push_back(std::move(o));
    } else if (word == "ELSE") {
      bare();
      if (stack_.back().kind != Open::Then) fail(ParseErrorKind::Syntax, line, col1, "ELSE outside QIF");
      stack_.back().kind = Open::Else;
      stack_.back().then_body = std::move(stack_.back().body);
      stack_.back().body.clear();
    } else if (word == "ENDQIF") {
      bare();
      if (stack_.back().kind != Open::Then && stack_.back().kind != Open::Else)
        fail(ParseErrorKind::Syntax, line, col1, "ENDQIF without matching QIF");
      Open o = pop();
      const bool has_else = o.kind == Open::Else;
      IfOp op;
      op.condition = std::move(o.cond);
      Program then_p(nq_, nc_);
      then_p.body = has_else ? std::move(o.then_body) : std::move(o.body);
      op.then_body = std::make_shared<const Program>(std::move(then_p));
      if (has_else) {
        Program else_p(nq_, nc_);
        else_p.body = std::move(o.body);
        op.else_body = std::make_shared<const Program>(std::move(else_p));
      }
      sink().push_back(std::move(op));
    } else if (word == "ENDQWHILE") {
      bare();
      if (stack_.back().kind != Open::Loop) fail(ParseErrorKind::Syntax, line, col1, "ENDQWHILE without matching QWHILE");
      Open o = pop();
      WhileOp op;
      op.condition = std::move(o.cond);
      Program body(nq_, nc_);
      body.body = std::move(o.body);
      op.body = std::make_shared<const Program>(std::move(body));
      sink().push_back(std::move(op));
    } else if (word == "MEASURE") {
      no_gate_block();
      const auto ops = operands(tail);
      if (ops.size() != 2) fail(ParseErrorKind::ArityError, line, col1, "MEASURE expects q[i],c[j]");
      const std::uint32_t q = read_ref(ops[0].text, 'q', line, tcol + ops[0].at);
      const std::uint32_t c = read_ref(ops[1].text, 'c', line, tcol + ops[1].at);
      check_qubit(q, line, col1);
      check_cbit(c, line, col1);
      sink().push_back(MeasureOp{q, c});
    } else {
      gate(word, tail, tcol, line, col1);
    }
  }

  void assignment(std::string_view st, std::size_t ind, std::uint32_t line) {
    const std::size_t col1 = ind + 1;
    if (!have_q_) fail(ParseErrorKind::Syntax, line, col1, "QINIT must precede instructions");
    if (in_gate_block()) fail(ParseErrorKind::Syntax, line, col1, "assignment not allowed inside DAGGER/CONTROL");
    const std::size_t rb = st.find(']');
    if (rb == std::string_view::npos) fail(ParseErrorKind::Syntax, line, col1, "expected ']'");
    const std::uint32_t cb = read_count(st.substr(2, rb - 2), line, ind + 2, "a cbit index");
    check_cbit(cb, line, col1);
    std::size_t eq = rb + 1;
    while (eq < st.size() && space(st[eq])) ++eq;
    if (eq >= st.size() || st[eq] != '=' || (eq + 1 < st.size() && st[eq + 1] == '='))
      fail(ParseErrorKind::Syntax, line, ind + eq + 1, "expected '=' in assignment");
    ClassicalExpr rhs = ExprReader(st.substr(eq + 1), line, ind + eq + 1).read();
    check_reads(rhs, "expression", line, col1);
    sink().push_back(AssignOp{cb, std::move(rhs)});
    started_ = true;
  }

  void gate(const std::string& word, std::string_view tail, std::size_t tcol, std::uint32_t line, std::size_t col1) {
    const auto kind = gate_kind_from_name(word);
    const bool custom = word == "CUSTOM";
    if (!kind && !custom) fail(ParseErrorKind::UnknownMnemonic, line, col1, "unknown mnemonic '" + word + "'");
    auto ops = operands(tail);
    std::vector<double> nums;
    if (!ops.empty() && !ops.back().text.empty() && ops.back().text.front() == '(') {
      const Piece tuple = ops.back();
      ops.pop_back();
      if (tuple.text.back() != ')')
        fail(ParseErrorKind::Syntax, line, tcol + tuple.at + 1, "unterminated parameter tuple");
      for (const Piece& x : operands(std::string_view(tuple.text).substr(1, tuple.text.size() - 2))) {
        char* stop = nullptr;
        const double v = std::strtod(x.text.c_str(), &stop);
        if (stop == x.text.c_str() || *stop != '\0')
          fail(ParseErrorKind::Syntax, line, tcol + tuple.at + 2 + x.at, "expected a number, got '" + x.text + "'");
        nums.push_back(v);
      }
    }
    Gate g;
    for (const Piece& x : ops) {
      if (!x.text.empty() && x.text.front() == '(')
        fail(ParseErrorKind::Syntax, line, tcol + x.at + 1, "parameter tuple must come last");
      const std::uint32_t q = read_ref(x.text, 'q', line, tcol + x.at);
      check_qubit(q, line, col1);
      g.targets.push_back(q);
    }
    if (custom) {
      const std::size_t k = g.targets.size();
      if (k == 0) fail(ParseErrorKind::ArityError, line, col1, "CUSTOM needs at least one target");
      const std::size_t dim = std::size_t(1) << k;
      if (nums.size() != 2 * dim * dim)
        fail(ParseErrorKind::ArityError, line, col1,
             "CUSTOM on " + std::to_string(k) + " qubit(s) needs " + std::to_string(2 * dim * dim) +
                 " matrix numbers, got " + std::to_string(nums.size()));
      CMatrix m(dim, dim);
      for (std::size_t r = 0; r < dim; ++r)
        for (std::size_t c = 0; c < dim; ++c) m(r, c) = cdouble(nums[2 * (r * dim + c)], nums[2 * (r * dim + c) + 1]);
      g.kind = GateKind::Custom;
      g.custom = std::make_shared<const CMatrix>(std::move(m));
    } else {
      g.kind = *kind;
      if (g.targets.size() != gate_target_arity(g.kind))
        fail(ParseErrorKind::ArityError, line, col1,
             word + " expects " + std::to_string(gate_target_arity(g.kind)) + " target(s), got " +
                 std::to_string(g.targets.size()));
      if (nums.size() != gate_param_arity(g.kind))
        fail(ParseErrorKind::ArityError, line, col1,
             word + " expects " + std::to_string(gate_param_arity(g.kind)) + " parameter(s), got " +
                 std::to_string(nums.size()));
      g.params = std::move(nums);
    }
    sink().push_back(GateOp{std::move(g)});
  }
};

}  // namespace detail::irtext

// Program -> text (ir.hpp:135-140): headers, then one instruction per line.
inline std::string emit_ir(const Program& p) {
  std::string o = "QINIT " + std::to_string(p.qubit_count) + "\nCREG " + std::to_string(p.cbit_count) + "\n";
  detail::irtext::write_body(p.body, o);
  return o;
}

// Text -> Program (ir.hpp:319-707); throws ParseError.
inline Program parse_ir(const std::string& text) { return detail::irtext::Reader().read(text); }

}  // namespace qforge
