// Host front end of the drop-in boundary:
//   * OpenQASM 2.0 subset parser         qasm_parser.cpp (ParseError line/column)
//   * gate kinds and matrices            gates.cpp:40-208
//   * u4 sidecar read/write + injection  runner.cpp:129-190
//   * fusion, SWAP lowering, layering    fusion.cpp:79-190
//   * circuit generators                 generators.cpp:52-145
//   * run_circuit + its JSON record      runner.cpp:219-328, docs/run_output.schema.json
// Parse / fuse / plan / generate are host-only. run_circuit drives the GPU
// engine through its own C ABI (mpsim_gpu.h): the MPS backends through
// mpsim_gpu_execute / mpsim_gpu_apply_layer and the sampler, the statevector
// backend through statevec.cu.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "engine.h"
#include "frontend.h"
#include "mpsim_gpu.h"

namespace mpsim_gpu {
namespace fe {

using cd = std::complex<double>;

// ------------------------------------------------------------------ errors

struct ParseFailure {
  int line, column;
  std::string message;
};
thread_local int t_parse_line = 0, t_parse_col = 0;

[[noreturn]] void config_error(const std::string& m) { fail(MPSIM_EINVAL, m); }

// ------------------------------------------------------------- gate table

enum Kind { H, X, Y, Z, S, Sdg, T, Tdg, Rx, Ry, Rz, U1, U2, U3, Cx, Cz, Swap, U4 };

struct KindInfo {
  const char* name;
  int params;
  bool two;
};
constexpr KindInfo kKinds[] = {{"h", 0, false},  {"x", 0, false},   {"y", 0, false},   {"z", 0, false},
                               {"s", 0, false},  {"sdg", 0, false}, {"t", 0, false},   {"tdg", 0, false},
                               {"rx", 1, false}, {"ry", 1, false},  {"rz", 1, false},  {"u1", 1, false},
                               {"u2", 2, false}, {"u3", 3, false},  {"cx", 0, true},   {"cz", 0, true},
                               {"swap", 0, true}, {"u4", 0, true}};

bool kind_of(std::string_view name, Kind& k) {  // gate_kind_from_name: u4 is sidecar-only
  for (int i = 0; i < U4; ++i)
    if (name == kKinds[i].name) {
      k = (Kind)i;
      return true;
    }
  return false;
}

struct Mat {  // 2x2 or 4x4, row-major
  int dim = 0;
  cd a[16];
  cd& operator()(int r, int c) { return a[r * dim + c]; }
  const cd& operator()(int r, int c) const { return a[r * dim + c]; }
};

Mat mat2(cd a, cd b, cd c, cd d) {
  Mat m;
  m.dim = 2;
  m.a[0] = a, m.a[1] = b, m.a[2] = c, m.a[3] = d;
  return m;
}

Mat mul(const Mat& x, const Mat& y) {
  Mat r;
  r.dim = x.dim;
  for (int i = 0; i < x.dim; ++i)
    for (int j = 0; j < x.dim; ++j) {
      cd acc = 0.0;
      for (int k = 0; k < x.dim; ++k) acc += x(i, k) * y(k, j);
      r(i, j) = acc;
    }
  return r;
}

// (low, high) <-> (high, low) basis change of a 4x4 (gates.cpp:31-42)
Mat swap_conj(const Mat& m) {
  auto flip = [](int x) { return ((x & 1) << 1) | (x >> 1); };
  Mat r;
  r.dim = 4;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) r(i, j) = m(flip(i), flip(j));
  return r;
}

// gate_matrix_1q, gates.cpp:119-172
Mat matrix_1q(Kind k, const std::vector<double>& p) {
  const cd I(0.0, 1.0);
  const double r2 = 1.0 / std::sqrt(2.0);
  switch (k) {
    case H: return mat2(r2, r2, r2, -r2);
    case X: return mat2(0.0, 1.0, 1.0, 0.0);
    case Y: return mat2(0.0, -I, I, 0.0);
    case Z: return mat2(1.0, 0.0, 0.0, -1.0);
    case S: return mat2(1.0, 0.0, 0.0, I);
    case Sdg: return mat2(1.0, 0.0, 0.0, -I);
    case T: return mat2(1.0, 0.0, 0.0, std::exp(I * (M_PI / 4.0)));
    case Tdg: return mat2(1.0, 0.0, 0.0, std::exp(-I * (M_PI / 4.0)));
    case Rx: {
      const double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
      return mat2(c, -I * s, -I * s, c);
    }
    case Ry: {
      const double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
      return mat2(c, -s, s, c);
    }
    case Rz: return mat2(std::exp(-I * (p[0] / 2.0)), 0.0, 0.0, std::exp(I * (p[0] / 2.0)));
    case U1: return mat2(1.0, 0.0, 0.0, std::exp(I * p[0]));
    case U2:
      return mat2(r2, -std::exp(I * p[1]) * r2, std::exp(I * p[0]) * r2, std::exp(I * (p[0] + p[1])) * r2);
    case U3: {
      const double c = std::cos(p[0] / 2.0), s = std::sin(p[0] / 2.0);
      return mat2(c, -std::exp(I * p[2]) * s, std::exp(I * p[1]) * s, std::exp(I * (p[1] + p[2])) * c);
    }
    default: fail(MPSIM_EINVAL, std::string("not a one-qubit gate: ") + kKinds[k].name);
  }
}

struct Op {  // PrimOp, circuit.hpp:48-56
  Kind kind = H;
  int q0 = 0, q1 = -1;
  std::vector<double> params;
  Mat u4;  // U4 only
  bool two() const { return q1 >= 0; }
};

// gate_matrix, gates.cpp:174-208: 4x4 in the (low, high) basis
Mat matrix_of(const Op& op) {
  if (!op.two()) return matrix_1q(op.kind, op.params);
  Mat m;
  m.dim = 4;
  switch (op.kind) {
    case Cx: m(0, 0) = m(1, 1) = m(2, 3) = m(3, 2) = 1.0; break;
    case Cz: m(0, 0) = m(1, 1) = m(2, 2) = 1.0, m(3, 3) = -1.0; break;
    case Swap: m(0, 0) = m(1, 2) = m(2, 1) = m(3, 3) = 1.0; break;
    case U4: m = op.u4; break;
    default: fail(MPSIM_EINVAL, std::string("not a two-qubit gate: ") + kKinds[op.kind].name);
  }
  return op.q0 < op.q1 ? m : swap_conj(m);
}

struct Circuit {  // circuit.hpp:58-63
  int n_qubits = 0, n_clbits = 0;
  bool measure_all = false;
  std::vector<Op> ops;
};

// ------------------------------------------------------------------ parser
// A cursor over the text that scans one token at a time (identifiers,
// numbers, strings, one-char symbols and "->"); '//' comments and white
// space are skipped; every token remembers its 1-based line and column.

class QasmParser {
 public:
  explicit QasmParser(std::string_view text) : src_(text) { scan(); }

  Circuit run() {
    header();
    while (tok_.type != End) statement();
    if (qreg_.empty()) error(tok_, "no qreg declared");
    c_.measure_all = measured_whole_ || (c_.n_qubits > 0 && (int)measured_.size() == c_.n_qubits);
    return std::move(c_);
  }

 private:
  enum Type { End, Ident, Number, String, Symbol };
  struct Tok {
    Type type = End;
    std::string text;
    double value = 0.0;
    bool integer = false;
    int line = 1, col = 1;
  };

  [[noreturn]] void error(const Tok& at, const std::string& msg) { throw ParseFailure{at.line, at.col, msg}; }

  static bool is_alpha(char c) { return std::isalpha((unsigned char)c) || c == '_'; }
  static bool is_digit(char c) { return std::isdigit((unsigned char)c); }
  char at(size_t i) const { return i < src_.size() ? src_[i] : '\0'; }
  void bump() { ++pos_, ++col_; }

  void scan() {
    for (;;) {  // skip blanks and // comments
      const char c = at(pos_);
      if (pos_ >= src_.size()) break;
      if (c == '\n') {
        ++pos_, ++line_, col_ = 1;
      } else if (std::isspace((unsigned char)c)) {
        bump();
      } else if (c == '/' && at(pos_ + 1) == '/') {
        while (pos_ < src_.size() && src_[pos_] != '\n') ++pos_;
      } else {
        break;
      }
    }
    tok_ = Tok{};
    tok_.line = line_, tok_.col = col_;
    if (pos_ >= src_.size()) {
      tok_.text = "<end of input>";
      return;
    }
    const char c = src_[pos_];
    if (is_alpha(c)) {
      tok_.type = Ident;
      while (pos_ < src_.size() && (is_alpha(src_[pos_]) || is_digit(src_[pos_]))) tok_.text += src_[pos_], bump();
    } else if (is_digit(c) || (c == '.' && is_digit(at(pos_ + 1)))) {
      tok_.type = Number;
      bool dot = false, exp = false;
      for (;;) {
        const char d = at(pos_);
        if (pos_ >= src_.size()) break;
        if (is_digit(d)) {
          tok_.text += d, bump();
        } else if (d == '.' && !dot && !exp) {
          dot = true, tok_.text += d, bump();
        } else if ((d == 'e' || d == 'E') && !exp) {
          exp = true, tok_.text += d, bump();
          if (at(pos_) == '+' || at(pos_) == '-') tok_.text += src_[pos_], bump();
        } else {
          break;
        }
      }
      tok_.integer = !dot && !exp;
      tok_.value = std::strtod(tok_.text.c_str(), nullptr);
    } else if (c == '"') {
      tok_.type = String;
      bump();
      while (pos_ < src_.size() && src_[pos_] != '"') tok_.text += src_[pos_], bump();
      if (pos_ >= src_.size()) error(tok_, "unterminated string");
      bump();
    } else {
      tok_.type = Symbol;
      tok_.text = c;
      bump();
      if (c == '-' && at(pos_) == '>') tok_.text += '>', bump();
    }
  }

  Tok take() {
    Tok t = tok_;
    scan();
    return t;
  }
  bool at_symbol(const char* s) const { return tok_.type == Symbol && tok_.text == s; }
  Tok symbol(const char* s) {
    Tok t = take();
    if (t.type != Symbol || t.text != s) error(t, std::string("expected '") + s + "', found '" + t.text + "'");
    return t;
  }
  Tok ident() {
    Tok t = take();
    if (t.type != Ident) error(t, "expected identifier, found '" + t.text + "'");
    return t;
  }
  int integer() {
    Tok t = take();
    if (t.type != Number || !t.integer) error(t, "expected integer, found '" + t.text + "'");
    return (int)t.value;
  }

  void header() {
    Tok t = take();
    if (t.type != Ident || t.text != "OPENQASM") error(t, "expected 'OPENQASM' header");
    Tok v = take();
    if (v.type != Number || v.text != "2.0")
      error(v, "unsupported OPENQASM version '" + v.text + "' (only 2.0 is supported)");
    symbol(";");
  }

  void statement() {
    if (tok_.type != Ident) error(tok_, "expected statement, found '" + tok_.text + "'");
    const std::string& w = tok_.text;
    if (w == "include") {
      take();
      Tok f = take();
      if (f.type != String) error(f, "expected file name string after include");
      if (f.text != "qelib1.inc") error(f, "unsupported include '" + f.text + "' (only qelib1.inc)");
      symbol(";");
    } else if (w == "qreg") {
      Tok kw = take();
      Tok name = ident();
      symbol("[");
      const int size = integer();
      symbol("]");
      symbol(";");
      if (!qreg_.empty()) error(kw, "multiple qregs are not supported");
      if (size <= 0) error(name, "qreg size must be positive");
      qreg_ = name.text;
      c_.n_qubits = size;
    } else if (w == "creg") {
      take();
      Tok name = ident();
      symbol("[");
      const int size = integer();
      symbol("]");
      symbol(";");
      if (size <= 0) error(name, "creg size must be positive");
      if (cregs_.count(name.text)) error(name, "creg '" + name.text + "' redeclared");
      cregs_[name.text] = size;
      c_.n_clbits += size;
    } else if (w == "measure") {
      take();
      const int q = qubit(true);
      symbol("->");
      Tok cn = ident();
      auto it = cregs_.find(cn.text);
      if (it == cregs_.end()) error(cn, "unknown creg '" + cn.text + "'");
      if (q >= 0) {
        symbol("[");
        Tok idx = tok_;
        const int bit = integer();
        symbol("]");
        if (bit >= it->second)
          error(idx, "bit index " + std::to_string(bit) + " out of range for creg of size " +
                         std::to_string(it->second));
        measured_.insert(q);
      } else {
        if (at_symbol("[")) error(tok_, "register-to-bit measure is not supported");
        measured_whole_ = true;
      }
      symbol(";");
    } else if (w == "barrier") {
      take();
      qubit(true);
      while (at_symbol(",")) take(), qubit(true);
      symbol(";");
    } else if (w == "gate" || w == "opaque" || w == "if" || w == "reset") {
      error(tok_, "unsupported statement '" + w + "'");
    } else {
      gate_call();
    }
  }

  // q[i] -> i; a bare register name -> -1 when allowed
  int qubit(bool whole_ok) {
    Tok name = ident();
    if (name.text != qreg_) error(name, "unknown register '" + name.text + "'");
    if (at_symbol("[")) {
      take();
      Tok idx = tok_;
      const int q = integer();
      symbol("]");
      if (q >= c_.n_qubits)
        error(idx, "qubit index " + std::to_string(q) + " out of range for qreg of size " +
                       std::to_string(c_.n_qubits));
      return q;
    }
    if (!whole_ok) error(tok_, "expected '[' after register name");
    return -1;
  }

  void gate_call() {
    Tok name = take();
    Kind k;
    if (!kind_of(name.text, k)) error(name, "unsupported gate '" + name.text + "'");
    Op op;
    op.kind = k;
    const int want = kKinds[k].params;
    if (at_symbol("(")) {
      Tok open = take();
      if (want == 0) error(open, "gate '" + name.text + "' takes no parameters");
      op.params.push_back(expr());
      while (at_symbol(",")) take(), op.params.push_back(expr());
      symbol(")");
    }
    if ((int)op.params.size() != want)
      error(name, "gate '" + name.text + "' expects " + std::to_string(want) + " parameter(s), got " +
                      std::to_string(op.params.size()));
    if (qreg_.empty()) error(name, "gate before qreg declaration");
    op.q0 = qubit(false);
    if (kKinds[k].two) {
      Tok comma = symbol(",");
      op.q1 = qubit(false);
      if (op.q0 == op.q1)
        error(comma, "two-qubit gate needs distinct qubits, got q[" + std::to_string(op.q0) + "] twice");
    }
    symbol(";");
    c_.ops.push_back(std::move(op));
  }

  // expr := term (('+'|'-') term)* ; term := factor (('*'|'/') factor)* ;
  // factor := '-' factor | '(' expr ')' | number | pi
  double expr() {
    double v = term();
    while (at_symbol("+") || at_symbol("-")) {
      const bool plus = take().text == "+";
      const double r = term();
      v = plus ? v + r : v - r;
    }
    return v;
  }
  double term() {
    double v = factor();
    while (at_symbol("*") || at_symbol("/")) {
      Tok o = take();
      const double r = factor();
      if (o.text == "/") {
        if (r == 0.0) error(o, "division by zero in parameter expression");
        v /= r;
      } else {
        v *= r;
      }
    }
    return v;
  }
  double factor() {
    Tok t = take();
    if (t.type == Symbol && t.text == "-") return -factor();
    if (t.type == Symbol && t.text == "(") {
      const double v = expr();
      symbol(")");
      return v;
    }
    if (t.type == Number) return t.value;
    if (t.type == Ident && t.text == "pi") return M_PI;
    error(t, "expected number, 'pi', or '(' in parameter expression, found '" + t.text + "'");
  }

  std::string_view src_;
  size_t pos_ = 0;
  int line_ = 1, col_ = 1;
  Tok tok_;
  Circuit c_;
  std::string qreg_;
  std::map<std::string, int> cregs_;
  std::set<int> measured_;
  bool measured_whole_ = false;
};

Circuit parse(std::string_view text) {
  try {
    return QasmParser(text).run();
  } catch (const ParseFailure& e) {
    t_parse_line = e.line, t_parse_col = e.column;
    fail(MPSIM_EPARSE, "line " + std::to_string(e.line) + ", column " + std::to_string(e.column) + ": " + e.message);
  }
}

// -------------------------------------------------------------- mini JSON
// Enough JSON for the u4 sidecar: objects, arrays, numbers, strings,
// literals. Malformed text -> ConfigError (runner.cpp:175-180).

struct Json {
  enum Type { Null, Bool, Num, Str, Arr, Obj } type = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JsonReader {
 public:
  explicit JsonReader(std::string_view s) : s_(s) {}
  Json document() {
    Json v = value();
    blank();
    if (i_ != s_.size()) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const std::string& why) {
    config_error("malformed sidecar: " + why + " at offset " + std::to_string(i_));
  }
  void blank() {
    while (i_ < s_.size() && std::isspace((unsigned char)s_[i_])) ++i_;
  }
  bool eat(char c) {
    blank();
    if (i_ < s_.size() && s_[i_] == c) return ++i_, true;
    return false;
  }
  std::string string() {
    if (!eat('"')) bad("expected string");
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\') {
        if (++i_ >= s_.size()) bad("bad escape");
        const char e = s_[i_];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        out += s_[i_];
      }
      ++i_;
    }
    if (i_ >= s_.size()) bad("unterminated string");
    ++i_;
    return out;
  }
  Json value() {
    blank();
    if (i_ >= s_.size()) bad("unexpected end");
    Json v;
    const char c = s_[i_];
    if (c == '{') {
      ++i_;
      v.type = Json::Obj;
      if (eat('}')) return v;
      do {
        std::string k = string();
        if (!eat(':')) bad("expected ':'");
        v.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      if (!eat('}')) bad("expected '}'");
    } else if (c == '[') {
      ++i_;
      v.type = Json::Arr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) bad("expected ']'");
    } else if (c == '"') {
      v.type = Json::Str;
      v.str = string();
    } else if (s_.substr(i_, 4) == "true" || s_.substr(i_, 5) == "false") {
      v.type = Json::Bool;
      v.b = s_[i_] == 't';
      i_ += v.b ? 4 : 5;
    } else if (s_.substr(i_, 4) == "null") {
      i_ += 4;
    } else {
      const char* b = s_.data() + i_;
      char* e = nullptr;
      std::string tmp(b, std::min<size_t>(64, s_.size() - i_));
      v.num = std::strtod(tmp.c_str(), &e);
      if (e == tmp.c_str()) bad("unexpected character");
      v.type = Json::Num;
      i_ += (size_t)(e - tmp.c_str());
    }
    return v;
  }
  std::string_view s_;
  size_t i_ = 0;
};

// ------------------------------------------------------------ sidecar I/O

struct SidecarGate {  // generators.hpp:52-57
  size_t op_index = 0;
  int q0 = 0, q1 = 0;
  Mat m;
};

// sidecar_from_json, runner.cpp:141-166
std::vector<SidecarGate> sidecar_from_json(const std::string& text) {
  const Json j = JsonReader(text).document();
  const Json* fmt = j.type == Json::Obj ? j.get("format") : nullptr;
  if (!fmt || fmt->type != Json::Str || fmt->str != "u4-sidecar-v1")
    config_error("sidecar file is not in u4-sidecar-v1 format");
  const Json* ents = j.get("entanglers");
  if (!ents || ents->type != Json::Arr) config_error("sidecar has no entanglers array");
  std::vector<SidecarGate> out;
  for (const Json& e : ents->arr) {
    const Json* oi = e.get("op_index");
    const Json* qs = e.get("qubits");
    const Json* m = e.get("matrix");
    if (!oi || !qs || !m || qs->type != Json::Arr || qs->arr.size() < 2 || m->type != Json::Arr)
      config_error("sidecar entry lacks op_index / qubits / matrix");
    SidecarGate g;
    g.op_index = (size_t)oi->num;
    g.q0 = (int)qs->arr[0].num;
    g.q1 = (int)qs->arr[1].num;
    if (m->arr.size() != 16) config_error("sidecar matrix must have 16 entries");
    g.m.dim = 4;
    for (int i = 0; i < 16; ++i) {
      const Json& z = m->arr[(size_t)i];
      if (z.type != Json::Arr || z.arr.size() < 2) config_error("sidecar matrix entries are [re, im] pairs");
      g.m.a[i] = cd(z.arr[0].num, z.arr[1].num);
    }
    double dev = 0.0;  // |U^H U - I|_max <= 1e-10
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) {
        cd acc = 0.0;
        for (int k = 0; k < 4; ++k) acc += std::conj(g.m(k, r)) * g.m(k, c);
        dev = std::max(dev, std::abs(acc - cd(r == c ? 1.0 : 0.0)));
      }
    if (dev > 1e-10) config_error("sidecar matrix " + std::to_string(out.size()) + " is not unitary");
    out.push_back(g);
  }
  return out;
}

std::string fmt_double(double v) {  // shortest round-trip text
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, r.ptr);
}

// sidecar_to_json, runner.cpp:129-139
std::string sidecar_to_json(const std::vector<SidecarGate>& gs) {
  std::string s = "{\"entanglers\":[";
  for (size_t i = 0; i < gs.size(); ++i) {
    const SidecarGate& g = gs[i];
    s += i ? ",{" : "{";
    s += "\"matrix\":[";
    for (int e = 0; e < 16; ++e) {
      s += e ? ",[" : "[";
      s += fmt_double(g.m.a[e].real()) + "," + fmt_double(g.m.a[e].imag()) + "]";
    }
    s += "],\"op_index\":" + std::to_string(g.op_index) + ",\"qubits\":[" + std::to_string(g.q0) + "," +
         std::to_string(g.q1) + "]}";
  }
  return s + "],\"format\":\"u4-sidecar-v1\"}";
}

// inject_sidecar, runner.cpp:168-190
void inject_sidecar(Circuit& c, std::vector<SidecarGate> gs) {
  std::stable_sort(gs.begin(), gs.end(),
                   [](const SidecarGate& a, const SidecarGate& b) { return a.op_index < b.op_index; });
  for (const SidecarGate& g : gs) {
    if (g.op_index > c.ops.size())
      config_error("sidecar op_index " + std::to_string(g.op_index) + " beyond end of circuit");
    if (g.q0 < 0 || g.q1 < 0 || g.q0 >= c.n_qubits || g.q1 >= c.n_qubits || g.q0 == g.q1)
      config_error("sidecar qubit pair out of range");
    Op op;
    op.kind = U4;
    op.q0 = g.q0, op.q1 = g.q1;
    op.u4 = g.m;
    c.ops.insert(c.ops.begin() + (std::ptrdiff_t)g.op_index, op);
  }
}

// ----------------------------------------------------------------- fusion

struct Block {  // FusedGate, circuit.hpp:71-81
  int q0 = 0, q1 = -1;
  bool flipped = false;
  Mat m;
  bool two() const { return q1 >= 0; }
  bool local() const { return !two() || q1 == q0 + 1; }
  bool touches(int q) const { return q0 == q || (two() && q1 == q); }
  bool overlaps(const Block& o) const { return touches(o.q0) || (o.two() && touches(o.q1)); }
};

// a 2x2 lifted to 4x4 on the low (row bit 1) or high (row bit 0) qubit,
// fusion.cpp:38-52
Mat lift(const Mat& g, bool on_low) {
  Mat r;
  r.dim = 4;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int ih = i >> 1, il = i & 1, jh = j >> 1, jl = j & 1;
      r(i, j) = on_low ? (il == jl ? g(ih, jh) : cd(0.0)) : (ih == jh ? g(il, jl) : cd(0.0));
    }
  return r;
}

Block block_of(const Op& op) {  // fusion.cpp:54-67
  Block b;
  if (op.two()) {
    b.q0 = std::min(op.q0, op.q1), b.q1 = std::max(op.q0, op.q1);
    b.flipped = op.q0 > op.q1;
  } else {
    b.q0 = op.q0;
  }
  b.m = matrix_of(op);
  return b;
}

Block swap_at(int q) {  // fusion.cpp:69-75
  Op op;
  op.kind = Swap;
  op.q0 = q, op.q1 = q + 1;
  return block_of(op);
}

// fuse_circuit, fusion.cpp:79-135: each op meets the most recent block that
// shares a qubit; same support -> multiply and retry; an earlier 1q block is
// folded into a 2q op; a 1q op joins an earlier 2q block if nothing after
// that block touched the block's other qubit.
std::vector<Block> fuse(const Circuit& c) {
  std::vector<Block> out;
  out.reserve(c.ops.size());
  for (const Op& op : c.ops) {
    Block cur = block_of(op);
    for (;;) {
      int j = (int)out.size() - 1;
      while (j >= 0 && !out[(size_t)j].overlaps(cur)) --j;
      if (j < 0) {
        out.push_back(cur);
        break;
      }
      Block& prev = out[(size_t)j];
      if (prev.q0 == cur.q0 && prev.q1 == cur.q1) {
        cur.m = mul(cur.m, prev.m);
        out.erase(out.begin() + j);
        continue;
      }
      if (!prev.two() && cur.two()) {
        cur.m = mul(cur.m, lift(prev.m, prev.q0 == cur.q0));
        out.erase(out.begin() + j);
        continue;
      }
      if (!cur.two() && prev.two()) {
        const int other = prev.q0 == cur.q0 ? prev.q1 : prev.q0;
        bool quiet = true;
        for (size_t k = (size_t)j + 1; k < out.size() && quiet; ++k) quiet = !out[k].touches(other);
        if (quiet) {
          prev.m = mul(lift(cur.m, cur.q0 == prev.q0), prev.m);
          break;
        }
      }
      out.push_back(cur);
      break;
    }
  }
  return out;
}

// decompose_nonlocal, fusion.cpp:137-161
std::vector<Block> lower_nonlocal(const std::vector<Block>& gs, int n) {
  std::vector<Block> out;
  for (const Block& g : gs) {
    if (g.two() && (g.q0 < 0 || g.q1 >= n)) fail(MPSIM_EINVAL, "gate qubits out of range");
    if (g.local()) {
      out.push_back(g);
      continue;
    }
    for (int i = g.q0; i < g.q1 - 1; ++i) out.push_back(swap_at(i));
    Block mid = g;
    mid.q0 = g.q1 - 1;
    out.push_back(mid);
    for (int i = g.q1 - 2; i >= g.q0; --i) out.push_back(swap_at(i));
  }
  return out;
}

// layerize, fusion.cpp:163-190: ASAP layer = 1 + last layer on the span
std::vector<std::vector<Block>> layers_of(const std::vector<Block>& gs) {
  int n = 0;
  for (const Block& g : gs) {
    if (!g.local())
      fail(MPSIM_EINVAL, "layerize requires local gates; found a gate on (" + std::to_string(g.q0) + "," +
                             std::to_string(g.q1) + ")");
    n = std::max(n, (g.two() ? g.q1 : g.q0) + 1);
  }
  std::vector<int> last((size_t)n, -1);
  std::vector<std::vector<Block>> plan;
  for (const Block& g : gs) {
    const int hi = g.two() ? g.q1 : g.q0;
    int L = 0;
    for (int q = g.q0; q <= hi; ++q) L = std::max(L, last[(size_t)q] + 1);
    if ((size_t)L >= plan.size()) plan.resize((size_t)L + 1);
    plan[(size_t)L].push_back(g);
    for (int q = g.q0; q <= hi; ++q) last[(size_t)q] = L;
  }
  return plan;
}

mpsim_gate to_abi(const Block& b) {
  mpsim_gate g;
  std::memset(&g, 0, sizeof g);
  g.q0 = b.q0, g.q1 = b.q1;
  const int k = b.m.dim * b.m.dim;
  for (int e = 0; e < k; ++e) g.u[2 * e] = b.m.a[e].real(), g.u[2 * e + 1] = b.m.a[e].imag();
  return g;
}

Block from_abi(const mpsim_gate& g) {
  Block b;
  b.q0 = g.q0, b.q1 = g.q1 < 0 ? -1 : g.q1;
  b.m.dim = b.q1 >= 0 ? 4 : 2;
  for (int e = 0; e < b.m.dim * b.m.dim; ++e) b.m.a[e] = cd(g.u[2 * e], g.u[2 * e + 1]);
  if (b.q1 >= 0 && b.q1 < b.q0) {  // fold a (high, low) order (gates.cpp:206)
    std::swap(b.q0, b.q1);
    b.m = swap_conj(b.m);
    b.flipped = true;
  }
  return b;
}

// ------------------------------------------------------------- generators

double unit01(std::mt19937_64& e) { return (double)(e() >> 11) * 0x1.0p-53; }  // generators.cpp:31-33
double gauss(std::mt19937_64& e) {                                             // generators.cpp:35-42
  double u1 = unit01(e);
  while (u1 <= 0.0) u1 = unit01(e);
  const double u2 = unit01(e);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

// haar_unitary(4, seed), generators.cpp:73-93: a complex Gaussian matrix
// orthonormalised column by column. Entries are drawn row-major; within an
// entry the reference's Complex(normal_unit(e), normal_unit(e)) is
// evaluated right to left by g++ (its toolchain), so the imaginary part is
// drawn first.
// The reference takes Householder QR and rephases Q's columns by R's
// diagonal phases, i.e. the unique Q whose R has a positive real diagonal;
// Gram-Schmidt with one re-orthogonalisation pass yields that Q directly,
// equal to rounding.
Mat haar4(uint64_t seed) {
  std::mt19937_64 e(seed);
  cd A[4][4];
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      const double im = gauss(e);
      const double re = gauss(e);
      A[r][c] = cd(re, im);
    }
  Mat m;
  m.dim = 4;
  for (int c = 0; c < 4; ++c) {
    cd v[4];
    for (int r = 0; r < 4; ++r) v[r] = A[r][c];
    for (int pass = 0; pass < 2; ++pass)
      for (int k = 0; k < c; ++k) {
        cd dot = 0.0;
        for (int r = 0; r < 4; ++r) dot += std::conj(m(r, k)) * v[r];
        for (int r = 0; r < 4; ++r) v[r] -= dot * m(r, k);
      }
    double nrm = 0.0;
    for (int r = 0; r < 4; ++r) nrm += std::norm(v[r]);
    nrm = std::sqrt(nrm);
    for (int r = 0; r < 4; ++r) m(r, c) = v[r] / nrm;
  }
  return m;
}

std::string angle(double v) {  // "%.17g", generators.cpp:44-48
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string ghz_qasm(int n, bool measure) {  // generators.cpp:52-71
  if (n < 2) config_error("ghz generator needs at least 2 qubits");
  std::ostringstream os;
  os << "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" << n << "];\n";
  if (measure) os << "creg c[" << n << "];\n";
  os << "h q[0];\n";
  for (int i = 0; i + 1 < n; ++i) os << "cx q[" << i << "],q[" << i + 1 << "];\n";
  if (measure) os << "measure q -> c;\n";
  return os.str();
}

// brickwork_qasm, generators.cpp:95-145: per unit, u3(theta, phi, lambda)
// on every qubit (draw order theta, phi, lambda), then entanglers on pairs
// (p, p+1), p = unit % 2, +2: cx, or a Haar 4x4 seeded by engine() recorded
// in the sidecar at its op position.
std::string brickwork_qasm(int n, int depth, uint64_t seed, bool measure, bool haar, std::vector<SidecarGate>& sc) {
  if (n < 2) config_error("brickwork generator needs at least 2 qubits");
  if (depth < 1) config_error("brickwork generator needs depth >= 1");
  std::mt19937_64 e(seed);
  std::ostringstream os;
  os << "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[" << n << "];\n";
  if (measure) os << "creg c[" << n << "];\n";
  size_t pos = 0;
  for (int u = 0; u < depth; ++u) {
    for (int q = 0; q < n; ++q, ++pos) {
      const double th = unit01(e) * 2.0 * M_PI;
      const double ph = unit01(e) * 2.0 * M_PI;
      const double la = unit01(e) * 2.0 * M_PI;
      os << "u3(" << angle(th) << "," << angle(ph) << "," << angle(la) << ") q[" << q << "];\n";
    }
    for (int p = u % 2; p + 1 < n; p += 2, ++pos) {
      if (!haar) {
        os << "cx q[" << p << "],q[" << p + 1 << "];\n";
        continue;
      }
      SidecarGate g;
      g.op_index = pos;
      g.q0 = p, g.q1 = p + 1;
      g.m = haar4(e());
      os << "// u4 " << sc.size() << " q[" << p << "],q[" << p + 1 << "];\n";
      sc.push_back(g);
    }
  }
  if (measure) os << "measure q -> c;\n";
  return os.str();
}

// ------------------------------------------------------------ run_circuit

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) config_error("cannot read input file '" + path + "'");
  std::ostringstream b;
  b << in.rdbuf();
  return b.str();
}

bool file_exists(const std::string& p) {
  std::ifstream in(p);
  return (bool)in;
}

std::string str_or(const char* s) { return s ? std::string(s) : std::string(); }

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\', o += c;
    else if (c == '\n') o += "\\n";
    else if ((unsigned char)c < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else o += c;
  }
  return o + "\"";
}

struct LayerStat {
  long long gates = 0;
  unsigned long long compute_ns = 0, sync_ns = 0;
};

struct StateHandle {  // RAII over the engine's C ABI
  mpsim_gpu_state* s = nullptr;
  ~StateHandle() {
    if (s) mpsim_gpu_state_destroy(s);
  }
};
struct SamplerHandle {
  mpsim_gpu_sampler* p = nullptr;
  ~SamplerHandle() {
    if (p) mpsim_gpu_sampler_destroy(p);
  }
};

void check(int rc) {
  if (rc != MPSIM_OK) fail(rc, mpsim_gpu_last_error());
}

using Clock = std::chrono::steady_clock;
unsigned long long ns_since(Clock::time_point t0) {
  return (unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count();
}

std::string run(const mpsim_run_config& cfg) {
  // validate_config, runner.cpp:42-62
  if (cfg.workers < 1) config_error("workers must be >= 1");
  if (cfg.max_bond < 0) config_error("max-bond must be >= 0 (0 means unbounded)");
  if (!(cfg.cutoff >= 0.0 && cfg.cutoff < 1.0)) config_error("cutoff must lie in [0, 1)");
  if (cfg.backend < MPSIM_BACKEND_MPS_SERIAL || cfg.backend > MPSIM_BACKEND_STATEVECTOR)
    config_error("unknown backend");
  if (cfg.nonlocal != MPSIM_NONLOCAL_SWAP && cfg.nonlocal != MPSIM_NONLOCAL_BONDPROP)
    config_error("unknown nonlocal method");
  if (cfg.backend == MPSIM_BACKEND_MPS_PARALLEL && cfg.nonlocal == MPSIM_NONLOCAL_BONDPROP)
    config_error(
        "bond propagation is only available on the serial backend; the parallel plan lowers non-local gates to "
        "SWAP chains");
  const std::string path = str_or(cfg.qasm_path), inline_text = str_or(cfg.qasm_text);
  if (path.empty() && inline_text.empty()) config_error("no circuit given");

  Circuit c = parse(path.empty() ? std::string_view(inline_text) : std::string_view(read_file(path)));
  std::string sc_text = str_or(cfg.sidecar_json), sc_path = str_or(cfg.sidecar_path);
  if (sc_text.empty()) {
    if (sc_path.empty() && !path.empty() && file_exists(path + ".u4.json")) sc_path = path + ".u4.json";
    if (!sc_path.empty()) sc_text = read_file(sc_path);
  }
  if (!sc_text.empty()) inject_sidecar(c, sidecar_from_json(sc_text));

  std::vector<LayerStat> layers;
  std::map<std::string, unsigned long long> counts;
  long long peak = 0;
  double total_w = 0.0;
  const auto t0 = Clock::now();
  if (cfg.backend == MPSIM_BACKEND_STATEVECTOR) {
    // runner.cpp:236-250: sv_run over the raw ops, then CDF sampling
    if (c.n_qubits > cfg.statevector_cap)
      fail(MPSIM_EINVAL, "statevector capped at " + std::to_string(cfg.statevector_cap) + " qubits, got " +
                             std::to_string(c.n_qubits));
    std::vector<SvOp> ops;
    ops.reserve(c.ops.size());
    for (const Op& op : c.ops) {
      SvOp s;
      s.q0 = op.two() ? std::min(op.q0, op.q1) : op.q0;
      s.q1 = op.two() ? std::max(op.q0, op.q1) : -1;
      const Mat m = matrix_of(op);
      for (int e = 0; e < m.dim * m.dim; ++e) s.u[e] = m.a[e];
      ops.push_back(s);
    }
    std::vector<cd> amps;
    sv_run_device(c.n_qubits, ops, cfg.device, amps, nullptr);
    LayerStat L;
    L.gates = (long long)c.ops.size();
    L.compute_ns = ns_since(t0);
    layers.push_back(L);
    if (cfg.shots > 0) {  // sample_statevector, runner.cpp:86-104
      std::vector<double> cdf(amps.size());
      double acc = 0.0;
      for (size_t i = 0; i < amps.size(); ++i) cdf[i] = acc += std::norm(amps[i]);
      std::mt19937_64 e(cfg.seed);
      const int n = c.n_qubits;
      for (uint64_t s = 0; s < cfg.shots; ++s) {
        const double u = unit01(e) * acc;
        size_t idx = (size_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
        idx = std::min(idx, amps.size() - 1);
        std::string bits((size_t)n, '0');
        for (int q = 0; q < n; ++q)
          if ((idx >> (n - 1 - q)) & 1U) bits[(size_t)q] = '1';
        ++counts[bits];
      }
    }
  } else {
    const std::vector<Block> fused = fuse(c);
    StateHandle st;
    check(mpsim_gpu_state_create(c.n_qubits, cfg.chi_hint > 0 ? cfg.chi_hint : 16, cfg.device, &st.s));
    mpsim_policy pol{cfg.max_bond == 0 ? (int64_t)MPSIM_UNBOUNDED : cfg.max_bond, cfg.cutoff};
    if (cfg.backend == MPSIM_BACKEND_MPS_PARALLEL) {
      // execute_parallel over layerize(decompose_nonlocal(fused)),
      // runner.cpp:256-260: one batched launch sequence per layer
      const auto plan = layers_of(lower_nonlocal(fused, c.n_qubits));
      peak = 1;
      std::vector<mpsim_gate> gs;
      std::vector<mpsim_report> reps;
      for (const auto& layer : plan) {
        const auto tl = Clock::now();
        gs.clear();
        for (const Block& b : layer) gs.push_back(to_abi(b));
        reps.assign(gs.size(), mpsim_report{});
        check(mpsim_gpu_apply_layer(st.s, gs.data(), (int32_t)gs.size(), &pol, reps.data()));
        LayerStat L;
        L.gates = (long long)layer.size();
        L.compute_ns = ns_since(tl);
        const auto ts = Clock::now();
        for (const mpsim_report& r : reps) {  // barrier merge, executor.cpp:144-177
          total_w += r.discarded_weight;
          peak = std::max<long long>(peak, r.new_bond);
        }
        L.sync_ns = ns_since(ts);
        layers.push_back(L);
      }
      check(mpsim_gpu_validate(st.s));
    } else {
      // execute_serial, executor.cpp:73-97: one LayerStat for the whole list
      std::vector<mpsim_gate> gs;
      gs.reserve(fused.size());
      for (const Block& b : fused) gs.push_back(to_abi(b));
      mpsim_exec_stats es{};
      check(mpsim_gpu_execute(st.s, gs.data(), (int32_t)gs.size(), &pol, cfg.nonlocal, &es, nullptr));
      LayerStat L;
      L.gates = (long long)fused.size();
      L.compute_ns = ns_since(t0);
      layers.push_back(L);
      peak = es.peak_bond;
      total_w = es.total_discarded_weight;
    }
    if (cfg.shots > 0) {  // sample(), runner.cpp:265-271
      SamplerHandle sp;
      check(mpsim_gpu_sampler_create(st.s, cfg.memoize ? 1 : 0, cfg.cache_cap, &sp.p));
      int32_t uniq = 0;
      check(mpsim_gpu_sample(sp.p, cfg.shots, cfg.seed, &uniq));
      std::string bits((size_t)c.n_qubits, '0');
      for (int32_t i = 0; i < uniq; ++i) {
        uint64_t cnt = 0;
        check(mpsim_gpu_sampler_result(sp.p, i, bits.data(), &cnt));
        counts[bits] = cnt;
      }
    }
  }
  const unsigned long long wall = ns_since(t0);

  // run_output_to_json, runner.cpp:291-328 (keys in nlohmann's sorted order)
  const char* backends[] = {"mps-serial", "mps-parallel", "statevector"};
  std::string label = str_or(cfg.input_label);
  if (label.empty()) label = path.empty() ? "<inline>" : path;
  std::string j = "{\"config\":{";
  j += "\"backend\":" + json_str(backends[cfg.backend]);
  j += ",\"cutoff\":" + fmt_double(cfg.cutoff);
  j += ",\"input\":" + json_str(label);
  j += ",\"max_bond\":" + std::to_string(cfg.max_bond);
  j += std::string(",\"memoize\":") + (cfg.memoize ? "true" : "false");
  j += ",\"nonlocal\":" + json_str(cfg.nonlocal == MPSIM_NONLOCAL_SWAP ? "swap" : "bondprop");
  j += ",\"seed\":" + std::to_string(cfg.seed);
  j += ",\"shots\":" + std::to_string(cfg.shots);
  j += ",\"workers\":" + std::to_string(cfg.workers) + "}";
  if (cfg.shots > 0) {
    j += ",\"counts\":{";
    bool first = true;
    for (const auto& kv : counts) {
      j += first ? "" : ",";
      j += json_str(kv.first) + ":" + std::to_string(kv.second);
      first = false;
    }
    j += "}";
  }
  j += ",\"layers\":[";
  for (size_t i = 0; i < layers.size(); ++i) {
    j += i ? "," : "";
    j += "{\"compute_ns\":" + std::to_string(layers[i].compute_ns) + ",\"gates\":" +
         std::to_string(layers[i].gates) + ",\"sync_ns\":" + std::to_string(layers[i].sync_ns) + "}";
  }
  j += "],\"n_qubits\":" + std::to_string(c.n_qubits);
  j += ",\"peak_bond\":" + std::to_string(peak);
  j += ",\"total_discarded_weight\":" + fmt_double(total_w);
  j += ",\"total_wall_ns\":" + std::to_string(wall) + "}";
  return j;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MPSIM_OK;
  } catch (const Error& e) {
    last_error_slot() = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    last_error_slot() = "host allocation failed";
    return MPSIM_ECUDA;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return MPSIM_ELOGIC;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class T>
T* dup_array(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace fe
}  // namespace mpsim_gpu

using namespace mpsim_gpu;

extern "C" {

void mpsim_free(void* p) { std::free(p); }

int mpsim_parse_qasm(const char* text, mpsim_circuit_info* info, mpsim_prim_op* ops, int32_t max_ops) {
  return fe::guard([&] {
    if (!text || !info) fail(MPSIM_EINVAL, "null argument");
    const fe::Circuit c = fe::parse(text);
    info->n_qubits = c.n_qubits;
    info->n_clbits = c.n_clbits;
    info->has_measure_all = c.measure_all ? 1 : 0;
    info->n_ops = (int32_t)c.ops.size();
    for (int32_t i = 0; ops && i < max_ops && i < (int32_t)c.ops.size(); ++i) {
      const fe::Op& o = c.ops[(size_t)i];
      mpsim_prim_op& d = ops[i];
      std::memset(&d, 0, sizeof d);
      d.kind = o.kind, d.q0 = o.q0, d.q1 = o.q1, d.nparams = (int32_t)o.params.size();
      for (size_t k = 0; k < o.params.size() && k < 3; ++k) d.params[k] = o.params[k];
    }
  });
}

int mpsim_last_parse_location(int32_t* line, int32_t* column) {
  if (line) *line = fe::t_parse_line;
  if (column) *column = fe::t_parse_col;
  return MPSIM_OK;
}

int mpsim_fuse_qasm(const char* qasm, const char* sidecar_json, int32_t* n_qubits, mpsim_gate** gates,
                    int32_t** flipped, int32_t* count) {
  return fe::guard([&] {
    if (!qasm || !gates || !count) fail(MPSIM_EINVAL, "null argument");
    fe::Circuit c = fe::parse(qasm);
    if (sidecar_json && *sidecar_json) fe::inject_sidecar(c, fe::sidecar_from_json(sidecar_json));
    const auto fused = fe::fuse(c);
    std::vector<mpsim_gate> g;
    std::vector<int32_t> fl;
    for (const auto& b : fused) g.push_back(fe::to_abi(b)), fl.push_back(b.flipped ? 1 : 0);
    if (n_qubits) *n_qubits = c.n_qubits;
    *gates = fe::dup_array(g);
    if (flipped) *flipped = fe::dup_array(fl);
    *count = (int32_t)g.size();
  });
}

int mpsim_plan_layers(const mpsim_gate* gates, int32_t count, int32_t n_qubits, mpsim_gate** out,
                      int32_t** layer_of, int32_t* out_count, int32_t* n_layers) {
  return fe::guard([&] {
    if ((!gates && count > 0) || !out || !out_count) fail(MPSIM_EINVAL, "null argument");
    std::vector<fe::Block> in;
    for (int32_t i = 0; i < count; ++i) in.push_back(fe::from_abi(gates[i]));
    const auto plan = fe::layers_of(fe::lower_nonlocal(in, n_qubits));
    std::vector<mpsim_gate> g;
    std::vector<int32_t> lo;
    for (size_t L = 0; L < plan.size(); ++L)
      for (const auto& b : plan[L]) g.push_back(fe::to_abi(b)), lo.push_back((int32_t)L);
    *out = fe::dup_array(g);
    if (layer_of) *layer_of = fe::dup_array(lo);
    *out_count = (int32_t)g.size();
    if (n_layers) *n_layers = (int32_t)plan.size();
  });
}

int mpsim_gen_ghz_qasm(int32_t n, int32_t measure, char** qasm) {
  return fe::guard([&] {
    if (!qasm) fail(MPSIM_EINVAL, "null argument");
    *qasm = fe::dup(fe::ghz_qasm(n, measure != 0));
  });
}

int mpsim_gen_brickwork_qasm(int32_t n, int32_t depth, uint64_t seed, int32_t measure, int32_t haar, char** qasm,
                             char** sidecar_json) {
  return fe::guard([&] {
    if (!qasm) fail(MPSIM_EINVAL, "null argument");
    std::vector<fe::SidecarGate> sc;
    const std::string q = fe::brickwork_qasm(n, depth, seed, measure != 0, haar != 0, sc);
    *qasm = fe::dup(q);
    if (sidecar_json) *sidecar_json = haar ? fe::dup(fe::sidecar_to_json(sc)) : nullptr;
  });
}

void mpsim_run_config_defaults(mpsim_run_config* c) {  // RunConfig, runner.hpp:46-62
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->backend = MPSIM_BACKEND_MPS_SERIAL;
  c->nonlocal = MPSIM_NONLOCAL_SWAP;
  c->max_bond = 0;
  c->cutoff = 0.0;
  c->shots = 0;
  c->seed = 1;
  c->workers = 1;
  c->memoize = 1;
  c->cache_cap = 0;
  c->statevector_cap = 20;
  c->device = 0;
  c->chi_hint = 16;
}

int mpsim_gpu_run_circuit(const mpsim_run_config* c, char** json) {
  return fe::guard([&] {
    if (!c || !json) fail(MPSIM_EINVAL, "null argument");
    *json = fe::dup(fe::run(*c));
  });
}

}  // extern "C"
