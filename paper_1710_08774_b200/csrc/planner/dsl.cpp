// Kernel-body expression DSL (R/SPEC.md:82): `out = expr` with + - * /, unary
// minus, parentheses, sqrt min max abs, numeric literals and parameter names.
// Parsed once into a tree and emitted as fully parenthesised C so that the
// evaluation order is fixed; min/max are `a < b ? a : b` / `a > b ? a : b`.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "dsl.hpp"

namespace lf {

namespace {

struct P {
  const std::string& s;
  size_t i = 0;
  std::string err;
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  std::unique_ptr<Expr> fail(const std::string& m) {
    if (err.empty()) err = m + " at column " + std::to_string(i + 1);
    return nullptr;
  }
  std::unique_ptr<Expr> primary() {
    ws();
    if (i >= s.size()) return fail("unexpected end of expression");
    char c = s[i];
    if (c == '(') {
      ++i;
      auto e = expr();
      if (!e) return nullptr;
      if (!eat(')')) return fail("expected ')'");
      return e;
    }
    if (c == '-') {
      ++i;
      auto e = factor();
      if (!e) return nullptr;
      auto n = std::make_unique<Expr>();
      n->kind = Expr::Neg;
      n->args.push_back(std::move(e));
      return n;
    }
    if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
      size_t j = i;
      while (j < s.size() && (std::isdigit(static_cast<unsigned char>(s[j])) || s[j] == '.')) ++j;
      if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
        ++j;
        if (j < s.size() && (s[j] == '+' || s[j] == '-')) ++j;
        while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
      }
      auto n = std::make_unique<Expr>();
      n->kind = Expr::Num;
      n->text = s.substr(i, j - i);
      char* end = nullptr;
      std::strtod(n->text.c_str(), &end);
      if (!end || *end) return fail("bad number '" + n->text + "'");
      i = j;
      return n;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      size_t j = i;
      while (j < s.size() && (std::isalnum(static_cast<unsigned char>(s[j])) || s[j] == '_')) ++j;
      std::string name = s.substr(i, j - i);
      i = j;
      ws();
      if (i < s.size() && s[i] == '(') {
        ++i;
        auto n = std::make_unique<Expr>();
        n->kind = Expr::Call;
        n->text = name;
        if (name != "sqrt" && name != "min" && name != "max" && name != "abs")
          return fail("unknown function '" + name + "' (sqrt, min, max, abs)");
        if (!eat(')')) {
          while (true) {
            auto a = expr();
            if (!a) return nullptr;
            n->args.push_back(std::move(a));
            if (eat(')')) break;
            if (!eat(',')) return fail("expected ',' or ')'");
          }
        }
        const size_t want = (name == "min" || name == "max") ? 2 : 1;
        if (n->args.size() != want) return fail(name + " takes " + std::to_string(want) + " argument(s)");
        return n;
      }
      auto n = std::make_unique<Expr>();
      n->kind = Expr::Var;
      n->text = name;
      return n;
    }
    return fail(std::string("unexpected character '") + c + "'");
  }
  std::unique_ptr<Expr> factor() { return primary(); }
  std::unique_ptr<Expr> term() {
    auto l = factor();
    while (l) {
      ws();
      if (i < s.size() && (s[i] == '*' || s[i] == '/')) {
        char op = s[i++];
        auto r = factor();
        if (!r) return nullptr;
        auto n = std::make_unique<Expr>();
        n->kind = op == '*' ? Expr::Mul : Expr::Div;
        n->args.push_back(std::move(l));
        n->args.push_back(std::move(r));
        l = std::move(n);
      } else {
        break;
      }
    }
    return l;
  }
  std::unique_ptr<Expr> expr() {
    auto l = term();
    while (l) {
      ws();
      if (i < s.size() && (s[i] == '+' || s[i] == '-')) {
        char op = s[i++];
        auto r = term();
        if (!r) return nullptr;
        auto n = std::make_unique<Expr>();
        n->kind = op == '+' ? Expr::Add : Expr::Sub;
        n->args.push_back(std::move(l));
        n->args.push_back(std::move(r));
        l = std::move(n);
      } else {
        break;
      }
    }
    return l;
  }
};

}  // namespace

std::unique_ptr<Expr> parse_expr(const std::string& text, std::string& err) {
  P p{text};
  auto e = p.expr();
  if (e) {
    p.ws();
    if (p.i != text.size()) {
      p.fail("trailing characters");
      e.reset();
    }
  }
  err = p.err;
  return e;
}

void expr_vars(const Expr& e, std::set<std::string>& out) {
  if (e.kind == Expr::Var) out.insert(e.text);
  for (const auto& a : e.args) expr_vars(*a, out);
}

// Division by a literal, strength-reduced where the result is provably the
// IEEE quotient: a power of two becomes a multiplication by its exact
// reciprocal (both round the same real number once), and fp32 division by 3
// becomes lf_div3f (userkernels/stencil_kernels.h: one multiply and an FMA
// correction, checked bit-identical for all 2^32 inputs by oracle/div3check).
// Empty: keep the division.
enum class LitDiv { none, pow2, three };
static LitDiv literal_divisor(const std::string& lit, bool f, std::string& recip) {
  char* end = nullptr;
  const double c = std::strtod(lit.c_str(), &end);
  if (!end || *end || !std::isfinite(c) || c == 0.0) return LitDiv::none;
  if (f && static_cast<double>(static_cast<float>(c)) != c) return LitDiv::none;
  int ex = 0;
  const double m = std::frexp(c, &ex);  // c = m * 2^ex, |m| in [0.5, 1)
  if (std::fabs(m) == 0.5) {
    const int k = ex - 1;  // |c| = 2^k; 1/c = 2^-k must be a normal number of the type
    if (f ? (k >= -126 && k <= 126) : (k >= -1022 && k <= 1022)) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%s0x1p%d%s", m < 0 ? "-" : "", -k, f ? "f" : "");
      recip = buf;
      return LitDiv::pow2;
    }
    return LitDiv::none;
  }
  if (f && c == 3.0) return LitDiv::three;
  return LitDiv::none;
}

static std::string div_by_literal(const std::string& num, const std::string& lit, bool f) {
  std::string recip;
  switch (literal_divisor(lit, f, recip)) {
    case LitDiv::pow2: return "(" + num + " * " + recip + ")";
    case LitDiv::three: return "lf_div3f(" + num + ")";
    case LitDiv::none: break;
  }
  return "";
}

std::string emit_c(const Expr& e, const std::string& type, const std::function<std::string(const std::string&)>& var) {
  const bool f = type == "float";
  auto A = [&](int k) { return emit_c(*e.args[k], type, var); };
  switch (e.kind) {
    case Expr::Num: return "static_cast<" + type + ">(" + (e.text.find_first_of(".eE") == std::string::npos ? e.text + ".0" : e.text) + ")";
    case Expr::Var: return var(e.text);
    case Expr::Neg: return "(-" + A(0) + ")";
    case Expr::Add: return "(" + A(0) + " + " + A(1) + ")";
    case Expr::Sub: return "(" + A(0) + " - " + A(1) + ")";
    case Expr::Mul: return "(" + A(0) + " * " + A(1) + ")";
    case Expr::Div:
      if (e.args[1]->kind == Expr::Num) {
        const std::string r = div_by_literal(A(0), e.args[1]->text, f);
        if (!r.empty()) return r;
      }
      return "(" + A(0) + " / " + A(1) + ")";
    case Expr::Call:
      if (e.text == "sqrt") return std::string(f ? "sqrtf(" : "sqrt(") + A(0) + ")";
      if (e.text == "abs") return std::string(f ? "fabsf(" : "fabs(") + A(0) + ")";
      if (e.text == "min") return "lf_min(" + A(0) + ", " + A(1) + ")";
      return "lf_max(" + A(0) + ", " + A(1) + ")";
  }
  return "?";
}

// fp32x2: the expression on two cells at once.  + and * map to the lanewise
// FADD2 / FMUL2 (a - b is a + (-b), as IEEE defines it), x / 3 to lf_div3f2,
// a power-of-two divisor to the product with its exact reciprocal; the other
// operations go lane by lane through the lf_*2 helpers the generated module
// defines -- each lane rounds exactly as emit_c's scalar code.
std::string emit_c2(const Expr& e, const std::function<std::string(const std::string&)>& var) {
  auto A = [&](int k) { return emit_c2(*e.args[k], var); };
  switch (e.kind) {
    case Expr::Num: return "lf_f2(static_cast<float>(" + (e.text.find_first_of(".eE") == std::string::npos ? e.text + ".0" : e.text) + "))";
    case Expr::Var: return var(e.text);
    case Expr::Neg: return "lf_neg2(" + A(0) + ")";
    case Expr::Add: return "__fadd2_rn(" + A(0) + ", " + A(1) + ")";
    case Expr::Sub: return "__fadd2_rn(" + A(0) + ", lf_neg2(" + A(1) + "))";
    case Expr::Mul: return "__fmul2_rn(" + A(0) + ", " + A(1) + ")";
    case Expr::Div:
      if (e.args[1]->kind == Expr::Num) {
        std::string recip;
        switch (literal_divisor(e.args[1]->text, true, recip)) {
          case LitDiv::pow2: return "__fmul2_rn(" + A(0) + ", lf_f2(" + recip + "))";
          case LitDiv::three: return "lf_div3f2(" + A(0) + ")";
          case LitDiv::none: break;
        }
      }
      return "lf_div2(" + A(0) + ", " + A(1) + ")";
    case Expr::Call:
      if (e.text == "sqrt") return "lf_sqrt2(" + A(0) + ")";
      if (e.text == "abs") return "lf_abs2(" + A(0) + ")";
      if (e.text == "min") return "lf_min2(" + A(0) + ", " + A(1) + ")";
      return "lf_max2(" + A(0) + ", " + A(1) + ")";
  }
  return "?";
}

}  // namespace lf
