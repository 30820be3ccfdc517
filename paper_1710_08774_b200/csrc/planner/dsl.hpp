// Kernel-body expression DSL of the rule file (R/SPEC.md:82).
#pragma once

#include <functional>
#include <memory>
#include <set>
#include <string>
#include <vector>

namespace lf {

struct Expr {
  enum Kind { Num, Var, Neg, Add, Sub, Mul, Div, Call } kind = Num;
  std::string text;  // number literal, variable or function name
  std::vector<std::unique_ptr<Expr>> args;
};

std::unique_ptr<Expr> parse_expr(const std::string& text, std::string& err);
void expr_vars(const Expr& e, std::set<std::string>& out);
// fully parenthesised C in element type `type` ("double" / "float");
// `var` maps a parameter name to its C expression
std::string emit_c(const Expr& e, const std::string& type, const std::function<std::string(const std::string&)>& var);
// fp32 only: the same expression on a float2 pair of cells (packed FADD2 /
// FMUL2 / FFMA2 where lanewise exact, per-lane helpers lf_*2 otherwise);
// `var` maps a parameter name to a float2 expression
std::string emit_c2(const Expr& e, const std::function<std::string(const std::string&)>& var);

}  // namespace lf
