// Minimal YAML reader for `.lf` rule files (yaml-cpp replacement; the
// reference loads the file with YAML::Load, rulespec.cpp:550-560).
#include <cctype>
#include <sstream>

#include "planner.hpp"

namespace lf {

const YNode* YNode::get(const std::string& key) const {
  if (kind != Map) return nullptr;
  for (const auto& [k, v] : map)
    if (k == key) return &v;
  return nullptr;
}

namespace {

struct Line {
  int no;          // 1-based
  int indent;      // leading spaces
  std::string raw; // full text without newline
  std::string content;  // after indent, comment stripped, right-trimmed
};

std::string rtrim(std::string s) {
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.pop_back();
  return s;
}

std::string trim(const std::string& s) {
  size_t a = 0;
  while (a < s.size() && (s[a] == ' ' || s[a] == '\t')) ++a;
  return rtrim(s.substr(a));
}

// strip a `#` comment that is at the start or preceded by whitespace, outside quotes
std::string strip_comment(const std::string& s) {
  char q = 0;
  for (size_t i = 0; i < s.size(); ++i) {
    char c = s[i];
    if (q) {
      if (c == '\\' && q == '"' && i + 1 < s.size()) {
        ++i;
        continue;
      }
      if (c == q) q = 0;
      continue;
    }
    if (c == '"' || c == '\'') {
      q = c;
      continue;
    }
    if (c == '#' && (i == 0 || s[i - 1] == ' ' || s[i - 1] == '\t')) return rtrim(s.substr(0, i));
  }
  return rtrim(s);
}

struct Parser {
  std::vector<Line> lines;
  size_t pos = 0;
  const std::string& file;
  DiagList& diags;
  bool failed = false;

  Parser(const std::string& text, const std::string& f, DiagList& d) : file(f), diags(d) {
    std::istringstream is(text);
    std::string ln;
    int no = 0;
    while (std::getline(is, ln)) {
      ++no;
      Line L;
      L.no = no;
      L.raw = rtrim(ln);
      int ind = 0;
      while (ind < static_cast<int>(L.raw.size()) && L.raw[ind] == ' ') ++ind;
      if (ind < static_cast<int>(L.raw.size()) && L.raw[ind] == '\t') {
        diags.error({file, no, ind + 1}, "tabs are not allowed for indentation");
        failed = true;
      }
      L.indent = ind;
      L.content = strip_comment(L.raw.substr(ind));
      lines.push_back(std::move(L));
    }
  }

  void err(int line, int col, const std::string& m) {
    if (!failed) diags.error({file, line, col}, "syntax error: " + m);
    failed = true;
  }

  void skip_blank() {
    while (pos < lines.size() && lines[pos].content.empty()) ++pos;
  }

  // ---- flow values --------------------------------------------------------
  struct Flow {
    const std::string& s;
    size_t i = 0;
    int line, col0;
    Parser& P;
    void ws() {
      while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n')) ++i;
    }
    YNode value() {
      ws();
      YNode n;
      n.line = line;
      n.column = col0 + static_cast<int>(i);
      if (i >= s.size()) {
        n.kind = YNode::Null;
        return n;
      }
      if (s[i] == '[') {
        ++i;
        n.kind = YNode::Seq;
        ws();
        if (i < s.size() && s[i] == ']') {
          ++i;
          return n;
        }
        while (true) {
          n.seq.push_back(value());
          ws();
          if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
          }
          if (i < s.size() && s[i] == ']') {
            ++i;
            break;
          }
          P.err(line, col0 + static_cast<int>(i), "expected ',' or ']' in flow sequence");
          return n;
        }
        return n;
      }
      if (s[i] == '{') {
        ++i;
        n.kind = YNode::Map;
        ws();
        if (i < s.size() && s[i] == '}') {
          ++i;
          return n;
        }
        while (true) {
          ws();
          YNode k = scalar(true);
          ws();
          if (i >= s.size() || s[i] != ':') {
            P.err(line, col0 + static_cast<int>(i), "expected ':' in flow mapping");
            return n;
          }
          ++i;
          n.map.emplace_back(k.scalar, value());
          ws();
          if (i < s.size() && s[i] == ',') {
            ++i;
            continue;
          }
          if (i < s.size() && s[i] == '}') {
            ++i;
            break;
          }
          P.err(line, col0 + static_cast<int>(i), "expected ',' or '}' in flow mapping");
          return n;
        }
        return n;
      }
      return scalar(false);
    }
    YNode scalar(bool key) {
      YNode n;
      n.kind = YNode::Scalar;
      n.line = line;
      n.column = col0 + static_cast<int>(i);
      if (i < s.size() && (s[i] == '"' || s[i] == '\'')) {
        char q = s[i++];
        std::string out;
        while (i < s.size() && s[i] != q) {
          if (q == '"' && s[i] == '\\' && i + 1 < s.size()) {
            char e = s[++i];
            out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
            ++i;
            continue;
          }
          out += s[i++];
        }
        if (i >= s.size()) P.err(line, n.column, "unterminated quoted scalar");
        ++i;
        n.scalar = out;
        return n;
      }
      size_t a = i;
      while (i < s.size() && s[i] != ',' && s[i] != ']' && s[i] != '}' && !(key && s[i] == ':'))
        ++i;
      n.scalar = trim(s.substr(a, i - a));
      if (n.scalar.empty() || n.scalar == "~" || n.scalar == "null") n.kind = YNode::Null;
      return n;
    }
  };

  // find `key:` at top level of a content string; returns position of ':'
  static size_t key_colon(const std::string& c) {
    if (c.empty() || c[0] == '[' || c[0] == '{' || c[0] == '-') {
      if (!(c.size() > 1 && c[0] == '-' && c[1] != ' ')) return std::string::npos;
    }
    char q = 0;
    for (size_t i = 0; i < c.size(); ++i) {
      char ch = c[i];
      if (q) {
        if (ch == q) q = 0;
        continue;
      }
      if (ch == '"' || ch == '\'') {
        if (i == 0) q = ch;
        continue;
      }
      if (ch == '[' || ch == '{' || ch == '(') return std::string::npos;
      if (ch == ':' && (i + 1 == c.size() || c[i + 1] == ' ')) return i;
    }
    return std::string::npos;
  }

  static bool is_seq_item(const std::string& c) { return c == "-" || (c.size() > 1 && c[0] == '-' && c[1] == ' '); }

  // value text after `key:` (or after `- `) starting on line `ln` at column `col`
  YNode inline_value(const std::string& rest_in, int ln_index, int col, int parent_indent) {
    std::string rest = trim(rest_in);
    const Line& L = lines[ln_index];
    YNode n;
    n.line = L.no;
    n.column = col;
    if (rest.empty()) {
      // nested block, or a sequence at the same indent as the key
      size_t save = pos;
      skip_blank();
      if (pos < lines.size() && (lines[pos].indent > parent_indent ||
                                 (lines[pos].indent == parent_indent && is_seq_item(lines[pos].content)))) {
        return block(lines[pos].indent);
      }
      pos = save;
      n.kind = YNode::Null;
      return n;
    }
    if (rest[0] == '|' || rest[0] == '>') {
      bool strip = rest.find('-') != std::string::npos;
      n.kind = YNode::Scalar;
      n.literal = true;
      std::vector<std::string> body;
      int content_indent = -1;
      while (pos < lines.size()) {
        const Line& B = lines[pos];
        bool blank = trim(B.raw).empty();
        if (!blank && B.indent <= parent_indent) break;
        if (!blank && content_indent < 0) content_indent = B.indent;
        if (!blank && B.indent < content_indent) break;
        body.push_back(blank ? std::string() : B.raw.substr(content_indent));
        ++pos;
      }
      while (!body.empty() && body.back().empty()) body.pop_back();
      std::string out;
      for (const auto& b : body) out += b + "\n";
      if (strip && !out.empty()) out.pop_back();
      n.scalar = out;
      n.line = L.no + 1;
      return n;
    }
    if (rest[0] == '[' || rest[0] == '{') {
      // flow value, possibly spanning lines until brackets balance
      std::string acc = rest;
      auto balanced = [](const std::string& s) {
        int d = 0;
        char q = 0;
        for (char c : s) {
          if (q) {
            if (c == q) q = 0;
            continue;
          }
          if (c == '"' || c == '\'') q = c;
          if (c == '[' || c == '{') ++d;
          if (c == ']' || c == '}') --d;
        }
        return d <= 0;
      };
      while (!balanced(acc) && pos < lines.size()) {
        acc += "\n" + lines[pos].content;
        ++pos;
      }
      Flow f{acc, 0, L.no, col, *this};
      YNode v = f.value();
      f.ws();
      if (f.i < acc.size()) err(L.no, col + static_cast<int>(f.i), "trailing characters after flow value");
      return v;
    }
    if (rest[0] == '"' || rest[0] == '\'') {
      Flow f{rest, 0, L.no, col, *this};
      return f.scalar(false);
    }
    // plain scalar with optional continuation lines
    std::string acc = rest;
    while (pos < lines.size()) {
      const Line& C = lines[pos];
      if (C.content.empty()) break;
      if (C.indent <= parent_indent) break;
      if (key_colon(C.content) != std::string::npos || is_seq_item(C.content)) break;
      acc += " " + C.content;
      ++pos;
    }
    n.kind = YNode::Scalar;
    n.scalar = acc;
    if (acc == "~" || acc == "null") n.kind = YNode::Null;
    return n;
  }

  YNode block(int indent) {
    skip_blank();
    YNode n;
    if (pos >= lines.size()) return n;
    const Line& first = lines[pos];
    n.line = first.no;
    n.column = first.indent + 1;
    if (is_seq_item(first.content)) {
      n.kind = YNode::Seq;
      while (true) {
        skip_blank();
        if (pos >= lines.size()) break;
        const Line& L = lines[pos];
        if (L.indent != indent || !is_seq_item(L.content)) {
          if (L.indent > indent) err(L.no, L.indent + 1, "bad indentation in sequence");
          break;
        }
        size_t li = pos++;
        std::string rest = L.content.size() > 1 ? L.content.substr(2) : "";
        n.seq.push_back(inline_value(rest, static_cast<int>(li), L.indent + 3, indent));
        if (failed) break;
      }
      return n;
    }
    if (key_colon(first.content) != std::string::npos) {
      n.kind = YNode::Map;
      while (true) {
        skip_blank();
        if (pos >= lines.size()) break;
        const Line& L = lines[pos];
        if (L.indent < indent) break;
        if (L.indent > indent) {
          err(L.no, L.indent + 1, "bad indentation of a mapping entry");
          break;
        }
        size_t c = key_colon(L.content);
        if (c == std::string::npos) {
          err(L.no, L.indent + 1, "expected `key: value`");
          break;
        }
        std::string key = trim(L.content.substr(0, c));
        if (key.size() >= 2 && (key[0] == '"' || key[0] == '\'')) key = key.substr(1, key.size() - 2);
        for (const auto& [k, v] : n.map)
          if (k == key) {
            err(L.no, L.indent + 1, "duplicate key '" + key + "'");
          }
        size_t li = pos++;
        std::string rest = L.content.substr(c + 1);
        n.map.emplace_back(key, inline_value(rest, static_cast<int>(li), L.indent + static_cast<int>(c) + 2, indent));
        if (failed) break;
      }
      return n;
    }
    size_t li = pos++;
    return inline_value(first.content, static_cast<int>(li), first.indent + 1, indent - 1);
  }
};

}  // namespace

std::optional<YNode> yaml_parse(const std::string& text, const std::string& file, DiagList& diags) {
  Parser p(text, file, diags);
  if (p.failed) return std::nullopt;
  p.skip_blank();
  YNode root;
  if (p.pos < p.lines.size()) root = p.block(p.lines[p.pos].indent);
  p.skip_blank();
  if (!p.failed && p.pos < p.lines.size())
    p.err(p.lines[p.pos].no, p.lines[p.pos].indent + 1, "unexpected content at lower indentation");
  if (p.failed) return std::nullopt;
  return root;
}

}  // namespace lf
