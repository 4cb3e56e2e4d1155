// source_model.cpp -- tokenizer + statement parser behind scan_loops, and the variant renderer.
// Contract: /root/reference/proj/src/source_model.cpp:57-376 (lexer modes, statement walk, render_variant).
#include "mmxhost/source_model.hpp"

#include "tokens.hpp"

#include <algorithm>
#include <cctype>
#include <fstream>
#include <sstream>
#include <utility>

namespace mmxhost {
namespace {

std::vector<std::size_t> index_lines(std::string_view text) {
  std::vector<std::size_t> starts{0};
  for (std::size_t i = 0; i < text.size(); ++i)
    if (text[i] == '\n') starts.push_back(i + 1);
  return starts;
}

bool ident_char(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }

// Code tokens only.  Dropped: // and /* */ comments, "..." and '...' literals (with escapes), and preprocessor
// lines (a '#' first on its line, continued by trailing backslashes).
}  // namespace

namespace detail {

std::vector<Token> tokenize(const SourceUnit& unit) {
  const std::string_view t = unit.text;
  std::vector<Token> out;
  auto fail = [&](std::size_t at, const char* what) -> void {
    throw ScanError(std::string(what) + " near line " + std::to_string(unit.line_of(std::min(at, t.size() ? t.size() - 1 : 0))) + " of " + unit.path);
  };
  bool line_has_code = false;  // a '#' opens a preprocessor line only as the first non-blank of its line
  std::size_t i = 0;
  while (i < t.size()) {
    const char c = t[i];
    if (c == '\n') { line_has_code = false; ++i; continue; }
    if (c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v') { ++i; continue; }
    if (c == '/' && i + 1 < t.size() && t[i + 1] == '/') {
      while (i < t.size() && t[i] != '\n') {
        if (t[i] == '\\' && i + 1 < t.size() && t[i + 1] == '\n') ++i;  // line splice keeps the comment going
        ++i;
      }
      continue;
    }
    if (c == '/' && i + 1 < t.size() && t[i + 1] == '*') {
      const std::size_t end = t.find("*/", i + 2);
      if (end == std::string_view::npos) fail(i, "unterminated comment");
      i = end + 2;
      continue;
    }
    if (c == '#' && !line_has_code) {
      while (i < t.size() && t[i] != '\n') {
        if (t[i] == '\\' && i + 1 < t.size() && t[i + 1] == '\n') ++i;
        ++i;
      }
      continue;
    }
    line_has_code = true;
    if (c == '"' || c == '\'') {
      std::size_t j = i + 1;
      while (j < t.size() && t[j] != c) {
        if (t[j] == '\n') fail(i, "unterminated literal");
        if (t[j] == '\\') ++j;
        ++j;
      }
      if (j >= t.size()) fail(i, "unterminated literal");
      i = j + 1;
      continue;
    }
    if (ident_char(c)) {
      std::size_t j = i;
      while (j < t.size() && ident_char(t[j])) ++j;
      out.push_back({Token::Word, i, t.substr(i, j - i)});
      i = j;
      continue;
    }
    out.push_back({Token::Punct, i, t.substr(i, 1)});
    ++i;
  }
  return out;
}

}  // namespace detail

namespace {

using detail::Token;
using detail::tokenize;

class Parser {
 public:
  Parser(const SourceUnit& unit, const std::vector<Token>& tokens) : unit_(unit), tok_(tokens) {}

  std::vector<LoopSite> run() {
    std::size_t p = 0;
    while (p < tok_.size()) p = statement(p, 0);
    return std::move(sites_);
  }

 private:
  const SourceUnit& unit_;
  const std::vector<Token>& tok_;
  std::vector<LoopSite> sites_;

  bool punct(std::size_t p, char c) const { return p < tok_.size() && tok_[p].kind == Token::Punct && tok_[p].s[0] == c; }
  bool word(std::size_t p, std::string_view w) const { return p < tok_.size() && tok_[p].kind == Token::Word && tok_[p].s == w; }
  // byte offset one past token p-1 (the end of what has been consumed)
  std::size_t end_offset(std::size_t p) const {
    if (p == 0) return 0;
    return tok_[p - 1].at + tok_[p - 1].s.size();
  }
  [[noreturn]] void fail(std::size_t p, const std::string& what) const {
    const std::size_t at = p < tok_.size() ? tok_[p].at : (unit_.text.empty() ? 0 : unit_.text.size() - 1);
    throw ScanError(what + " near line " + std::to_string(unit_.line_of(at)) + " of " + unit_.path);
  }

  // p on the opening delimiter; returns the index one past its partner
  std::size_t balanced(std::size_t p, char open, char close) const {
    long depth = 0;
    for (std::size_t q = p; q < tok_.size(); ++q) {
      if (punct(q, open)) ++depth;
      if (punct(q, close) && --depth == 0) return q + 1;
    }
    fail(p, std::string("unterminated '") + open + "' group");
  }

  std::size_t block(std::size_t p, int depth) {  // p on '{'
    std::size_t q = p + 1;
    for (;;) {
      if (q >= tok_.size()) fail(p, "unterminated '{' block");
      if (punct(q, '}')) return q + 1;
      q = statement(q, depth);
    }
  }

  std::size_t paren_then_body(std::size_t p, int depth, std::size_t at, const char* what) {
    if (punct(p, '(')) p = balanced(p, '(', ')');
    if (p >= tok_.size()) fail(at, what);
    return statement(p, depth);
  }

  std::size_t statement(std::size_t p, int depth) {
    if (punct(p, '{')) return block(p, depth);
    if (punct(p, ';')) return p + 1;
    if (word(p, "for")) return for_statement(p, depth);
    if (word(p, "if")) {
      std::size_t q = paren_then_body(p + 1, depth, p, "if without a body");
      if (word(q, "else")) {
        if (q + 1 >= tok_.size()) fail(p, "else without a body");
        return statement(q + 1, depth);
      }
      return q;
    }
    if (word(p, "while") || word(p, "switch")) return paren_then_body(p + 1, depth, p, "loop/switch without a body");
    if (word(p, "do")) {
      if (p + 1 >= tok_.size()) fail(p, "do without a body");
      std::size_t q = statement(p + 1, depth);
      if (word(q, "while")) {
        ++q;
        if (punct(q, '(')) q = balanced(q, '(', ')');
        if (punct(q, ';')) ++q;
      }
      return q;
    }
    // expression, declaration or definition: ends at a ';' outside parentheses; brace groups on the way (function
    // bodies, initialiser lists) are parsed for loops, and one at parenthesis depth 0 that is not followed by ';'
    // ends the statement (a function definition)
    long paren = 0;
    std::size_t q = p;
    while (q < tok_.size()) {
      if (punct(q, '(') || punct(q, '[')) {
        ++paren;
      } else if (punct(q, ')') || punct(q, ']')) {
        --paren;
      } else if (punct(q, '{')) {
        q = block(q, depth);
        if (paren > 0) continue;
        return punct(q, ';') ? q + 1 : q;
      } else if (punct(q, ';') && paren <= 0) {
        return q + 1;
      } else if (punct(q, '}')) {
        return q;  // malformed statement running into the enclosing block: let the caller see the brace
      }
      ++q;
    }
    return q;
  }

  std::size_t for_statement(std::size_t p, int depth) {
    LoopSite site;
    site.header_start = tok_[p].at;
    site.depth = depth;
    site.line = unit_.line_of(site.header_start);
    const std::size_t ls = unit_.line_start_of(site.header_start);
    std::size_t we = ls;
    while (we < unit_.text.size() && (unit_.text[we] == ' ' || unit_.text[we] == '\t')) ++we;
    site.indent = unit_.text.substr(ls, we - ls);
    if (!punct(p + 1, '(')) fail(p, "for without a '(' header");
    const std::size_t body = balanced(p + 1, '(', ')');
    if (body >= tok_.size()) fail(p, "for without a body");
    const std::size_t index = sites_.size();  // ids follow header order
    site.id = static_cast<int>(index);
    site.body_begin = tok_[body].at;
    sites_.push_back(site);
    const std::size_t after = statement(body, depth + 1);
    sites_[index].body_end = end_offset(after);
    return after;
  }
};

}  // namespace

SourceUnit SourceUnit::from_string(std::string path, std::string text) {
  SourceUnit u;
  u.path = std::move(path);
  u.text = std::move(text);
  u.line_starts = index_lines(u.text);
  return u;
}

SourceUnit SourceUnit::from_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError("cannot read source file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return from_string(path, ss.str());
}

std::size_t SourceUnit::line_of(std::size_t offset) const {
  const auto it = std::upper_bound(line_starts.begin(), line_starts.end(), offset);
  return static_cast<std::size_t>(it - line_starts.begin());
}

std::size_t SourceUnit::line_start_of(std::size_t offset) const { return line_starts[line_of(offset) - 1]; }

std::vector<LoopSite> scan_loops(const SourceUnit& unit) {
  const std::vector<Token> tokens = tokenize(unit);
  return Parser(unit, tokens).run();
}

CandidateSet all_loops_candidate_set(SourceUnit unit) {
  CandidateSet cs;
  cs.unit = std::move(unit);
  cs.all_loops = scan_loops(cs.unit);
  for (const LoopSite& l : cs.all_loops) cs.candidate_ids.push_back(l.id);
  return cs;
}

std::string render_variant(const CandidateSet& cs, const Genome& genome) {
  if (genome.size() != cs.gene_length())
    throw GenomeLengthMismatch("genome length " + std::to_string(genome.size()) + " does not match gene length " +
                               std::to_string(cs.gene_length()));
  // insertion points are line starts of the ORIGINAL text, so nothing existing is ever split; the stable sort keeps
  // directives of loops that share a line in gene order
  std::vector<std::pair<std::size_t, std::string>> inserts;
  for (std::size_t k = 0; k < genome.size(); ++k) {
    if (!genome.test(k)) continue;
    const LoopSite& site = cs.candidate(k);
    inserts.emplace_back(cs.unit.line_start_of(site.header_start), site.indent + std::string(kOffloadDirective) + "\n");
  }
  std::stable_sort(inserts.begin(), inserts.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::string out;
  std::size_t from = 0;
  for (const auto& [at, line] : inserts) {
    out.append(cs.unit.text, from, at - from);
    out.append(line);
    from = at;
  }
  out.append(cs.unit.text, from, std::string::npos);
  return out;
}

std::string strip_directives(std::string_view text) {
  std::string out;
  std::size_t pos = 0;
  while (pos < text.size()) {
    std::size_t nl = text.find('\n', pos);
    const std::size_t end = nl == std::string_view::npos ? text.size() : nl + 1;
    std::string_view line = text.substr(pos, end - pos);
    std::size_t b = 0;
    while (b < line.size() && (line[b] == ' ' || line[b] == '\t')) ++b;
    std::string_view rest = line.substr(b);
    while (!rest.empty() && (rest.back() == '\n' || rest.back() == '\r')) rest.remove_suffix(1);
    if (rest != kOffloadDirective) out.append(line);
    pos = end;
  }
  return out;
}

}  // namespace mmxhost
