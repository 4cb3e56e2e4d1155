// kernel_match.cpp -- loop nest -> kernel family by idiom (see kernel_match.hpp).
#include "mmxhost/kernel_match.hpp"

#include <algorithm>
#include <cctype>
#include <cstdlib>

#include "tokens.hpp"

namespace mmxhost {

using detail::Token;

std::string_view to_string(LoopIdiom idiom) {
  switch (idiom) {
    case LoopIdiom::FillAffine: return "fill_affine";
    case LoopIdiom::FillZero: return "fill_zero";
    case LoopIdiom::Transpose: return "transpose";
    case LoopIdiom::Contraction: return "contraction";
    case LoopIdiom::DiagonalSum: return "diagonal_sum";
    case LoopIdiom::Unknown: break;
  }
  return "unknown";
}

namespace {

struct Cursor {
  const Token* t;
  std::size_t p, end;

  bool done() const { return p >= end; }
  bool punct(char c) const { return p < end && t[p].kind == Token::Punct && t[p].s[0] == c; }
  bool word() const { return p < end && t[p].kind == Token::Word; }
  bool word(std::string_view w) const { return word() && t[p].s == w; }
  bool eat(char c) {
    if (!punct(c)) return false;
    ++p;
    return true;
  }
  bool eat_word(std::string_view w) {
    if (!word(w)) return false;
    ++p;
    return true;
  }
  bool take_word(std::string& out) {
    if (!word()) return false;
    out = std::string(t[p].s);
    ++p;
    return true;
  }
};

bool is_type_word(std::string_view w) {
  static constexpr std::string_view ty[] = {"int", "long", "unsigned", "signed", "short", "size_t", "ptrdiff_t", "const", "register"};
  return std::find(std::begin(ty), std::end(ty), w) != std::end(ty);
}

std::size_t token_at(const std::vector<Token>& t, std::size_t offset) {
  return static_cast<std::size_t>(std::lower_bound(t.begin(), t.end(), offset, [](const Token& x, std::size_t at) { return x.at < at; }) - t.begin());
}

// tokens of `for ( ... )`: c.p on '(' -> parses `[type] v = lo ; v < bound ; step`
LoopHeader parse_header(Cursor c) {
  LoopHeader h;
  if (!c.eat('(')) return h;
  while (c.word() && is_type_word(c.t[c.p].s)) ++c.p;
  if (!c.take_word(h.var) || !c.eat('=') || !c.take_word(h.lower) || !c.eat(';')) return h;
  if (!c.eat_word(h.var) || !c.eat('<') || !c.take_word(h.bound) || !c.eat(';')) return h;
  bool step = false;
  if (c.eat_word(h.var)) {
    if (c.eat('+')) step = c.eat('+') || (c.eat('=') && c.eat_word("1"));
  } else if (c.eat('+') && c.eat('+')) {
    step = c.eat_word(h.var);
  }
  h.canonical = step && c.eat(')') && std::isdigit(static_cast<unsigned char>(h.lower[0])) != 0;
  return h;
}

// X [ a ] [ b ]
bool take_ref2(Cursor& c, std::string& name, std::string& a, std::string& b) {
  Cursor s = c;
  if (!s.take_word(name) || !s.eat('[') || !s.take_word(a) || !s.eat(']') || !s.eat('[') || !s.take_word(b) || !s.eat(']')) return false;
  c = s;
  return true;
}

struct Nest {
  std::vector<int> chain;  // loop indexes (into `loops`), outermost first; perfectly nested
};

}  // namespace

std::vector<KernelBinding> match_kernels(const SourceUnit& unit, const std::vector<LoopSite>& loops) {
  const std::vector<Token> tok = detail::tokenize(unit);
  std::vector<KernelBinding> out(loops.size());
  int nest_count = 0;
  std::vector<int> nest_of(loops.size(), -1);
  for (std::size_t k = 0; k < loops.size(); ++k) {
    const LoopSite& s = loops[k];
    KernelBinding& b = out[k];
    b.loop_id = s.id;
    b.line = s.line;
    b.depth = s.depth;
    if (s.depth == 0) nest_of[k] = nest_count++;
    else if (k > 0) nest_of[k] = nest_of[k - 1];  // document order: an inner loop follows its nest's loops
    b.nest = nest_of[k];
    Cursor c{tok.data(), token_at(tok, s.header_start) + 1, tok.size()};
    b.header = parse_header(c);
  }

  // a loop's body holds exactly one statement: returns the token range of that statement (braces stripped)
  auto single_statement = [&](const LoopSite& s, std::size_t& b, std::size_t& e) {
    b = token_at(tok, s.body_begin);
    e = token_at(tok, s.body_end);
    while (e - b >= 2 && tok[b].kind == Token::Punct && tok[b].s[0] == '{' && tok[e - 1].kind == Token::Punct && tok[e - 1].s[0] == '}') {
      ++b;
      --e;
    }
  };

  for (std::size_t root = 0; root < loops.size(); ++root) {
    if (loops[root].depth != 0) continue;
    // the chain of perfectly nested loops under this root
    std::vector<std::size_t> chain{root};
    std::string why;
    for (;;) {
      const LoopSite& cur = loops[chain.back()];
      std::size_t b, e;
      single_statement(cur, b, e);
      const std::size_t next = chain.back() + 1;
      const bool has_inner = next < loops.size() && loops[next].depth == cur.depth + 1 && loops[next].header_start < cur.body_end;
      if (!has_inner) break;
      if (b >= e || tok[b].at != loops[next].header_start || token_at(tok, loops[next].body_end) != e) {
        why = "loop nest is not perfectly nested";
        break;
      }
      chain.push_back(next);
    }
    // loops of this nest that are not on the chain (siblings, deeper imperfect nests)
    std::size_t nest_end = root + 1;
    while (nest_end < loops.size() && loops[nest_end].depth > 0) ++nest_end;
    if (why.empty() && nest_end - root != chain.size()) why = "loop nest is not perfectly nested";

    LoopIdiom idiom = LoopIdiom::Unknown;
    std::string writes, fill_op;
    std::vector<std::string> reads;
    std::vector<std::string> kernels;
    if (why.empty()) {
      std::vector<std::string> v;
      std::string bound;
      for (std::size_t k : chain) {
        const LoopHeader& h = out[k].header;
        if (!h.canonical || h.lower != "0") why = "loop header is not `for (v = 0; v < N; v++)`";
        else if (!bound.empty() && h.bound != bound) why = "loops of the nest have different bounds";
        bound = h.bound;
        v.push_back(h.var);
      }
      if (why.empty()) {
        std::size_t b, e;
        single_statement(loops[chain.back()], b, e);
        Cursor c{tok.data(), b, e};
        std::string w, x, y;
        if (v.size() == 2 && take_ref2(c, w, x, y) && x == v[0] && y == v[1] && c.eat('=')) {
          writes = w;
          Cursor r = c;
          std::string rn, ra, rb;
          if (take_ref2(r, rn, ra, rb) && ra == v[1] && rb == v[0] && r.eat(';') && r.done()) {
            idiom = LoopIdiom::Transpose;
            reads = {rn};
            kernels = {"transpose_tiled", "transpose_row_gather"};
          } else {
            // [ ( type ) ] ( i (+|-) j ) / N ;
            r = c;
            Cursor t2 = r;
            if (t2.eat('(') && t2.word() && (t2.t[t2.p].s == "double" || t2.t[t2.p].s == "float")) {
              ++t2.p;
              if (t2.eat(')')) r = t2;
            }
            Cursor a = r;
            char sign = 0;
            if (a.eat('(') && a.eat_word(v[0]) && ((a.punct('+') && (sign = '+')) || (a.punct('-') && (sign = '-'))) && (++a.p, true) &&
                a.eat_word(v[1]) && a.eat(')') && a.eat('/') && a.eat_word(bound) && a.eat(';') && a.done()) {
              idiom = LoopIdiom::FillAffine;
              fill_op = sign == '+' ? "init_a" : "init_b";
            } else if (c.p < e && tok[e - 1].kind == Token::Punct && tok[e - 1].s[0] == ';') {
              // a literal zero: the raw text between '=' and ';' parses as 0 with an optional f/F suffix
              const std::size_t from = tok[c.p].at, to = tok[e - 1].at;
              std::string lit = unit.text.substr(from, to - from);
              while (!lit.empty() && std::isspace(static_cast<unsigned char>(lit.back()))) lit.pop_back();
              if (!lit.empty() && (lit.back() == 'f' || lit.back() == 'F')) lit.pop_back();
              char* endp = nullptr;
              const double val = lit.empty() ? 1.0 : std::strtod(lit.c_str(), &endp);
              if (!lit.empty() && endp == lit.c_str() + lit.size() && val == 0.0 && std::isdigit(static_cast<unsigned char>(lit[0]))) {
                idiom = LoopIdiom::FillZero;
                fill_op = "zero";
              }
            }
            if (idiom != LoopIdiom::Unknown) kernels = {"fill2d<" + fill_op + ">", "fill_row<" + fill_op + ">"};
          }
        } else if (c = Cursor{tok.data(), b, e}; v.size() == 3 && take_ref2(c, w, x, y) && x == v[0] && y == v[1] && c.eat('+') && c.eat('=')) {
          std::string f1, f1a, f1b, f2, f2a, f2b;
          if (take_ref2(c, f1, f1a, f1b) && c.eat('*') && take_ref2(c, f2, f2a, f2b) && c.eat(';') && c.done() && f1b == v[2] && f2b == v[2]) {
            if (f1a == v[1] && f2a == v[0]) {  // B[j][k] * A[i][k]
              std::swap(f1, f2);
              std::swap(f1a, f2a);
            }
            if (f1a == v[0] && f2a == v[1]) {
              idiom = LoopIdiom::Contraction;
              writes = w;
              reads = {f1, f2, w};
              kernels = {"matmul_nt", "gemv_row", "dot_rows"};
            }
          }
        } else if (c = Cursor{tok.data(), b, e}; v.size() == 1 && c.take_word(w) && c.eat('+') && c.eat('=')) {
          std::string rn, ra, rb;
          if (take_ref2(c, rn, ra, rb) && ra == v[0] && rb == v[0] && c.eat(';') && c.done()) {
            idiom = LoopIdiom::DiagonalSum;
            writes = w;
            reads = {rn};
            kernels = {"trace_diag"};
          }
        }
        if (idiom == LoopIdiom::Unknown) why = "the nest's statement matches no kernel idiom";
      }
    }
    for (std::size_t k = root; k < nest_end; ++k) {
      KernelBinding& b = out[k];
      b.idiom = idiom;
      b.writes = writes;
      b.reads = reads;
      const auto pos = std::find(chain.begin(), chain.end(), k);
      if (idiom != LoopIdiom::Unknown && pos != chain.end() && static_cast<std::size_t>(pos - chain.begin()) < kernels.size())
        b.kernel = kernels[static_cast<std::size_t>(pos - chain.begin())];
      else
        b.why_unmatched = why.empty() ? "no kernel for this depth of the nest" : why;
    }
  }
  return out;
}

std::vector<DataflowEdge> derive_dataflow(const std::vector<KernelBinding>& bindings) {
  // one record per nest (its depth-0 loop carries the nest's reads and writes)
  std::vector<const KernelBinding*> nests;
  for (const KernelBinding& b : bindings)
    if (b.depth == 0) nests.push_back(&b);
  std::vector<DataflowEdge> edges;
  for (std::size_t q = 0; q < nests.size(); ++q)
    for (const std::string& r : nests[q]->reads) {
      // the latest earlier nest that wrote r
      for (std::size_t p = q; p-- > 0;)
        if (nests[p]->writes == r) {
          edges.push_back({r, nests[p]->nest, nests[q]->nest});
          break;
        }
    }
  return edges;
}

}  // namespace mmxhost
