// feasibility.cpp -- static accept/reject rules over the token stream (see feasibility.hpp).
#include "mmxhost/feasibility.hpp"

#include <algorithm>
#include <cctype>

#include "mmxhost/json_lite.hpp"
#include "tokens.hpp"

namespace mmxhost {

using detail::Token;

std::string_view to_string(RejectClass c) {
  switch (c) {
    case RejectClass::ExternalCall: return "external_call";
    case RejectClass::NestedOverlap: return "nested_overlap";
    case RejectClass::EarlyExit: return "early_exit";
    case RejectClass::DataDependency: return "data_dependency";
    case RejectClass::Other: break;
  }
  return "other";
}

namespace {

// words that may be followed by '(' without being a call (mockacc.cpp:117-124)
bool call_like_keyword(std::string_view w) {
  static constexpr std::string_view kw[] = {"if", "for", "while", "switch", "sizeof", "do", "else", "return", "case", "defined"};
  return std::find(std::begin(kw), std::end(kw), w) != std::end(kw);
}

bool all_digits(std::string_view w) {
  return !w.empty() && std::all_of(w.begin(), w.end(), [](char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; });
}

bool ends_with(std::string_view s, std::string_view suffix) {
  return s.size() >= suffix.size() && s.substr(s.size() - suffix.size()) == suffix;
}

// a `#pragma acc kernels` line: optional blanks, '#', optional blanks, the three words, then a non-word byte
bool is_directive_line(std::string_view line) {
  std::size_t i = 0;
  auto blanks = [&] { while (i < line.size() && (line[i] == ' ' || line[i] == '\t')) ++i; };
  auto word = [&](std::string_view w, bool need_blank_before) {
    const std::size_t start = i;
    blanks();
    if (need_blank_before && i == start) return false;
    if (line.substr(i, w.size()) != w) return false;
    i += w.size();
    return true;
  };
  blanks();
  if (i >= line.size() || line[i] != '#') return false;
  ++i;
  if (!word("pragma", false) || !word("acc", true) || !word("kernels", true)) return false;
  return i >= line.size() || !(std::isalnum(static_cast<unsigned char>(line[i])) || line[i] == '_');
}

}  // namespace

struct FeasibilityAnalyzer::Impl {
  const SourceUnit& unit;
  const std::vector<LoopSite>& loops;
  std::vector<Token> tokens;
  std::vector<int> pre;  // loops annotated by the source itself

  Impl(const SourceUnit& u, const std::vector<LoopSite>& l) : unit(u), loops(l), tokens(detail::tokenize(u)) {
    // every directive line of the raw text belongs to the first loop whose header starts after that line
    const std::string_view t = unit.text;
    std::size_t pos = 0;
    while (pos < t.size()) {
      std::size_t eol = t.find('\n', pos);
      if (eol == std::string_view::npos) eol = t.size();
      if (is_directive_line(t.substr(pos, eol - pos))) {
        for (const LoopSite& s : loops)
          if (s.header_start > eol) {
            if (pre.empty() || pre.back() != s.id) pre.push_back(s.id);
            break;
          }
      }
      pos = eol + 1;
    }
  }

  const LoopSite& site(int id) const {
    for (const LoopSite& s : loops)
      if (s.id == id) return s;
    throw Error("feasibility: unknown loop id " + std::to_string(id));
  }

  // token index range [first, last) of the loop body
  std::pair<std::size_t, std::size_t> body_tokens(const LoopSite& s) const {
    auto lo = std::lower_bound(tokens.begin(), tokens.end(), s.body_begin, [](const Token& t, std::size_t at) { return t.at < at; });
    auto hi = std::lower_bound(tokens.begin(), tokens.end(), s.body_end, [](const Token& t, std::size_t at) { return t.at < at; });
    return {static_cast<std::size_t>(lo - tokens.begin()), static_cast<std::size_t>(hi - tokens.begin())};
  }

  bool punct(std::size_t p, char c) const { return tokens[p].kind == Token::Punct && tokens[p].s[0] == c; }

  // rule 2: first word followed by '(' that is not a control keyword
  bool find_call(std::size_t b, std::size_t e, std::string& name) const {
    for (std::size_t p = b; p + 1 < e; ++p) {
      const Token& w = tokens[p];
      if (w.kind != Token::Word || std::isdigit(static_cast<unsigned char>(w.s[0]))) continue;
      if (punct(p + 1, '(') && !call_like_keyword(w.s)) {
        name = std::string(w.s);
        return true;
      }
    }
    return false;
  }

  // rule 3
  bool find_exit(std::size_t b, std::size_t e, std::string& word) const {
    for (std::size_t p = b; p < e; ++p) {
      const Token& w = tokens[p];
      if (w.kind == Token::Word && (w.s == "break" || w.s == "return" || w.s == "goto")) {
        word = std::string(w.s);
        return true;
      }
    }
    return false;
  }

  // rule 4: X [ I ] = <not '=' or ';'> ... (no ';') ... Y [ I (+|-) digits ]   with Y a suffix of X
  // (the reference's pattern is unanchored on the left of X, mockacc.cpp:198-199, so `xa[i] = a[i-1]` counts)
  bool find_dependence(std::size_t b, std::size_t e, std::string& name) const {
    for (std::size_t p = b; p + 5 < e; ++p) {
      if (tokens[p].kind != Token::Word || !punct(p + 1, '[') || tokens[p + 2].kind != Token::Word || !punct(p + 3, ']') ||
          !punct(p + 4, '='))
        continue;
      if (punct(p + 5, '=') || punct(p + 5, ';')) continue;
      // `=` must not be the tail of a compound operator or comparison: the byte before it has to be ']' or blank
      // (that is what "]\s*=" in the reference pattern demands)
      const std::size_t eq = tokens[p + 4].at, close = tokens[p + 3].at;
      bool only_blanks = true;
      for (std::size_t i = close + 1; i < eq; ++i)
        if (!std::isspace(static_cast<unsigned char>(unit.text[i]))) only_blanks = false;
      if (!only_blanks) continue;
      const std::string_view lhs = tokens[p].s, idx = tokens[p + 2].s;
      for (std::size_t q = p + 5; q + 5 < e + 1 && q + 5 <= e; ++q) {
        if (punct(q, ';')) break;
        if (tokens[q].kind == Token::Word && ends_with(lhs, tokens[q].s) && punct(q + 1, '[') && tokens[q + 2].kind == Token::Word &&
            tokens[q + 2].s == idx && (punct(q + 3, '-') || punct(q + 3, '+')) && tokens[q + 4].kind == Token::Word &&
            all_digits(tokens[q + 4].s) && q + 5 < e && punct(q + 5, ']')) {
          name = std::string(tokens[q].s);
          return true;
        }
      }
    }
    return false;
  }

  // the compiler reports lines of the VARIANT: every inserted directive line at or above the loop shifts it by one
  std::string located(const std::string& what, const LoopSite& s, const std::vector<int>& inserted) const {
    std::size_t line = s.line;
    for (int id : inserted)
      if (site(id).line <= s.line) ++line;
    return what + " (" + unit.path + ": line " + std::to_string(line) + ")";
  }

  // the rules for one annotated loop given the full annotation set (`inserted` = the loops whose directive the variant adds)
  ProbeResult judge(const LoopSite& s, const std::vector<int>& annotated, const std::vector<int>& inserted) const {
    ProbeResult r;
    r.loop_id = s.id;
    auto reject = [&](RejectClass c, const std::string& what) {
      r.verdict = ProbeVerdict::Rejected;
      r.reject_class = c;
      r.compiler_message = located(what, s, inserted);
      return r;
    };
    for (int other : annotated) {
      if (other == s.id) continue;
      const LoopSite& o = site(other);
      if (o.body_begin <= s.header_start && s.header_start < o.body_end) return reject(RejectClass::NestedOverlap, "compute regions may not be nested");
    }
    const auto [b, e] = body_tokens(s);
    std::string name;
    if (find_call(b, e, name)) return reject(RejectClass::ExternalCall, "call to '" + name + "' with no acc routine information");
    if (find_exit(b, e, name)) return reject(RejectClass::EarlyExit, "branching out of compute region ('" + name + "')");
    if (find_dependence(b, e, name)) return reject(RejectClass::DataDependency, "loop carried dependence of '" + name + "' prevents parallelization");
    r.verdict = ProbeVerdict::Parallelizable;
    return r;
  }

  std::vector<int> with_pre(std::vector<int> ids) const {
    ids.insert(ids.end(), pre.begin(), pre.end());
    std::sort(ids.begin(), ids.end(), [&](int x, int y) { return site(x).header_start < site(y).header_start; });
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    return ids;
  }
};

FeasibilityAnalyzer::FeasibilityAnalyzer(const SourceUnit& unit, const std::vector<LoopSite>& loops) : impl_(new Impl(unit, loops)) {}
FeasibilityAnalyzer::~FeasibilityAnalyzer() { delete impl_; }

const std::vector<int>& FeasibilityAnalyzer::preannotated() const { return impl_->pre; }

std::vector<ProbeResult> FeasibilityAnalyzer::check(const std::vector<int>& annotated) const {
  const std::vector<int> all = impl_->with_pre(annotated);
  std::vector<ProbeResult> rejected;
  for (int id : all) {
    ProbeResult r = impl_->judge(impl_->site(id), all, annotated);
    if (r.verdict == ProbeVerdict::Rejected) rejected.push_back(std::move(r));
  }
  return rejected;
}

ProbeResult FeasibilityAnalyzer::probe(int loop_id) const {
  impl_->site(loop_id);  // validates the id
  // the compiler judges the whole file: a diagnostic on ANY annotated loop fails the probe, and the log holds
  // all of them, one per line
  const std::vector<ProbeResult> rejected = check({loop_id});
  ProbeResult r;
  r.loop_id = loop_id;
  if (rejected.empty()) {
    r.verdict = ProbeVerdict::Parallelizable;
    return r;
  }
  r.verdict = ProbeVerdict::Rejected;
  // the log is classified as one text by ordered rules (probe.cpp:49-67): external call, nested, early exit, dependence
  static constexpr RejectClass order[] = {RejectClass::ExternalCall, RejectClass::NestedOverlap, RejectClass::EarlyExit,
                                          RejectClass::DataDependency};
  for (RejectClass c : order)
    if (std::any_of(rejected.begin(), rejected.end(), [&](const ProbeResult& x) { return x.reject_class == c; })) {
      r.reject_class = c;
      break;
    }
  for (const ProbeResult& x : rejected) {
    if (!r.compiler_message.empty()) r.compiler_message += "\n";
    r.compiler_message += x.compiler_message;
  }
  return r;
}

ProbeResult probe_loop(const SourceUnit& unit, const std::vector<LoopSite>& loops, int loop_id) {
  return FeasibilityAnalyzer(unit, loops).probe(loop_id);
}

CandidateSet build_candidate_set(const SourceUnit& unit, const std::vector<LoopSite>& loops, std::vector<ProbeResult>* report_out) {
  const FeasibilityAnalyzer an(unit, loops);
  std::vector<ProbeResult> results;
  results.reserve(loops.size());
  for (const LoopSite& s : loops) results.push_back(an.probe(s.id));
  if (report_out) *report_out = results;
  CandidateSet cs;
  cs.unit = unit;
  cs.all_loops = loops;
  for (std::size_t i = 0; i < loops.size(); ++i)
    if (results[i].verdict == ProbeVerdict::Parallelizable) cs.candidate_ids.push_back(loops[i].id);
  if (cs.candidate_ids.empty()) throw NoCandidates("probe rejected every loop; nothing to tune");
  return cs;
}

bool variant_feasible(const CandidateSet& cs, const Genome& genome, std::vector<ProbeResult>* rejected_out) {
  if (genome.size() != cs.gene_length())
    throw GenomeLengthMismatch("genome length " + std::to_string(genome.size()) + " does not match gene length " +
                               std::to_string(cs.gene_length()));
  std::vector<int> annotated;
  for (std::size_t k = 0; k < genome.size(); ++k)
    if (genome.test(k)) annotated.push_back(cs.candidate_ids[k]);
  std::vector<ProbeResult> rejected = FeasibilityAnalyzer(cs.unit, cs.all_loops).check(annotated);
  const bool ok = rejected.empty();
  if (rejected_out) *rejected_out = std::move(rejected);
  return ok;
}

std::string probe_report_jsonl(const SourceUnit& unit, const std::vector<LoopSite>& loops, const std::vector<ProbeResult>& results) {
  std::string out;
  for (const ProbeResult& r : results) {
    const auto it = std::find_if(loops.begin(), loops.end(), [&](const LoopSite& s) { return s.id == r.loop_id; });
    if (it == loops.end()) throw Error("probe report: unknown loop id " + std::to_string(r.loop_id));
    (void)unit;
    out += "{\"id\":" + std::to_string(r.loop_id) + ",\"line\":" + std::to_string(it->line) + ",\"verdict\":";
    out += r.verdict == ProbeVerdict::Parallelizable ? "\"parallelizable\"" : "\"rejected\"";
    out += ",\"reject_class\":";
    out += r.verdict == ProbeVerdict::Rejected ? json::dump_string(std::string(to_string(r.reject_class))) : std::string("null");
    out += ",\"message\":" + json::dump_string(r.compiler_message) + ",\"timed_out\":" + (r.timed_out ? "true" : "false") + "}\n";
  }
  return out;
}

}  // namespace mmxhost
