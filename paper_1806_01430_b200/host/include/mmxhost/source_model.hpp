// source_model.hpp -- the loop catalogue of a C source file and the variant renderer.
//
// Mirrors the reference's scan_loops / render_variant contract
// (/root/reference/proj/include/acctune/source_model.hpp:58-88, src/source_model.cpp:342-376):
//   * every `for` statement outside comments, string / char literals and preprocessor lines, in document order,
//     with its for-nesting depth, the byte span of its body and the indentation of its line;
//   * gene k of a genome <-> all_loops[candidate_ids[k]];
//   * a variant is the original text with one line `indent + "#pragma acc kernels"` inserted at the start of
//     the line of every loop whose gene is 1 (all other bytes unchanged).
// On the CUDA path the catalogue is what ties a source file to the kernel library: CudaBackend serves exactly the
// catalogue of fixtures/matmul.c (mmx_loop_catalogue), and `tune` checks the scanned source against it; the
// renderer produces the `best/<source>` artifact a maintainer can hand to an OpenACC compiler.
//
// The implementation is a tokenizer (comments, literals, preprocessor lines dropped; every token keeps its byte
// offset) followed by a recursive statement parser over the token stream.
#pragma once

#include <cstddef>
#include <string>
#include <string_view>
#include <vector>

#include "mmxhost/errors.hpp"
#include "mmxhost/genome.hpp"

namespace mmxhost {

inline constexpr std::string_view kOffloadDirective = "#pragma acc kernels";

struct SourceUnit {
  std::string path;
  std::string text;
  std::vector<std::size_t> line_starts;  // line_starts[k] = offset of line k + 1

  static SourceUnit from_file(const std::string& path);  // ConfigError when unreadable
  static SourceUnit from_string(std::string path, std::string text);
  std::size_t line_of(std::size_t offset) const;        // 1-based
  std::size_t line_start_of(std::size_t offset) const;  // offset of the start of that line
};

struct LoopSite {
  int id = 0;                    // 0..n-1 in document order
  std::size_t header_start = 0;  // offset of the `for` keyword
  std::size_t body_begin = 0;    // loop body: brace block or single statement
  std::size_t body_end = 0;      // one past its last byte
  int depth = 0;                 // for-nesting depth, 0 = outermost
  std::string indent;            // whitespace prefix of the line holding the header
  std::size_t line = 0;          // 1-based line of the header
};

std::vector<LoopSite> scan_loops(const SourceUnit& unit);

struct CandidateSet {
  SourceUnit unit;
  std::vector<LoopSite> all_loops;
  std::vector<int> candidate_ids;  // document order, subset of loop ids

  std::size_t gene_length() const { return candidate_ids.size(); }
  const LoopSite& candidate(std::size_t gene) const { return all_loops[static_cast<std::size_t>(candidate_ids[gene])]; }
};

// every scanned loop is a candidate (what the reference does for the sim backend, commands.cpp:93-106)
CandidateSet all_loops_candidate_set(SourceUnit unit);

// GenomeLengthMismatch when genome.size() != cs.gene_length()
std::string render_variant(const CandidateSet& cs, const Genome& genome);

// Removes every line that consists of optional blanks + the directive: render followed by strip is the identity.
std::string strip_directives(std::string_view text);

}  // namespace mmxhost
