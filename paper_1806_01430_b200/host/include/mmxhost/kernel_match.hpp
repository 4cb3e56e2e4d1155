// kernel_match.hpp -- derives the loop catalogue the CUDA kernel library serves from the SOURCE, instead of
// trusting a hard-coded table: every loop nest of a C file is parsed (canonical `for` headers, one innermost
// statement) and matched against the idioms the library has kernels for.
//
// The reference has no counterpart: it hands each candidate loop to an OpenACC compiler
// (/root/reference/proj/src/evaluator.cpp:61-142) and never looks inside a loop body.  A kernel-library backend
// must know WHAT each loop computes; this is the step in front of the hot path.
//
//   idiom (innermost statement; i, j, k = induction variables by depth; N = the common bound)    kernels by depth
//   FillAffine   W[i][j] = (T)(i + j) / N        or (i - j)            fill2d<init_a|init_b>, fill_row<...>
//   FillZero     W[i][j] = 0.0                                          fill2d<zero>, fill_row<zero>
//   Transpose    W[i][j] = R[j][i]                                      transpose_tiled, transpose_row_gather
//   Contraction  W[i][j] += A[i][k] * B[j][k]    (either factor order)  matmul_nt, gemv_row, dot_rows
//   DiagonalSum  s += C[i][i]                                           trace_diag
// Anything else is Unknown: no kernel, and `tune` with the cuda backend refuses the source (ConfigError).
// The arrays each nest reads and writes give the producer -> consumer edges the residency planner moves data
// along (csrc/plan.cpp); tests check the derived edges against the planner's.
#pragma once

#include <string>
#include <vector>

#include "mmxhost/source_model.hpp"

namespace mmxhost {

enum class LoopIdiom { FillAffine, FillZero, Transpose, Contraction, DiagonalSum, Unknown };
std::string_view to_string(LoopIdiom idiom);

// for (int v = 0; v < N; v++)  -- also `++v`, `v += 1`, no declaration, unsigned / long / size_t types
struct LoopHeader {
  bool canonical = false;
  std::string var, lower, bound;
};

struct KernelBinding {
  int loop_id = 0;
  std::size_t line = 0;
  int depth = 0;
  int nest = -1;             // index of the enclosing depth-0 loop among the depth-0 loops, document order
  LoopHeader header;
  LoopIdiom idiom = LoopIdiom::Unknown;  // of the nest this loop belongs to
  std::string kernel;        // kernel family serving the loop; empty = none
  std::string writes;        // array (or scalar) the nest's statement assigns
  std::vector<std::string> reads;
  std::string why_unmatched; // empty when a kernel was found
};

std::vector<KernelBinding> match_kernels(const SourceUnit& unit, const std::vector<LoopSite>& loops);

// producer nest -> consumer nest for every array written by one matched nest and read by a later one
struct DataflowEdge {
  std::string array;
  int producer_nest = 0, consumer_nest = 0;
};
std::vector<DataflowEdge> derive_dataflow(const std::vector<KernelBinding>& bindings);

}  // namespace mmxhost
