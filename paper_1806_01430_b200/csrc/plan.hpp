// plan.hpp -- genome -> execution plan (pure host code, no CUDA).
//
// Replaces, on this path, render_variant (/root/reference/proj/src/source_model.cpp:347-376)
// plus the accept/reject verdict the reference gets from its external compiler
// (nested compute regions are a compile error: tools/mockacc.cpp:205-221).
#pragma once

#include <cstddef>
#include <cstdint>

#include "mmx.h"

namespace mmx {

// Static facts about the 12 loops of fixtures/matmul.c.
struct LoopRow {
  int gene, line, depth, nest;
  const char* induction;
  const char* kernel;
};
extern const LoopRow kCatalogue[MMX_GENE_LENGTH];

// First gene of each nest and how many loops deep it is.
struct NestRow {
  int first_gene, depth_count;
};
extern const NestRow kNests[MMX_NUM_NESTS];

inline std::size_t elem_size(int dtype) { return dtype == MMX_F32 ? 4 : 8; }

// Fills `out`; returns MMX_OK or MMX_E_LENGTH / MMX_E_INVALID.
int build_plan(const std::uint8_t* bits, std::size_t gene_len, std::int32_t n, std::int32_t dtype,
               mmx_plan_info* out);

}  // namespace mmx
