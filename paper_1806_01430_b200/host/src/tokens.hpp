// tokens.hpp -- the code-token stream shared by the loop scanner (source_model.cpp), the static feasibility
// rules (feasibility.cpp) and the kernel matcher (kernel_match.cpp).  Internal to the host library.
#pragma once

#include <cstddef>
#include <string_view>
#include <vector>

#include "mmxhost/source_model.hpp"

namespace mmxhost::detail {

struct Token {
  enum Kind { Word, Punct } kind;
  std::size_t at;      // byte offset in the source
  std::string_view s;  // the word (identifier, keyword or number), or one punctuation byte
};

// Code tokens only, in document order.  Dropped: // and /* */ comments, "..." and '...' literals (with escapes),
// and preprocessor lines (a '#' first on its line, continued by trailing backslashes).  Throws ScanError on an
// unterminated comment or literal.
std::vector<Token> tokenize(const SourceUnit& unit);

}  // namespace mmxhost::detail
