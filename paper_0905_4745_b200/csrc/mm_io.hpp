// Dense complex Matrix Market I/O (include/minnorm/matrix_market.hpp of the reference).
#pragma once

#include <string>

#include "common_host.hpp"

namespace mnb {

// minnorm::ParseError (include/minnorm/errors.hpp:34-49): 1-based line / column, 0 when unknown.
struct ParseFail : Error {
    int64_t line, column;
    explicit ParseFail(const std::string& what, int64_t l = 0, int64_t c = 0)
        : Error(MNB_ERR_PARSE, l == 0 ? what : what + " (line " + std::to_string(l) + ", column " + std::to_string(c) + ")"),
          line(l), column(c) {}
};

void mm_dims(const std::string& path, int64_t* rows, int64_t* cols);              // header + size line
void mm_read(const std::string& path, double* out, int64_t rows, int64_t cols);  // column-major re,im pairs
void mm_write(const std::string& path, const double* data, int64_t rows, int64_t cols);

}  // namespace mnb
