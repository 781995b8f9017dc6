// Dense complex Matrix Market I/O: the file format of the reference's front end
// (include/minnorm/matrix_market.hpp; src/matrix_market.cpp:65-130), host side.
//
// Format: header line "%%MatrixMarket matrix array complex general" (case-insensitive),
// '%' comment lines and blank lines, a size line "rows cols", then rows*cols entries in
// column-major order, one "real imag" pair per line (comment / blank lines may appear
// between entries).  Values are written with 17 significant digits ("%.17g %.17g"), so
// equal values round-trip to byte-identical files.  Malformed input raises
// ParseError with the reference's 1-based line / column.
//
// The whole file is read into memory once and scanned in place (std::from_chars), so a
// 2 GiB text matrix parses at memory speed instead of stream-extraction speed.
#include "mm_io.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>

namespace mnb {

namespace {

constexpr const char* kHeader = "%%matrixmarket matrix array complex general";

struct Text {
    std::unique_ptr<char[]> buf;
    size_t size = 0;
};

Text slurp(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw ParseFail("cannot open '" + path + "' for reading");
    Text t;
    std::fseek(f, 0, SEEK_END);
    const long len = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    t.size = len > 0 ? size_t(len) : 0;
    t.buf.reset(new char[t.size + 1]);
    if (t.size && std::fread(t.buf.get(), 1, t.size, f) != t.size) {
        std::fclose(f);
        throw ParseFail("cannot read '" + path + "'");
    }
    std::fclose(f);
    t.buf[t.size] = '\n';
    return t;
}

// Line cursor over the buffer: [b, e) is the current line without its '\n' (and '\r').
struct Lines {
    const char* p;
    const char* end;
    const char* b = nullptr;
    const char* e = nullptr;
    int64_t number = 0;

    bool next() {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
        b = p;
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        if (e > b && e[-1] == '\r') --e;
        ++number;
        return true;
    }
    bool skippable() const {  // comment or blank
        if (b < e && *b == '%') return true;
        for (const char* q = b; q < e; ++q)
            if (*q != ' ' && *q != '\t') return false;
        return true;
    }
};

// Exactly `count` doubles on the line [b, e); errors carry the 1-based column of the offending character.
void parse_fields(const char* b, const char* e, int64_t lineno, double* out, int count) {
    const char* p = b;
    for (int k = 0; k < count; ++k) {
        while (p < e && (*p == ' ' || *p == '\t')) ++p;
        if (p == e)
            throw ParseFail("expected " + std::to_string(count) + " numeric fields", lineno, int64_t(p - b) + 1);
        const auto [next, ec] = std::from_chars(p, e, out[k]);
        if (ec != std::errc{} || (next < e && *next != ' ' && *next != '\t'))
            throw ParseFail("malformed number", lineno, int64_t(p - b) + 1);
        p = next;
    }
    while (p < e && (*p == ' ' || *p == '\t')) ++p;
    if (p != e)
        throw ParseFail("trailing characters after " + std::to_string(count) + " fields", lineno, int64_t(p - b) + 1);
}

// Header + comments + size line; leaves the cursor on the size line.
void read_header(Lines& L, int64_t* rows, int64_t* cols) {
    if (!L.next()) throw ParseFail("empty file", 1, 1);
    std::string h(L.b, L.e);
    std::transform(h.begin(), h.end(), h.begin(), [](unsigned char c) { return char(std::tolower(c)); });
    if (h != kHeader)
        throw ParseFail("unsupported header; expected \"%%MatrixMarket matrix array complex general\"", 1, 1);
    for (;;) {
        if (!L.next()) throw ParseFail("missing size line", L.number + 1, 1);
        if (!L.skippable()) break;
    }
    double dims[2];
    parse_fields(L.b, L.e, L.number, dims, 2);
    if (dims[0] < 1 || dims[1] < 1 || dims[0] != std::floor(dims[0]) || dims[1] != std::floor(dims[1]))
        throw ParseFail("size line must hold two positive integers", L.number, 1);
    *rows = int64_t(dims[0]);
    *cols = int64_t(dims[1]);
}

}  // namespace

void mm_dims(const std::string& path, int64_t* rows, int64_t* cols) {
    // only the head of the file is needed: the header, the comments and the size line
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseFail("cannot open '" + path + "' for reading");
    std::string head, line;
    while (std::getline(in, line)) {
        head += line;
        head += '\n';
        const bool comment_or_blank = (!line.empty() && line[0] == '%') ||
                                      line.find_first_not_of(" \t\r") == std::string::npos;
        if (head.size() > line.size() + 1 && !comment_or_blank) break;  // the size line
    }
    Lines L{head.data(), head.data() + head.size()};
    read_header(L, rows, cols);
}

void mm_read(const std::string& path, double* out, int64_t rows, int64_t cols) {
    Text t = slurp(path);
    Lines L{t.buf.get(), t.buf.get() + t.size};
    int64_t r = 0, c = 0;
    read_header(L, &r, &c);
    if (r != rows || c != cols) throw ParseFail("size line changed between reads of '" + path + "'");
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) {
            do {
                if (!L.next())
                    throw ParseFail("file ends before entry " + std::to_string(i + 1) + "," + std::to_string(j + 1),
                                    L.number + 1, 1);
            } while (L.skippable());
            parse_fields(L.b, L.e, L.number, out + 2 * (j * rows + i), 2);
        }
}

void mm_write(const std::string& path, const double* data, int64_t rows, int64_t cols) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw Error(MNB_ERR_INVALID_ARGUMENT, "cannot open '" + path + "' for writing");
    std::string buf = "%%MatrixMarket matrix array complex general\n" + std::to_string(rows) + " " +
                      std::to_string(cols) + "\n";
    char line[96];
    const int64_t total = rows * cols;
    for (int64_t k = 0; k < total; ++k) {
        const int len = std::snprintf(line, sizeof line, "%.17g %.17g\n", data[2 * k], data[2 * k + 1]);
        buf.append(line, size_t(len));
        if (buf.size() > (size_t(1) << 22)) {
            if (std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) break;
            buf.clear();
        }
    }
    const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size() && std::fclose(f) == 0;
    if (!ok) throw Error(MNB_ERR_INVALID_ARGUMENT, "failed while writing '" + path + "'");
}

}  // namespace mnb
