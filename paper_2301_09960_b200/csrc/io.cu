// io.cu -- MPMAT v1 matrix files behind the C-ABI (host code only).
//
// Format (proj/include/mpmat/matrix_io.hpp:8-13, proj/src/matrix_io.cpp):
//   MPMAT v1 <tag> <m> <n>\n
//   one matrix row per line; elements separated by one space; an element is
//   its K words as C99 hex-float literals ("%a") separated by one space.
// Tags d / dd / td / qd (K = 1..4).  Reading accepts any whitespace between
// tokens (the reference reads with operator>> and strtod); each element must
// parse completely (matrix_io.cpp:47-69, multifloat.hpp:335-350).  "ts"
// (three binary32 words) is this build's extension for the triple-single
// format the reference does not have; its words are written as the equal
// binary64 literals, so reading them back is exact.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ozk.h"
#include "ozk_internal.cuh"

namespace {

ozk_status io_fail(const std::string& msg) {
    ozk::set_last_error(msg);
    return OZK_EIO;
}

const char* tag_of(int fmt) {
    switch (fmt) {
    case OZK_D: return "d";
    case OZK_DD: return "dd";
    case OZK_TD: return "td";
    case OZK_QD: return "qd";
    case OZK_TS: return "ts";
    default: return nullptr;
    }
}
int fmt_of_tag(const std::string& t) {
    if (t == "d") return OZK_D;
    if (t == "dd") return OZK_DD;
    if (t == "td") return OZK_TD;
    if (t == "qd") return OZK_QD;
    if (t == "ts") return OZK_TS;
    return 0;
}
int words_of_fmt(int fmt) { return fmt == OZK_TS ? 3 : fmt; }

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

// Whitespace-separated token reader over a FILE (the reference's operator>>).
bool next_token(FILE* f, std::string& tok) {
    tok.clear();
    int c;
    do {
        c = std::fgetc(f);
    } while (c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f');
    while (c != EOF && !(c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f')) {
        tok.push_back((char)c);
        c = std::fgetc(f);
    }
    return !tok.empty();
}

ozk_status read_header(FILE* f, int* fmt, size_t* m, size_t* n) {
    std::string magic, version, tag, sm, sn;
    if (!next_token(f, magic) || !next_token(f, version) || !next_token(f, tag) ||
        !next_token(f, sm) || !next_token(f, sn))
        return io_fail("read_matrix: bad header");
    char* end = nullptr;
    const unsigned long long mm = std::strtoull(sm.c_str(), &end, 10);
    if (*end) return io_fail("read_matrix: bad header");
    const unsigned long long nn = std::strtoull(sn.c_str(), &end, 10);
    if (*end) return io_fail("read_matrix: bad header");
    if (magic != "MPMAT" || version != "v1") return io_fail("read_matrix: not an MPMAT v1 file");
    *fmt = fmt_of_tag(tag);
    if (!*fmt) return io_fail("read_matrix: unknown precision tag " + tag);
    *m = (size_t)mm;
    *n = (size_t)nn;
    return OZK_OK;
}

}  // namespace

extern "C" {

ozk_status ozk_mpmat_write(const char* path, int fmt, size_t m, size_t n, const void* a) {
    const char* tag = tag_of(fmt);
    if (!tag) return io_fail("write_matrix: unknown format");
    if (!path || !a) return io_fail("write_matrix: null argument");
    File out;
    out.f = std::fopen(path, "w");
    if (!out.f) return io_fail(std::string("cannot open for writing: ") + path);
    const int K = words_of_fmt(fmt);
    std::fprintf(out.f, "MPMAT v1 %s %zu %zu\n", tag, m, n);
    std::vector<char> line;
    char buf[48];
    for (size_t i = 0; i < m; ++i) {
        line.clear();
        for (size_t j = 0; j < n; ++j) {
            for (int k = 0; k < K; ++k) {
                const size_t idx = (i * n + j) * K + k;
                const double v = fmt == OZK_TS ? (double)static_cast<const float*>(a)[idx]
                                               : static_cast<const double*>(a)[idx];
                const int len = std::snprintf(buf, sizeof buf, "%a", v);
                if (j || k) line.push_back(' ');
                line.insert(line.end(), buf, buf + len);
            }
        }
        line.push_back('\n');
        if (std::fwrite(line.data(), 1, line.size(), out.f) != line.size())
            return io_fail("write_matrix: stream failure");
    }
    if (std::fflush(out.f) != 0) return io_fail("write_matrix: stream failure");
    return OZK_OK;
}

ozk_status ozk_mpmat_read_header(const char* path, int* fmt, size_t* m, size_t* n) {
    if (!path || !fmt || !m || !n) return io_fail("read_matrix: null argument");
    File in;
    in.f = std::fopen(path, "r");
    if (!in.f) return io_fail(std::string("cannot open for reading: ") + path);
    return read_header(in.f, fmt, m, n);
}

ozk_status ozk_mpmat_read(const char* path, int fmt, size_t m, size_t n, void* a) {
    const char* want = tag_of(fmt);
    if (!want) return io_fail("read_matrix: unknown format");
    if (!path || !a) return io_fail("read_matrix: null argument");
    File in;
    in.f = std::fopen(path, "r");
    if (!in.f) return io_fail(std::string("cannot open for reading: ") + path);
    int got = 0;
    size_t fm = 0, fn = 0;
    if (ozk_status s = read_header(in.f, &got, &fm, &fn)) return s;
    if (got != fmt)
        return io_fail(std::string("read_matrix: precision tag mismatch: expected ") + want +
                       ", got " + tag_of(got));
    if (fm == 0 || fn == 0) return io_fail("read_matrix: bad dimensions");
    if (fm != m || fn != n) return io_fail("read_matrix: dimensions differ from the buffer's");
    const int K = words_of_fmt(fmt);
    std::string tok, joined;
    for (size_t e = 0; e < m * n; ++e) {
        joined.clear();
        for (int k = 0; k < K; ++k) {
            if (!next_token(in.f, tok)) return io_fail("read_matrix: truncated row");
            if (k) joined += ' ';
            joined += tok;
            char* end = nullptr;
            const double v = std::strtod(tok.c_str(), &end);
            if (end != tok.c_str() + tok.size()) {
                // the whole element is reported, as the reference does
                for (int r = k + 1; r < K && next_token(in.f, tok); ++r) joined += ' ' + tok;
                return io_fail("read_matrix: bad element: " + joined);
            }
            if (fmt == OZK_TS) {
                const float w = (float)v;
                if ((double)w != v && v == v)
                    return io_fail("read_matrix: bad element (not a binary32 word): " + joined);
                static_cast<float*>(a)[e * K + k] = w;
            } else {
                static_cast<double*>(a)[e * K + k] = v;
            }
        }
    }
    return OZK_OK;
}

}  // extern "C"
