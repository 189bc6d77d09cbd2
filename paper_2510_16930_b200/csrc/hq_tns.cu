// hq_tns.cu — `.tns` ingestion at scale: the text parse
// of load_tns (sparse_tensor.cpp:136-215) split over host threads, feeding the
// device layout build.
//
// Semantics are the reference's, line for line: '#' comments and blank lines
// skipped; a "dims:" header only as the first content line; the order fixed by
// the override, the header or the first entry line; per line the field-count,
// integer-index, 1-based, 32-bit and finite-value checks in that order; the
// first failing line (in file order) decides the error.  Work split: a short
// sequential scan finds the first content line (order / header); then chunks
// cut at newlines parse independently into per-chunk arrays with per-chunk
// line counts, first errors and observed maxima, merged in chunk order.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "hq_internal.cuh"
#include "hq_plan.cuh"

#include "hq_tns.cuh"

namespace hq {
namespace {

inline bool blank_char(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// tokens of one line (whitespace-separated), at most `cap` recorded, count returned
inline size_t tokens(std::string_view line, std::string_view* out, size_t cap) {
    size_t n = 0, i = 0;
    while (i < line.size()) {
        while (i < line.size() && blank_char(line[i])) ++i;
        const size_t b = i;
        while (i < line.size() && !blank_char(line[i])) ++i;
        if (i > b) {
            if (n < cap) out[n] = line.substr(b, i - b);
            ++n;
        }
    }
    return n;
}

inline bool skippable(std::string_view line) {
    if (line.empty() || line[0] == '#') return true;
    for (char c : line)
        if (!blank_char(c)) return false;
    return true;
}

struct ParseFail {
    int code = 0;  // 0 none, else hq_status
    uint64_t line = 0;
    std::string msg;
};

inline bool parse_index(std::string_view t, uint64_t& v) {
    auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    return r.ec == std::errc{} && r.ptr == t.data() + t.size();
}

struct Chunk {
    const char* b;
    const char* e;
    uint64_t lines = 0;
    std::vector<uint32_t> coords;
    std::vector<double> values;
    std::vector<uint64_t> maxi;
    ParseFail fail;
};

// entry lines of [c.b, c.e); failures record chunk-local line numbers, rebased after the merge
void parse_chunk(Chunk& c, int order, const char* skip_line_start) {
    c.maxi.assign(order, 0);
    std::vector<std::string_view> tok(order + 2);
    const char* p = c.b;
    while (p < c.e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', c.e - p));
        const char* le = nl ? nl : c.e;
        std::string_view line(p, le - p);
        ++c.lines;
        const char* start = p;
        p = nl ? nl + 1 : c.e;
        if (start == skip_line_start || skippable(line)) continue;  // the header line / comments / blanks
        const size_t nt = tokens(line, tok.data(), tok.size());
        auto fail = [&](int code, std::string msg) {
            c.fail = {code, c.lines, std::move(msg)};
        };
        if (nt != (size_t)order + 1) {
            fail(HQ_ERR_PARSE, "expected " + std::to_string(order + 1) + " fields, got " + std::to_string(nt));
            return;
        }
        for (int m = 0; m < order; ++m) {
            uint64_t idx = 0;
            if (!parse_index(tok[m], idx)) {
                fail(HQ_ERR_PARSE, "expected an integer index, got '" + std::string(tok[m]) + "'");
                return;
            }
            if (idx < 1) {
                fail(HQ_ERR_RANGE, ": indices are 1-based, got " + std::to_string(idx));
                return;
            }
            if (idx - 1 > 0xFFFFFFFFull) {
                fail(HQ_ERR_RANGE, ": index " + std::to_string(idx) + " too large");
                return;
            }
            c.coords.push_back(static_cast<uint32_t>(idx - 1));
            c.maxi[m] = std::max(c.maxi[m], idx);
        }
        double v = 0.0;
        const std::string_view vt = tok[order];
        auto r = std::from_chars(vt.data(), vt.data() + vt.size(), v);
        if (r.ec != std::errc{} || r.ptr != vt.data() + vt.size()) {
            fail(HQ_ERR_PARSE, "expected a real value, got '" + std::string(vt) + "'");
            return;
        }
        if (!std::isfinite(v)) {
            fail(HQ_ERR_VALUE, ": non-finite value");
            return;
        }
        c.values.push_back(v);
    }
}

}  // namespace

void tns_parse(const char* text, uint64_t len, int ovr_order, const uint64_t* ovr_dims, hq_tns& out) {
    // 1. first content line: header or the line that fixes the order (sequential, short)
    int order = ovr_order;
    std::vector<uint64_t> header;
    const char* header_line = nullptr;
    uint64_t line_no = 0;
    const char* p = text;
    const char* end = text + len;
    while (p < end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        const char* le = nl ? nl : end;
        std::string_view line(p, le - p);
        ++line_no;
        if (!skippable(line)) {
            if (line.substr(0, 5) == "dims:") {
                std::vector<std::string_view> tk(64);
                size_t nt = tokens(line.substr(5), tk.data(), tk.size());
                if (nt > tk.size()) {
                    tk.resize(nt);
                    nt = tokens(line.substr(5), tk.data(), tk.size());
                }
                if (nt == 0) fail(HQ_ERR_PARSE, "empty dims header", line_no);
                for (size_t i = 0; i < nt; ++i) {
                    uint64_t d = 0;
                    if (!parse_index(tk[i], d))
                        fail(HQ_ERR_PARSE, "expected an integer index, got '" + std::string(tk[i]) + "'", line_no);
                    if (d == 0) fail(HQ_ERR_RANGE, "line " + std::to_string(line_no) + ": extent must be at least 1");
                    header.push_back(d);
                }
                if (order && header.size() != (size_t)order)
                    fail(HQ_ERR_PARSE, "dims header order does not match override", line_no);
                if (!order) order = (int)header.size();
                header_line = p;
            } else if (!order) {
                std::string_view tk[2];
                const size_t nt = tokens(line, tk, 2);
                if (nt < 2)
                    fail(HQ_ERR_PARSE, "entry line needs at least one index and a value", line_no);
                order = (int)nt - 1;
            }
            break;
        }
        p = nl ? nl + 1 : end;
    }
    if (order > kMaxOrder) fail(HQ_ERR_CAPACITY, "tensor order above the engine limit");
    // 2. chunks cut at newlines, parsed in parallel
    std::vector<Chunk> chunks;
    if (order > 0) {
        const unsigned nt = len < (1u << 20) ? 1u : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        const char* b = text;
        for (unsigned t = 0; t < nt && b < end; ++t) {
            const char* e = (t + 1 == nt) ? end : text + len * (t + 1) / nt;
            if (e < b) e = b;
            if (e < end) {
                const char* nl = static_cast<const char*>(std::memchr(e, '\n', end - e));
                e = nl ? nl + 1 : end;
            }
            chunks.push_back(Chunk{b, e});
            b = e;
        }
        std::vector<std::thread> th;
        for (size_t i = 1; i < chunks.size(); ++i) th.emplace_back(parse_chunk, std::ref(chunks[i]), order, header_line);
        if (!chunks.empty()) parse_chunk(chunks[0], order, header_line);
        for (auto& t : th) t.join();
    }
    // 3. merge in file order: the first failing line wins (the reference stops there)
    uint64_t base = 0, nnz = 0;
    std::vector<uint64_t> observed(order > 0 ? order : 0, 0);
    for (const Chunk& c : chunks) {
        if (c.fail.code) {
            const uint64_t ln = base + c.fail.line;
            if (c.fail.code == HQ_ERR_PARSE) fail(HQ_ERR_PARSE, c.fail.msg, (int64_t)ln);
            fail(c.fail.code, "line " + std::to_string(ln) + c.fail.msg);
        }
        base += c.lines;
        nnz += c.values.size();
        for (int m = 0; m < order; ++m) observed[m] = std::max(observed[m], c.maxi[m]);
    }
    out.order = order;
    out.coords.resize(nnz * (size_t)order);
    out.values.resize(nnz);
    size_t at = 0;
    for (const Chunk& c : chunks) {
        std::copy(c.coords.begin(), c.coords.end(), out.coords.begin() + at * order);
        std::copy(c.values.begin(), c.values.end(), out.values.begin() + at);
        at += c.values.size();
    }
    // dims: override, else header, else observed maxima (sparse_tensor.cpp:199-211)
    if (ovr_order > 0)
        out.dims.assign(ovr_dims, ovr_dims + ovr_order);
    else if (!header.empty())
        out.dims = header;
    else if (order > 0 && nnz > 0)
        out.dims = observed;
    else
        fail(HQ_ERR_PARSE, "no entries and no dims header; cannot infer tensor order");
    for (auto& d : out.dims)
        if (d == 0) d = 1;
}

}  // namespace hq
