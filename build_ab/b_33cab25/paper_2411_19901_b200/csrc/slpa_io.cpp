// slpa_io.cpp -- graph files: parallel host parsers and writers
// (the C++ side of sketchlpa/graph.py:165-375).
//
// The parsers feed the device assembly (slpa_build_graph, graph.py:107-139
// rules), so a multi-GB edge list goes file -> parallel parse -> device sort
// / merge without any Python per-line work.  Semantics follow the
// reference's Python parsers line for line:
//
//  * lines split on \n, \r\n and \r (text-mode universal newlines); line
//    numbers count every line (blank and comment lines included);
//  * str.strip() / str.split() whitespace: space, \t, \n, \v, \f, \r and
//    \x1c-\x1f;
//  * int(): [+-]digits (leading zeros allowed); float(): the decimal / inf /
//    infinity / nan grammar of Python's float(), correctly rounded
//    (std::from_chars);
//  * the first failing line (in file order) decides the error, with the
//    reference's per-line check order (graph.py:170-195, :256-284).
//
// Inputs the byte-level grammar does not cover exactly -- non-ASCII bytes
// (Python decodes and may accept Unicode digits / whitespace), digit
// underscores ("1_000"), ids with more than 18 digits (Python ints are
// unbounded) -- return SLPA_IO_EXOTIC and the Python layer parses that file
// with its own restatement of the reference parser (graph_io.py).  That is a
// parsing path, not a compute path: assembly and everything after it run on
// the device either way.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <string>
#include <sys/mman.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <unordered_map>
#include <vector>

#include "../../include/slpa.h"

namespace {

inline bool py_space(unsigned char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

struct Tok {
    const char *p;
    int len;
};

enum IntRes { INT_OK = 0, INT_BAD = 1, INT_EXOTIC = 2 };

// Python int(token) for an ASCII token.  Values beyond 18 significant
// digits (Python ints are unbounded) and digit underscores go the Python way.
IntRes parse_int(const Tok &t, int64_t &out) {
    const char *p = t.p, *e = t.p + t.len;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p == e) return INT_BAD;
    for (const char *q = p; q < e; ++q) {
        if (*q == '_') return INT_EXOTIC;
        if (!is_digit((unsigned char)*q)) return INT_BAD;
    }
    while (p < e - 1 && *p == '0') ++p;
    if (e - p > 18) return INT_EXOTIC;
    int64_t v = 0;
    for (; p < e; ++p) v = v * 10 + (*p - '0');
    out = neg ? -v : v;
    return INT_OK;
}

enum FloatRes { FL_OK = 0, FL_BAD = 1, FL_EXOTIC = 2 };

inline bool ieq(const char *p, int len, const char *word) {
    const int wl = (int)strlen(word);
    if (len != wl) return false;
    for (int i = 0; i < len; ++i) {
        char c = p[i];
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
        if (c != word[i]) return false;
    }
    return true;
}

// Python float(token) for an ASCII token.
FloatRes parse_float(const Tok &t, double &out) {
    const char *p = t.p, *e = t.p + t.len;
    for (const char *q = p; q < e; ++q)
        if (*q == '_') return FL_EXOTIC;
    bool neg = false;
    const char *s = p;
    if (s < e && (*s == '+' || *s == '-')) {
        neg = *s == '-';
        ++s;
    }
    const int rl = (int)(e - s);
    if (ieq(s, rl, "inf") || ieq(s, rl, "infinity")) {
        out = neg ? -INFINITY : INFINITY;
        return FL_OK;
    }
    if (ieq(s, rl, "nan")) {
        out = NAN;
        return FL_OK;
    }
    // decimal: (D+ ('.' D*)? | '.' D+) ([eE] [+-]? D+)?
    const char *q = s;
    int nint = 0, nfrac = 0;
    while (q < e && is_digit((unsigned char)*q)) ++q, ++nint;
    if (q < e && *q == '.') {
        ++q;
        while (q < e && is_digit((unsigned char)*q)) ++q, ++nfrac;
    }
    if (nint + nfrac == 0) return FL_BAD;
    if (q < e && (*q == 'e' || *q == 'E')) {
        ++q;
        if (q < e && (*q == '+' || *q == '-')) ++q;
        int nexp = 0;
        while (q < e && is_digit((unsigned char)*q)) ++q, ++nexp;
        if (nexp == 0) return FL_BAD;
    }
    if (q != e) return FL_BAD;
    double v = 0.0;
    auto r = std::from_chars(s, e, v, std::chars_format::general);
    if (r.ec == std::errc::result_out_of_range) {
        // overflow / underflow (possibly to a subnormal): glibc strtod is
        // correctly rounded and returns inf, 0 or the subnormal like Python
        std::string z(s, e);
        v = strtod(z.c_str(), nullptr);
    } else if (r.ec != std::errc() || r.ptr != e) {
        return FL_BAD;
    }
    out = neg ? -v : v;
    return FL_OK;
}

// Tokenise one stripped line into at most `cap` tokens; returns the count.
inline int split(const char *p, const char *e, Tok *tok, int cap) {
    int n = 0;
    while (p < e) {
        while (p < e && py_space((unsigned char)*p)) ++p;
        if (p >= e) break;
        const char *s = p;
        while (p < e && !py_space((unsigned char)*p)) ++p;
        if (n < cap) tok[n] = Tok{s, (int)(p - s)};
        ++n;
    }
    return n;
}

// Next line of [p, end): sets [ls, le) (terminator excluded), returns the
// start of the following line.
inline const char *next_line(const char *p, const char *end, const char *&ls, const char *&le) {
    ls = p;
    const char *t = p;
    while (t < end && *t != '\n' && *t != '\r') ++t;
    le = t;
    if (t >= end) return end;
    if (*t == '\r' && t + 1 < end && t[1] == '\n') return t + 2;
    return t + 1;
}

inline bool has_high(const char *p, const char *e) {
    for (; p < e; ++p)
        if ((unsigned char)*p >= 0x80) return true;
    return false;
}

// A line starts at q iff q == begin, or q-1 is '\n', or q-1 is '\r' not followed by '\n' at q.
const char *align_line(const char *q, const char *begin, const char *end) {
    while (q < end) {
        if (q == begin) return q;
        const char c = q[-1];
        if (c == '\n') return q;
        if (c == '\r' && *q != '\n') return q;
        ++q;
    }
    return end;
}

struct Chunk {
    const char *b = nullptr, *e = nullptr;
    std::vector<int64_t> src, dst;
    std::vector<double> w;
    int64_t lines = 0;      // lines fully inside the chunk (parsed up to the error)
    int32_t err = 0;        // first error in the chunk
    int64_t err_line = 0;   // chunk-local 0-based line index
    int64_t err_aux = 0;
    bool exotic = false;
};

enum {
    MODE_EL = 0,
    MODE_MM_PATTERN = 1,
    MODE_MM_REAL = 2,
};

// Parse the entry lines of one chunk (edge-list lines or MatrixMarket entries).
void parse_chunk(Chunk &c, int mode, int64_t rows) {
    const char *p = c.b;
    const int64_t reserve = (c.e - c.b) / 12 + 16;
    c.src.reserve(reserve);
    c.dst.reserve(reserve);
    c.w.reserve(reserve);
    Tok tok[4];
    int64_t li = 0;
    for (; p < c.e; ++li) {
        const char *ls, *le;
        p = next_line(p, c.e, ls, le);
        if (has_high(ls, le)) { c.exotic = true; c.lines = li; return; }
        while (ls < le && py_space((unsigned char)*ls)) ++ls;
        while (le > ls && py_space((unsigned char)le[-1])) --le;
        if (ls == le) continue;
        if (mode == MODE_EL) {
            if (*ls == '#' || *ls == '%') continue;
        } else if (*ls == '%') {
            continue;
        }
        const int nt = split(ls, le, tok, 4);
        auto fail = [&](int code, int64_t aux) {
            c.err = code;
            c.err_line = li;
            c.err_aux = aux;
            c.lines = li;
        };
        if (mode == MODE_EL) {
            if (nt != 2 && nt != 3) return fail(SLPA_IO_EL_FIELDS, nt);
        } else {
            const int want = mode == MODE_MM_REAL ? 3 : 2;
            if (nt != want) return fail(SLPA_IO_MM_ENTRY_FIELDS, want);
        }
        int64_t i = 0, j = 0;
        const IntRes r0 = parse_int(tok[0], i);
        const IntRes r1 = r0 == INT_OK ? parse_int(tok[1], j) : INT_OK;
        if (r0 == INT_EXOTIC || r1 == INT_EXOTIC) { c.exotic = true; c.lines = li; return; }
        if (r0 != INT_OK || r1 != INT_OK) return fail(mode == MODE_EL ? SLPA_IO_EL_NONINT : SLPA_IO_MM_NONINT, 0);
        double wt = 1.0;
        if (mode == MODE_EL) {
            if (i < 0 || j < 0) return fail(SLPA_IO_EL_NEGATIVE, 0);
            if (nt == 3) {
                const FloatRes fr = parse_float(tok[2], wt);
                if (fr == FL_EXOTIC) { c.exotic = true; c.lines = li; return; }
                if (fr != FL_OK) return fail(SLPA_IO_EL_BADWEIGHT, 0);
                if (!(wt > 0 && std::isfinite(wt))) return fail(SLPA_IO_EL_WEIGHT, 0);
            }
        } else {
            if (!(1 <= i && i <= rows && 1 <= j && j <= rows)) return fail(SLPA_IO_MM_RANGE, 0);
            if (mode == MODE_MM_REAL) {
                const FloatRes fr = parse_float(tok[2], wt);
                if (fr == FL_EXOTIC) { c.exotic = true; c.lines = li; return; }
                if (fr != FL_OK) return fail(SLPA_IO_MM_BADVALUE, 0);
                if (!(wt > 0 && std::isfinite(wt))) return fail(SLPA_IO_MM_VALUE, 0);
            }
            --i;
            --j;
        }
        c.src.push_back(i);
        c.dst.push_back(j);
        c.w.push_back(wt);
    }
    c.lines = li;
}

int hw_threads(int want) {
    if (want > 0) return want;
    unsigned h = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(h, 64u));
}

}  // namespace

struct slpa_edges {
    std::vector<int64_t> src, dst;
    std::vector<double> w;
    std::vector<int64_t> raw_ids;  // dense id -> raw id (edge lists only)
    int64_t n = 0;
    int32_t remapped = 0;
    int32_t err = 0;
    int64_t err_line = 0, err_aux = 0, err_aux2 = 0;
    std::string header_tok[3];  // MatrixMarket layout / field / symmetry (for messages)
};

namespace {

struct Mapped {
    const char *p = nullptr;
    size_t len = 0;
    int fd = -1;
    std::vector<char> heap;
    ~Mapped() {
        if (p && fd >= 0 && len) munmap((void *)p, len);
        if (fd >= 0) close(fd);
    }
};

int map_file(const char *path, Mapped &m) {
    m.fd = open(path, O_RDONLY);
    if (m.fd < 0) return SLPA_IO_OSERROR;
    struct stat st;
    if (fstat(m.fd, &st) != 0) return SLPA_IO_OSERROR;
    m.len = (size_t)st.st_size;
    if (m.len == 0) {
        m.p = "";
        return 0;
    }
    void *a = mmap(nullptr, m.len, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (a == MAP_FAILED) {  // e.g. a pipe: read it
        m.heap.resize(m.len);
        size_t got = 0;
        while (got < m.len) {
            ssize_t r = read(m.fd, m.heap.data() + got, m.len - got);
            if (r <= 0) return SLPA_IO_OSERROR;
            got += (size_t)r;
        }
        m.p = m.heap.data();
        m.fd = -1;
        return 0;
    }
    madvise(a, m.len, MADV_SEQUENTIAL);
    m.p = (const char *)a;
    return 0;
}

// Parse [b, e) in parallel; entries appended to `out` in file order.  Returns
// SLPA_IO_OK, an error code (out->err_line = global 1-based line number given
// `line0` lines before b), or SLPA_IO_EXOTIC.
int parse_region(const char *b, const char *e, int mode, int64_t rows, int64_t line0, int threads, slpa_edges *out) {
    const size_t bytes = (size_t)(e - b);
    int T = hw_threads(threads);
    if (bytes < ((size_t)1 << 20)) T = 1;
    std::vector<Chunk> ch(T);
    const char *cur = b;
    for (int t = 0; t < T; ++t) {
        ch[t].b = cur;
        const char *nx = t + 1 == T ? e : align_line(b + bytes * (t + 1) / T, b, e);
        if (nx < cur) nx = cur;
        ch[t].e = nx;
        cur = nx;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back([&, t] { parse_chunk(ch[t], mode, rows); });
    parse_chunk(ch[0], mode, rows);
    for (auto &x : th) x.join();
    // first error / exotic line in file order
    int64_t before = line0;
    size_t total = 0;
    for (int t = 0; t < T; ++t) {
        Chunk &c = ch[t];
        if (c.exotic) return SLPA_IO_EXOTIC;
        if (c.err) {
            out->err = c.err;
            out->err_line = before + c.err_line + 1;
            out->err_aux = c.err_aux;
            return c.err;
        }
        // a chunk's line count excludes a final unterminated line only if
        // the chunk is not the last one, which align_line prevents
        before += c.lines;
        total += c.src.size();
    }
    out->src.resize(total);
    out->dst.resize(total);
    out->w.resize(total);
    std::vector<size_t> at(T + 1, 0);
    for (int t = 0; t < T; ++t) at[t + 1] = at[t] + ch[t].src.size();
    std::vector<std::thread> cp;
    for (int t = 0; t < T; ++t)
        cp.emplace_back([&, t] {
            std::copy(ch[t].src.begin(), ch[t].src.end(), out->src.begin() + at[t]);
            std::copy(ch[t].dst.begin(), ch[t].dst.end(), out->dst.begin() + at[t]);
            std::copy(ch[t].w.begin(), ch[t].w.end(), out->w.begin() + at[t]);
            std::vector<int64_t>().swap(ch[t].src);
            std::vector<int64_t>().swap(ch[t].dst);
            std::vector<double>().swap(ch[t].w);
        });
    for (auto &x : cp) x.join();
    out->err_aux2 = before - line0;  // entry-region line count (diagnostics)
    return SLPA_IO_OK;
}

// _remap_ids (graph.py:200-218): dense ids kept verbatim, else first-seen
// order over the interleaved (src, dst) sequence.
void remap_ids(slpa_edges *E, int threads) {
    const size_t cnt = E->src.size();
    int64_t mx = 0;
    for (size_t k = 0; k < cnt; ++k) {
        mx = std::max(mx, E->src[k]);
        mx = std::max(mx, E->dst[k]);
    }
    const uint64_t span = (uint64_t)mx + 1;
    if (span <= 4 * (uint64_t)cnt + 1024) {
        std::vector<uint8_t> seen(span, 0);
        for (size_t k = 0; k < cnt; ++k) {
            seen[E->src[k]] = 1;
            seen[E->dst[k]] = 1;
        }
        int64_t distinct = 0;
        for (uint64_t v = 0; v < span; ++v) distinct += seen[v];
        if ((uint64_t)distinct == span) {
            E->n = (int64_t)span;
            E->remapped = 0;
            return;
        }
        std::vector<int64_t> id(span, -1);
        int64_t next = 0;
        E->raw_ids.clear();
        for (size_t k = 0; k < cnt; ++k) {
            int64_t &a = id[E->src[k]];
            if (a < 0) { a = next++; E->raw_ids.push_back(E->src[k]); }
            E->src[k] = a;
            int64_t &b = id[E->dst[k]];
            if (b < 0) { b = next++; E->raw_ids.push_back(E->dst[k]); }
            E->dst[k] = b;
        }
        E->n = next;
        E->remapped = 1;
        return;
    }
    std::unordered_map<int64_t, int64_t> id;
    id.reserve(cnt * 2);
    E->raw_ids.clear();
    for (size_t k = 0; k < cnt; ++k) {
        auto a = id.emplace(E->src[k], (int64_t)id.size());
        if (a.second) E->raw_ids.push_back(E->src[k]);
        E->src[k] = a.first->second;
        auto b = id.emplace(E->dst[k], (int64_t)id.size());
        if (b.second) E->raw_ids.push_back(E->dst[k]);
        E->dst[k] = b.first->second;
    }
    E->n = (int64_t)id.size();
    E->remapped = 1;
    (void)threads;
}

std::string lower_ascii(std::string s) {
    for (auto &c : s)
        if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
    return s;
}

int parse_mm(const Mapped &m, int threads, slpa_edges *E) {
    const char *p = m.p, *end = m.p + m.len;
    // header = f.readline(): tokens of header.lower().split()
    const char *ls, *le;
    const char *q = p < end ? next_line(p, end, ls, le) : end;
    if (p >= end) { ls = le = p; }
    if (has_high(ls, le)) return SLPA_IO_EXOTIC;  // Python decodes and lower()s the header
    Tok tok[8];
    const int nt = split(ls, le, tok, 8);
    auto tstr = [&](int i) { return lower_ascii(std::string(tok[i].p, tok[i].len)); };
    if (nt != 5 || tstr(0) != "%%matrixmarket" || tstr(1) != "matrix") return E->err = SLPA_IO_MM_HEADER;
    const std::string layout = tstr(2), field = tstr(3), sym = tstr(4);
    E->header_tok[0] = layout;
    E->header_tok[1] = field;
    E->header_tok[2] = sym;
    if (layout != "coordinate") return E->err = SLPA_IO_MM_LAYOUT;
    if (field != "pattern" && field != "real") return E->err = SLPA_IO_MM_FIELD;
    if (sym != "general" && sym != "symmetric") return E->err = SLPA_IO_MM_SYMMETRY;
    int64_t lineno = 1;
    const char *size_s = nullptr, *size_e = nullptr;
    while (q < end) {
        q = next_line(q, end, ls, le);
        ++lineno;
        if (has_high(ls, le)) return SLPA_IO_EXOTIC;
        while (ls < le && py_space((unsigned char)*ls)) ++ls;
        while (le > ls && py_space((unsigned char)le[-1])) --le;
        if (ls == le || *ls == '%') continue;
        size_s = ls;
        size_e = le;
        break;
    }
    if (!size_s) return E->err = SLPA_IO_MM_NOSIZE;
    const int ns = split(size_s, size_e, tok, 8);
    E->err_line = lineno;
    if (ns != 3) return E->err = SLPA_IO_MM_SIZE_FIELDS;
    int64_t dims[3];
    for (int i = 0; i < 3; ++i) {
        const IntRes r = parse_int(tok[i], dims[i]);
        if (r == INT_EXOTIC) return SLPA_IO_EXOTIC;
        if (r != INT_OK) return E->err = SLPA_IO_MM_SIZE_NONINT;
    }
    E->err_line = 0;
    if (dims[0] != dims[1]) {
        E->err_aux = dims[0];
        E->err_aux2 = dims[1];
        return E->err = SLPA_IO_MM_NOT_SQUARE;
    }
    if (dims[0] < 1) return E->err = SLPA_IO_MM_EMPTY;
    const int rc = parse_region(q, end, field == "real" ? MODE_MM_REAL : MODE_MM_PATTERN, dims[0], lineno, threads, E);
    if (rc != SLPA_IO_OK) return rc;
    if ((int64_t)E->src.size() != dims[2]) {
        E->err_line = 0;
        E->err_aux = dims[2];
        E->err_aux2 = (int64_t)E->src.size();
        return E->err = SLPA_IO_MM_COUNT;
    }
    if (E->src.empty()) return E->err = SLPA_IO_NO_EDGES;
    E->n = dims[0];
    return SLPA_IO_OK;
}

}  // namespace

extern "C" {

int32_t slpa_edges_parse(const char *path, int32_t format, int32_t threads, slpa_edges **out) {
    if (!path || !out) return SLPA_IO_OSERROR;
    *out = nullptr;
    Mapped m;
    if (map_file(path, m) != 0) return SLPA_IO_OSERROR;
    slpa_edges *E = new slpa_edges();
    *out = E;
    try {
        if (format == SLPA_FORMAT_EDGE_LIST) {
            const int rc = parse_region(m.p, m.p + m.len, MODE_EL, 0, 0, threads, E);
            if (rc != SLPA_IO_OK) return rc;
            if (E->src.empty()) return E->err = SLPA_IO_NO_EDGES;
            remap_ids(E, threads);
            return SLPA_IO_OK;
        }
        if (format == SLPA_FORMAT_MATRIX_MARKET) return parse_mm(m, threads, E);
        return E->err = SLPA_IO_OSERROR;
    } catch (const std::bad_alloc &) {
        return E->err = SLPA_IO_NOMEM;
    }
}

int32_t slpa_edges_info(const slpa_edges *E, int64_t *count, int64_t *n, int32_t *remapped, int32_t *err,
                        int64_t *err_line, int64_t *err_aux, int64_t *err_aux2) {
    if (!E) return SLPA_EINVAL;
    if (count) *count = (int64_t)E->src.size();
    if (n) *n = E->n;
    if (remapped) *remapped = E->remapped;
    if (err) *err = E->err;
    if (err_line) *err_line = E->err_line;
    if (err_aux) *err_aux = E->err_aux;
    if (err_aux2) *err_aux2 = E->err_aux2;
    return SLPA_OK;
}

int32_t slpa_edges_copy(const slpa_edges *E, int64_t *src, int64_t *dst, double *w, int64_t *raw_ids) {
    if (!E) return SLPA_EINVAL;
    const size_t c = E->src.size();
    if (src) std::memcpy(src, E->src.data(), c * sizeof(int64_t));
    if (dst) std::memcpy(dst, E->dst.data(), c * sizeof(int64_t));
    if (w) std::memcpy(w, E->w.data(), c * sizeof(double));
    if (raw_ids && E->remapped) std::memcpy(raw_ids, E->raw_ids.data(), E->raw_ids.size() * sizeof(int64_t));
    return SLPA_OK;
}

void slpa_edges_free(slpa_edges *E) { delete E; }

// ----------------------------------------------------------------- writers
// write_edgelist (graph.py:352-361): "i j w" for arcs with i <= j;
// write_matrix_market (graph.py:364-375): "i+1 j+1 w" for arcs with i >= j.
// Weights as Python's f"{w:.6g}" of the stored value (float32 widened to
// double, as numpy's __format__ does) -- C's %.6g prints the same digits.
int64_t slpa_format_count(int64_t n, const int64_t *off, const int32_t *tgt, int32_t lower) {
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = off[i]; t < off[i + 1]; ++t) c += lower ? (tgt[t] <= i) : (tgt[t] >= i);
    return c;
}

int32_t slpa_format_rows(int64_t row_begin, int64_t row_end, const int64_t *off, const int32_t *tgt,
                         const void *w, int32_t w_f64, int32_t lower, int32_t threads, char **buf, int64_t *len) {
    *buf = nullptr;
    *len = 0;
    if (row_end <= row_begin) return SLPA_OK;
    int T = hw_threads(threads);
    const int64_t arcs = off[row_end] - off[row_begin];
    if (arcs < (1 << 16)) T = 1;
    std::vector<int64_t> rb(T + 1);
    rb[0] = row_begin;
    rb[T] = row_end;
    for (int t = 1; t < T; ++t) {  // balance by arcs
        const int64_t target = off[row_begin] + arcs * t / T;
        rb[t] = std::max<int64_t>(rb[t - 1], std::upper_bound(off + row_begin, off + row_end, target) - off - 1);
    }
    std::vector<std::string> parts(T);
    auto work = [&](int t) {
        std::string &s = parts[t];
        s.reserve((size_t)(off[rb[t + 1]] - off[rb[t]]) * 12);
        char line[96];
        for (int64_t i = rb[t]; i < rb[t + 1]; ++i) {
            for (int64_t a = off[i]; a < off[i + 1]; ++a) {
                const int64_t j = tgt[a];
                if (lower ? !(i >= j) : !(i <= j)) continue;
                const double wv = w_f64 ? ((const double *)w)[a] : (double)((const float *)w)[a];
                int k;
                if (lower)
                    k = snprintf(line, sizeof line, "%lld %lld %.6g\n", (long long)(i + 1), (long long)(j + 1), wv);
                else
                    k = snprintf(line, sizeof line, "%lld %lld %.6g\n", (long long)i, (long long)j, wv);
                s.append(line, (size_t)k);
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    size_t total = 0;
    for (auto &s : parts) total += s.size();
    char *out = (char *)malloc(total + 1);
    if (!out) return SLPA_EINVAL;
    size_t at = 0;
    for (auto &s : parts) {
        std::memcpy(out + at, s.data(), s.size());
        at += s.size();
    }
    out[total] = 0;
    *buf = out;
    *len = (int64_t)total;
    return SLPA_OK;
}

void slpa_free_buffer(char *buf) { free(buf); }

}  // extern "C"
