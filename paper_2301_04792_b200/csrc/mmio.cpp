// mmio.cpp — host-native ingestion: Matrix Market coordinate text -> COO, and
// COO -> CSR (sort by (row, col), duplicates summed in input order).
//
// Replaces the reference's line-by-line Python reader (mmio.py:24-107) and the
// numpy lexsort/bincount packing (sparse.py:130-150) with multi-threaded C++
// over the raw bytes. Accepted inputs, the order in which errors are detected
// and the error texts follow mmio.py exactly: the first offending line in file
// order wins, entries beyond the declared count are reported before their
// content is looked at, and symmetric files append the mirrored off-diagonal
// entries after all stored entries, in file order (mmio.py:99-104).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "lw_b200.h"

namespace {

bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

struct Span {
    const char* p;
    size_t n;
};

Span strip(const char* b, const char* e) {
    while (b < e && is_ws(*b)) ++b;
    while (e > b && is_ws(e[-1])) --e;
    return Span{b, (size_t)(e - b)};
}

int split(Span s, Span* out, int max_out) {
    int k = 0;
    const char* p = s.p;
    const char* e = s.p + s.n;
    while (p < e) {
        while (p < e && is_ws(*p)) ++p;
        if (p >= e) break;
        const char* q = p;
        while (q < e && !is_ws(*q)) ++q;
        if (k < max_out) out[k] = Span{p, (size_t)(q - p)};
        ++k;
        p = q;
    }
    return k;
}

// Python repr() of a str (single quotes unless the text holds ' and no ").
std::string py_repr(Span s) {
    const bool has_sq = memchr(s.p, '\'', s.n) != nullptr, has_dq = memchr(s.p, '"', s.n) != nullptr;
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string r(1, q);
    for (size_t i = 0; i < s.n; ++i) {
        const unsigned char c = (unsigned char)s.p[i];
        if (c == '\\') r += "\\\\";
        else if (c == (unsigned char)q) { r += '\\'; r += (char)c; }
        else if (c == '\n') r += "\\n";
        else if (c == '\r') r += "\\r";
        else if (c == '\t') r += "\\t";
        else if (c < 0x20 || c == 0x7f) {
            char buf[8];
            snprintf(buf, sizeof buf, "\\x%02x", c);
            r += buf;
        } else r += (char)c;
    }
    r += q;
    return r;
}

// Python int(): optional sign, decimal digits with single underscores between them.
bool parse_int(Span s, int64_t* out) {
    size_t i = 0;
    bool neg = false;
    if (i < s.n && (s.p[i] == '+' || s.p[i] == '-')) { neg = s.p[i] == '-'; ++i; }
    if (i >= s.n) return false;
    __int128 v = 0;
    bool digit_before = false;
    for (; i < s.n; ++i) {
        const char c = s.p[i];
        if (c >= '0' && c <= '9') {
            v = v * 10 + (c - '0');
            if (v > ((__int128)1 << 100)) v = ((__int128)1 << 100);   // saturate: stays out of bounds
            digit_before = true;
        } else if (c == '_' && digit_before && i + 1 < s.n && s.p[i + 1] >= '0' && s.p[i + 1] <= '9') {
            digit_before = false;
        } else {
            return false;
        }
    }
    if (neg) v = -v;
    const __int128 lim = (__int128)INT64_MAX;
    *out = v > lim ? INT64_MAX : (v < -lim ? -INT64_MAX : (int64_t)v);
    return true;
}

// Python float(): decimal / exponent forms, inf / infinity / nan (any case, signed);
// no hex floats; single underscores between digits.
bool parse_float(Span s, double* out) {
    if (s.n == 0 || s.n > 400) return false;
    char buf[416];
    size_t k = 0;
    for (size_t i = 0; i < s.n; ++i) {
        const char c = s.p[i];
        if (c == '_') {
            const bool ok = i > 0 && i + 1 < s.n && isdigit((unsigned char)s.p[i - 1]) &&
                            isdigit((unsigned char)s.p[i + 1]);
            if (!ok) return false;
            continue;
        }
        if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
        buf[k++] = c;
    }
    buf[k] = 0;
    // strtod also takes "inf"/"nan(...)": accept only Python's spellings
    const char* b = buf + ((buf[0] == '+' || buf[0] == '-') ? 1 : 0);
    if (isalpha((unsigned char)*b)) {
        if (strcasecmp(b, "inf") && strcasecmp(b, "infinity") && strcasecmp(b, "nan")) return false;
    }
    char* end = nullptr;
    errno = 0;
    const double v = strtod(buf, &end);
    if (end != buf + k) return false;
    *out = v;
    return true;
}

void set_err(char* err, size_t errlen, const char* fmt, ...) {
    if (!err || !errlen) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
}

enum Field { F_REAL = 0, F_INTEGER = 1, F_PATTERN = 2 };

struct Line {
    const char* b;
    const char* e;
};

// next line [b, e) starting at p (without the '\n'); returns the start of the following line
const char* next_line(const char* p, const char* end, Line* ln) {
    const char* q = (const char*)memchr(p, '\n', (size_t)(end - p));
    if (!q) q = end;
    ln->b = p;
    ln->e = q;
    return q < end ? q + 1 : end;
}

bool skippable(Span s) { return s.n == 0 || s.p[0] == '%'; }

std::string lower(Span s) {
    std::string r(s.p, s.n);
    for (auto& c : r) c = (char)tolower((unsigned char)c);
    return r;
}

}  // namespace

extern "C" {

int lw_mm_parse_header(const char* buf, size_t len, lw_mm_header_t* h, char* err, size_t errlen) {
    if (!h || (!buf && len)) return LW_E_INVALID_ARG;
    const char* p = buf;
    const char* end = buf + len;
    if (len == 0) {
        set_err(err, errlen, "empty input: missing Matrix Market banner");
        return LW_E_FORMAT;
    }
    Line ln;
    p = next_line(p, end, &ln);
    Span banner = strip(ln.b, ln.e);
    Span tok[6];
    const int nt = split(banner, tok, 6);
    if (nt != 5 || lower(tok[0]) != "%%matrixmarket") {
        set_err(err, errlen, "malformed banner: %s", py_repr(banner).c_str());
        return LW_E_FORMAT;
    }
    const std::string obj = lower(tok[1]), fmt = lower(tok[2]), field = lower(tok[3]),
                      sym = lower(tok[4]);
    if (obj != "matrix") {
        set_err(err, errlen, "unsupported object %s: only 'matrix' is supported",
                py_repr(Span{obj.data(), obj.size()}).c_str());
        return LW_E_FORMAT;
    }
    if (fmt != "coordinate") {
        set_err(err, errlen, "unsupported format %s: only 'coordinate' is supported",
                py_repr(Span{fmt.data(), fmt.size()}).c_str());
        return LW_E_FORMAT;
    }
    int f;
    if (field == "real") f = F_REAL;
    else if (field == "integer") f = F_INTEGER;
    else if (field == "pattern") f = F_PATTERN;
    else {
        set_err(err, errlen, "unsupported field %s: expected one of ('real', 'integer', 'pattern')",
                py_repr(Span{field.data(), field.size()}).c_str());
        return LW_E_FORMAT;
    }
    int symmetric;
    if (sym == "general") symmetric = 0;
    else if (sym == "symmetric") symmetric = 1;
    else {
        set_err(err, errlen, "unsupported symmetry %s: expected one of ('general', 'symmetric')",
                py_repr(Span{sym.data(), sym.size()}).c_str());
        return LW_E_FORMAT;
    }
    Span header{nullptr, 0};
    bool found = false;
    while (p < end) {
        p = next_line(p, end, &ln);
        Span s = strip(ln.b, ln.e);
        if (skippable(s)) continue;
        header = s;
        found = true;
        break;
    }
    if (!found) {
        set_err(err, errlen, "missing size header line");
        return LW_E_FORMAT;
    }
    Span ht[4];
    if (split(header, ht, 4) != 3) {
        set_err(err, errlen, "malformed size header: %s", py_repr(header).c_str());
        return LW_E_FORMAT;
    }
    int64_t v[3];
    for (int i = 0; i < 3; ++i)
        if (!parse_int(ht[i], v + i)) {
            set_err(err, errlen, "malformed size header: %s", py_repr(header).c_str());
            return LW_E_FORMAT;
        }
    if (v[0] < 0 || v[1] < 0 || v[2] < 0) {
        set_err(err, errlen, "negative dimension in size header: %s", py_repr(header).c_str());
        return LW_E_FORMAT;
    }
    h->rows = v[0];
    h->cols = v[1];
    h->entries = v[2];
    h->field = f;
    h->symmetric = symmetric;
    h->data_offset = (int64_t)(p - buf);
    return LW_OK;
}

int lw_mm_parse_entries(const char* buf, size_t len, const lw_mm_header_t* h, int64_t* row,
                        int64_t* col, double* val, int64_t capacity, int64_t* count_out,
                        int32_t threads, char* err, size_t errlen) {
    if (!h || !count_out || h->data_offset < 0 || (size_t)h->data_offset > len) return LW_E_INVALID_ARG;
    const int64_t declared = h->entries;
    const int64_t need = h->symmetric ? 2 * declared : declared;
    if (capacity < need || (need > 0 && (!row || !col || !val))) return LW_E_INVALID_ARG;
    const char* data = buf + h->data_offset;
    const char* end = buf + len;
    const size_t bytes = (size_t)(end - data);
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (T < 1) T = 1;
    if (bytes < ((size_t)1 << 20)) T = 1;
    // chunk boundaries at line starts
    std::vector<const char*> cut(T + 1);
    cut[0] = data;
    cut[T] = end;
    for (int t = 1; t < T; ++t) {
        const char* q = data + bytes * (size_t)t / (size_t)T;
        if (q < cut[t - 1]) q = cut[t - 1];
        const char* nl = (const char*)memchr(q, '\n', (size_t)(end - q));
        cut[t] = nl ? nl + 1 : end;
    }
    // pass 1: entry lines per chunk
    std::vector<int64_t> lines(T + 1, 0);
    auto count_chunk = [&](int t) {
        int64_t c = 0;
        Line ln;
        for (const char* p = cut[t]; p < cut[t + 1];) {
            p = next_line(p, cut[t + 1], &ln);
            if (!skippable(strip(ln.b, ln.e))) ++c;
        }
        lines[t + 1] = c;
    };
    {
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(count_chunk, t);
        count_chunk(0);
        for (auto& th : pool) th.join();
    }
    for (int t = 0; t < T; ++t) lines[t + 1] += lines[t];
    const int64_t found = lines[T];
    // pass 2: parse; each chunk records its first error (entry index, message)
    const int tpe = h->field == F_PATTERN ? 2 : 3;
    std::vector<int64_t> err_at(T, INT64_MAX);
    std::vector<std::string> err_msg(T);
    auto parse_chunk = [&](int t) {
        int64_t k = lines[t];
        Line ln;
        for (const char* p = cut[t]; p < cut[t + 1];) {
            p = next_line(p, cut[t + 1], &ln);
            Span s = strip(ln.b, ln.e);
            if (skippable(s)) continue;
            if (k >= declared) {
                char m[160];
                snprintf(m, sizeof m,
                         "entry count mismatch: header declares %lld entries but more follow",
                         (long long)declared);
                err_at[t] = k;
                err_msg[t] = m;
                return;
            }
            Span f[4];
            const int nf = split(s, f, 4);
            int64_t i = 0, j = 0;
            double v = 1.0;
            bool ok = nf == tpe && parse_int(f[0], &i) && parse_int(f[1], &j);
            if (ok && tpe == 3) ok = parse_float(f[2], &v);
            if (!ok) {
                err_at[t] = k;
                err_msg[t] = "malformed entry line: " + py_repr(s);
                return;
            }
            if (!(1 <= i && i <= h->rows && 1 <= j && j <= h->cols)) {
                char m[200];
                snprintf(m, sizeof m, "entry (%lld, %lld) out of declared bounds %lld x %lld",
                         (long long)i, (long long)j, (long long)h->rows, (long long)h->cols);
                err_at[t] = k;
                err_msg[t] = m;
                return;
            }
            row[k] = i - 1;
            col[k] = j - 1;
            val[k] = v;
            ++k;
        }
    };
    {
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(parse_chunk, t);
        parse_chunk(0);
        for (auto& th : pool) th.join();
    }
    for (int t = 0; t < T; ++t)
        if (err_at[t] != INT64_MAX) {
            set_err(err, errlen, "%s", err_msg[t].c_str());
            return LW_E_FORMAT;
        }
    if (found != declared) {
        set_err(err, errlen, "entry count mismatch: header declares %lld entries, found %lld",
                (long long)declared, (long long)found);
        return LW_E_FORMAT;
    }
    int64_t n = declared;
    if (h->symmetric) {
        for (int64_t k = 0; k < declared; ++k)
            if (row[k] != col[k]) {
                row[n] = col[k];
                col[n] = row[k];
                val[n] = val[k];
                ++n;
            }
    }
    *count_out = n;
    return LW_OK;
}

int lw_coo_to_csr_host(int64_t rows, int64_t cols, int64_t n, const int64_t* row,
                       const int64_t* col, const double* val, int64_t* row_offsets,
                       int64_t* col_out, double* val_out, int64_t* nnz_out, int32_t threads) {
    if (rows < 0 || cols < 0 || n < 0 || !row_offsets || !nnz_out) return LW_E_INVALID_ARG;
    if (n > 0 && (!row || !col || !val || !col_out || !val_out)) return LW_E_INVALID_ARG;
    for (int64_t k = 0; k < n; ++k)
        if (row[k] < 0 || row[k] >= rows || col[k] < 0 || col[k] >= cols) return LW_E_INVALID_ARG;
    struct E {
        int64_t r, c, i;
    };
    std::vector<E> e((size_t)n);
    for (int64_t k = 0; k < n; ++k) e[k] = E{row[k], col[k], k};
    auto less = [](const E& a, const E& b) {
        return a.r != b.r ? a.r < b.r : (a.c != b.c ? a.c < b.c : a.i < b.i);
    };
    // parallel sort: sorted runs per thread, then pairwise merges (keys are unique
    // thanks to the input index, so the order is the stable (row, col) order)
    int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (T < 1) T = 1;
    if (n < (1 << 16)) T = 1;
    std::vector<int64_t> b(T + 1);
    for (int t = 0; t <= T; ++t) b[t] = n * t / T;
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] { std::sort(e.begin() + b[t], e.begin() + b[t + 1], less); });
        for (auto& th : pool) th.join();
    }
    for (int w = 1; w < T; w *= 2) {
        std::vector<std::thread> pool;
        for (int t = 0; t + w < T; t += 2 * w) {
            const int64_t lo = b[t], mid = b[t + w], hi = b[std::min(T, t + 2 * w)];
            pool.emplace_back([&, lo, mid, hi] {
                std::inplace_merge(e.begin() + lo, e.begin() + mid, e.begin() + hi, less);
            });
        }
        for (auto& th : pool) th.join();
    }
    // runs of equal (row, col) summed in input order, starting from 0.0 like np.bincount
    for (int64_t r = 0; r <= rows; ++r) row_offsets[r] = 0;
    int64_t m = 0;
    for (int64_t k = 0; k < n;) {
        int64_t q = k;
        double s = 0.0;
        while (q < n && e[q].r == e[k].r && e[q].c == e[k].c) s += val[e[q++].i];
        col_out[m] = e[k].c;
        val_out[m] = s;
        row_offsets[e[k].r + 1] += 1;
        ++m;
        k = q;
    }
    for (int64_t r = 0; r < rows; ++r) row_offsets[r + 1] += row_offsets[r];
    *nnz_out = m;
    return LW_OK;
}

}  // extern "C"
