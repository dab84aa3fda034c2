// mmio.cpp — §8(f) rank 2: the on-disk format either side of the build path.
//
// Host-side (multi-threaded C++) restatement of
//   mcspai::CsrMatrix::from_triplets   src/csr.cpp:17-58
//   mcspai::parse_matrix_market        src/matrix_market.cpp:27-147
//   mcspai::read_matrix_market_file    src/matrix_market.cpp:149-153
//   mcspai::write_matrix_market(_file) src/matrix_market.cpp:155-177
// with the same results byte for byte:
//   * tokens are recognised exactly as libstdc++'s istream extractors do
//     (num_get: sign, digits, one '.', an exponent only after a mantissa
//     digit), values converted by a correctly rounded conversion (strtod's),
//     overflow to +-inf rejected like num_get;
//   * lines are split like std::getline, so error line numbers match;
//   * duplicates are summed in the order the reference's std::sort leaves
//     them.  Pairs commute, so the parallel path (counting sort by row, column
//     sort within rows) is exact unless some coordinate repeats 3+ times; then
//     libstdc++'s introsort is replayed on the index array (restated below);
//   * "%.17g" is produced by std::to_chars(general, 17), the same digits.
// The reference reads line by line through std::istringstream (about 1 us per
// entry) and writes with snprintf; here the text is split into chunks at line
// boundaries and parsed / formatted by one thread per chunk.
#include <algorithm>
#include <array>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "mcmi.h"

// Uninitialised host array (std::vector would zero-fill hundreds of MB first).
template <class T>
struct HostArray {
    std::unique_ptr<T[]> p;
    int64_t size = 0;
    void reset(int64_t n) {
        p.reset(new T[static_cast<size_t>(std::max<int64_t>(n, 1))]);
        size = n;
    }
    T* data() { return p.get(); }
    const T* data() const { return p.get(); }
    T& operator[](int64_t i) { return p[i]; }
    const T& operator[](int64_t i) const { return p[i]; }
};

struct mcmi_host_csr {
    int64_t n = 0;
    HostArray<int64_t> row_ptr, col_idx;
    HostArray<double> values;
};

namespace mcmi {
namespace mmio {
namespace {

struct Error {
    int code;
    std::string msg;
};

int io_threads() {
    static const int t = [] {
        const char* e = std::getenv("MCMI_IO_THREADS");
        int v = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
        return std::max(1, std::min(v, 64));
    }();
    return t;
}

// MCMI_IO_TRACE=1: phase timings on stderr (tuning aid).
struct Trace {
    bool on = std::getenv("MCMI_IO_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mmio] %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

// Runs f(t) for t in [0, T) on T threads (the caller's thread takes t = 0).
template <class F>
void parallel(int T, F&& f) {
    if (T <= 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T - 1);
    for (int t = 1; t < T; ++t) th.emplace_back([&f, t] { f(t); });
    f(0);
    for (auto& x : th) x.join();
}

// ------------------------------------------------ libstdc++ std::sort replay
// The introsort of libstdc++ (bits/stl_algo.h, stl_heap.h), restated: depth
// limit 2*floor(log2 n), median-of-three pivot moved to the front, unguarded
// Hoare partition, heapsort when the depth runs out, insertion sort of runs
// <= 16 at the end.  It decides the order of equal keys, hence the order in
// which from_triplets sums duplicates.
template <class T, class Less>
struct Introsort {
    Less less;
    static constexpr ptrdiff_t kThreshold = 16;

    void push_heap(T* first, ptrdiff_t hole, ptrdiff_t top, T value) {
        ptrdiff_t parent = (hole - 1) / 2;
        while (hole > top && less(first[parent], value)) {
            first[hole] = first[parent];
            hole = parent;
            parent = (hole - 1) / 2;
        }
        first[hole] = value;
    }
    void adjust_heap(T* first, ptrdiff_t hole, ptrdiff_t len, T value) {
        const ptrdiff_t top = hole;
        ptrdiff_t child = hole;
        while (child < (len - 1) / 2) {
            child = 2 * (child + 1);
            if (less(first[child], first[child - 1])) --child;
            first[hole] = first[child];
            hole = child;
        }
        if ((len & 1) == 0 && child == (len - 2) / 2) {
            child = 2 * (child + 1);
            first[hole] = first[child - 1];
            hole = child - 1;
        }
        push_heap(first, hole, top, value);
    }
    void make_heap(T* first, T* last) {
        const ptrdiff_t len = last - first;
        if (len < 2) return;
        for (ptrdiff_t parent = (len - 2) / 2;; --parent) {
            adjust_heap(first, parent, len, first[parent]);
            if (parent == 0) return;
        }
    }
    void pop_heap(T* first, T* last, T* result) {
        const T value = *result;
        *result = *first;
        adjust_heap(first, 0, last - first, value);
    }
    void heap_sort(T* first, T* last) {  // __partial_sort(first, last, last)
        make_heap(first, last);
        while (last - first > 1) {
            --last;
            pop_heap(first, last, last);
        }
    }
    void move_median_to_first(T* result, T* a, T* b, T* c) {
        if (less(*a, *b)) {
            if (less(*b, *c)) std::swap(*result, *b);
            else if (less(*a, *c)) std::swap(*result, *c);
            else std::swap(*result, *a);
        } else if (less(*a, *c)) {
            std::swap(*result, *a);
        } else if (less(*b, *c)) {
            std::swap(*result, *c);
        } else {
            std::swap(*result, *b);
        }
    }
    T* partition(T* first, T* last, T* pivot) {
        for (;;) {
            while (less(*first, *pivot)) ++first;
            --last;
            while (less(*pivot, *last)) --last;
            if (!(first < last)) return first;
            std::swap(*first, *last);
            ++first;
        }
    }
    void loop(T* first, T* last, int depth) {
        while (last - first > kThreshold) {
            if (depth == 0) {
                heap_sort(first, last);
                return;
            }
            --depth;
            T* mid = first + (last - first) / 2;
            move_median_to_first(first, first + 1, mid, last - 1);
            T* cut = partition(first + 1, last, first);
            loop(cut, last, depth);
            last = cut;
        }
    }
    void linear_insert(T* last) {
        const T value = *last;
        T* next = last - 1;
        while (less(value, *next)) {
            *last = *next;
            last = next;
            --next;
        }
        *last = value;
    }
    void insertion_sort(T* first, T* last) {
        if (first == last) return;
        for (T* i = first + 1; i != last; ++i) {
            if (less(*i, *first)) {
                const T value = *i;
                std::move_backward(first, i, i + 1);
                *first = value;
            } else {
                linear_insert(i);
            }
        }
    }
    void sort(T* first, T* last) {
        if (first == last) return;
        const ptrdiff_t n = last - first;
        int lg = 63 - __builtin_clzll(static_cast<unsigned long long>(n));
        loop(first, last, 2 * lg);
        if (n > kThreshold) {
            insertion_sort(first, first + kThreshold);
            for (T* i = first + kThreshold; i != last; ++i) linear_insert(i);
        } else {
            insertion_sort(first, last);
        }
    }
};

// ------------------------------------------------------------ from_triplets
// Triplets may arrive in several segments (one per parse chunk); the logical
// array is their concatenation.
struct Seg {
    const int64_t* r;
    const int64_t* c;
    const double* v;
    int64_t m;
};

// Exact replay: the reference's own algorithm over an index permutation.
void triplets_replay(int64_t n, const int64_t* rows, const int64_t* cols, const double* vals,
                     int64_t m, mcmi_host_csr* out) {
    std::vector<size_t> order(static_cast<size_t>(m));
    for (int64_t k = 0; k < m; ++k) order[k] = static_cast<size_t>(k);
    auto less = [rows, cols](size_t a, size_t b) {
        if (rows[a] != rows[b]) return rows[a] < rows[b];
        return cols[a] < cols[b];
    };
    Introsort<size_t, decltype(less)> s{less};
    s.sort(order.data(), order.data() + m);
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0), ci;
    std::vector<double> va;
    ci.reserve(static_cast<size_t>(m));
    va.reserve(static_cast<size_t>(m));
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        while (k < m && rows[order[k]] == i) {
            const int64_t c = cols[order[k]];
            double v = vals[order[k]];
            ++k;
            while (k < m && rows[order[k]] == i && cols[order[k]] == c) {
                v += vals[order[k]];  // duplicates are summed (csr.cpp:45-48)
                ++k;
            }
            if (v != 0.0) {
                ci.push_back(c);
                va.push_back(v);
            }
        }
        rp[i + 1] = static_cast<int64_t>(ci.size());
    }
    out->n = n;
    out->row_ptr.reset(n + 1);
    out->col_idx.reset(static_cast<int64_t>(ci.size()));
    out->values.reset(static_cast<int64_t>(va.size()));
    std::copy(rp.begin(), rp.end(), out->row_ptr.data());
    std::copy(ci.begin(), ci.end(), out->col_idx.data());
    std::copy(va.begin(), va.end(), out->values.data());
}

struct Ent {
    int64_t c;
    double v;
};

// Work pieces over the segments: (segment, begin, end), about 64k entries each.
std::vector<std::array<int64_t, 3>> pieces_of(const std::vector<Seg>& segs) {
    std::vector<std::array<int64_t, 3>> w;
    for (size_t s = 0; s < segs.size(); ++s)
        for (int64_t a = 0; a < segs[s].m; a += 65536)
            w.push_back({static_cast<int64_t>(s), a, std::min<int64_t>(segs[s].m, a + 65536)});
    return w;
}

template <class F>
void for_pieces(const std::vector<std::array<int64_t, 3>>& w, int T, F&& f) {
    std::atomic<size_t> next{0};
    parallel(T, [&](int) {
        for (size_t i; (i = next.fetch_add(1, std::memory_order_relaxed)) < w.size();) f(w[i]);
    });
}

// Parallel path: range check + counting sort by row, column sort within each
// row.  Exact when no coordinate occurs 3+ times (a + b == b + a).  Returns
// 1 = done, 0 = a coordinate repeats 3+ times (replay needed), -1 = range error.
int triplets_parallel(int64_t n, const std::vector<Seg>& segs, int64_t m, mcmi_host_csr* out) {
    const int T = static_cast<int>(std::min<int64_t>(io_threads(), std::max<int64_t>(1, m / 65536)));
    const auto work = pieces_of(segs);
    std::unique_ptr<std::atomic<int64_t>[]> cnt(new std::atomic<int64_t>[static_cast<size_t>(n) + 1]);
    parallel(T, [&](int t) {
        for (int64_t i = (n + 1) * t / T; i < (n + 1) * (t + 1) / T; ++i) cnt[i].store(0, std::memory_order_relaxed);
    });
    std::atomic<bool> bad{false};
    for_pieces(work, T, [&](const std::array<int64_t, 3>& p) {
        const Seg& g = segs[p[0]];
        for (int64_t k = p[1]; k < p[2]; ++k) {
            const int64_t r = g.r[k], c = g.c[k];
            if (r < 0 || r >= n || c < 0 || c >= n) {  // csr.cpp:23-26
                bad.store(true, std::memory_order_relaxed);
                return;
            }
            cnt[r + 1].fetch_add(1, std::memory_order_relaxed);
        }
    });
    if (bad.load()) return -1;
    HostArray<int64_t> start;
    start.reset(n + 1);
    start[0] = 0;
    for (int64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i + 1].load(std::memory_order_relaxed);
    parallel(T, [&](int t) {
        for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) cnt[i].store(start[i], std::memory_order_relaxed);
    });
    HostArray<Ent> ent;
    ent.reset(m);
    for_pieces(work, T, [&](const std::array<int64_t, 3>& p) {
        const Seg& g = segs[p[0]];
        for (int64_t k = p[1]; k < p[2]; ++k)
            ent[cnt[g.r[k]].fetch_add(1, std::memory_order_relaxed)] = Ent{g.c[k], g.v[k]};
    });
    // per row: sort by column, sum equal columns (at most pairs), prune zeros
    HostArray<int64_t> kept;
    kept.reset(n);
    std::atomic<bool> triple{false};
    parallel(T, [&](int t) {
        for (int64_t i = n * t / T; i < n * (t + 1) / T && !triple.load(std::memory_order_relaxed); ++i) {
            Ent* a = ent.data() + start[i];
            Ent* b = ent.data() + start[i + 1];
            if (b - a > 1) std::sort(a, b, [](const Ent& x, const Ent& y) { return x.c < y.c; });
            int64_t o = 0;
            for (Ent* q = a; q < b;) {
                Ent* nx = q + 1;
                double v = q->v;
                if (nx < b && nx->c == q->c) {
                    if (nx + 1 < b && (nx + 1)->c == q->c) {
                        triple.store(true, std::memory_order_relaxed);
                        break;
                    }
                    v += nx->v;
                    ++nx;
                }
                if (v != 0.0) a[o++] = Ent{q->c, v};
                q = nx;
            }
            kept[i] = o;
        }
    });
    if (triple.load()) return 0;
    out->n = n;
    out->row_ptr.reset(n + 1);
    out->row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) out->row_ptr[i + 1] = out->row_ptr[i] + kept[i];
    const int64_t nnz = out->row_ptr[n];
    out->col_idx.reset(nnz);
    out->values.reset(nnz);
    parallel(T, [&](int t) {
        for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) {
            const Ent* a = ent.data() + start[i];
            int64_t o = out->row_ptr[i];
            for (int64_t k = 0; k < kept[i]; ++k, ++o) {
                out->col_idx[o] = a[k].c;
                out->values[o] = a[k].v;
            }
        }
    });
    return 1;
}

Error from_triplets(int64_t n, const std::vector<Seg>& segs, mcmi_host_csr* out) {
    int64_t m = 0;
    for (const Seg& g : segs) m += g.m;
    // the reference builds an n = -1 matrix with no row_ptr, or throws
    // std::length_error, for a negative n; refuse it outright (after the
    // reference's own range check, which fails first when there are entries)
    if (n < 0) return m > 0 ? Error{MCMI_ERANGE, "triplet index out of range"} : Error{MCMI_EINVAL, "negative dimension"};
    const int st = triplets_parallel(n, segs, m, out);
    if (st < 0) return {MCMI_ERANGE, "triplet index out of range"};
    if (st == 0) {  // flatten and replay the reference's sort
        std::vector<int64_t> r, c;
        std::vector<double> v;
        r.reserve(static_cast<size_t>(m));
        c.reserve(static_cast<size_t>(m));
        v.reserve(static_cast<size_t>(m));
        for (const Seg& g : segs) {
            r.insert(r.end(), g.r, g.r + g.m);
            c.insert(c.end(), g.c, g.c + g.m);
            v.insert(v.end(), g.v, g.v + g.m);
        }
        triplets_replay(n, r.data(), c.data(), v.data(), m, out);
    }
    return {MCMI_OK, {}};
}

// ----------------------------------------------------------- token scanning
// istream >> long long / >> double / >> std::string in the "C" locale, over
// [p, e) of one line (no '\n' inside).

inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

inline const char* skip_ws(const char* p, const char* e) {
    while (p < e && is_space(*p)) ++p;
    return p;
}

// >> std::string: skip whitespace, take the run of non-space characters
const char* scan_word(const char* p, const char* e, std::string& w) {
    p = skip_ws(p, e);
    const char* s = p;
    while (p < e && !is_space(*p)) ++p;
    w.assign(s, p);
    return p;
}

// >> int64: [+-] digits+, base 10; no digit or overflow fails.
bool scan_int(const char*& p, const char* e, int64_t& out) {
    const char* q = skip_ws(p, e);
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) {
        neg = *q == '-';
        ++q;
    }
    const char* d = q;
    unsigned long long v = 0;
    bool over = false;
    const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
    while (q < e && *q >= '0' && *q <= '9') {
        const unsigned dig = static_cast<unsigned>(*q - '0');
        if (v > (lim - dig) / 10) over = true;
        else v = v * 10 + dig;
        ++q;
    }
    if (q == d || over) {
        p = q;
        return false;
    }
    out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
    p = q;
    return true;
}

// >> double: the characters num_get::_M_extract_float accumulates — [+-],
// digits with at most one '.', then 'e'/'E' [+-] digits once a mantissa digit
// was seen — converted with strtod's correct rounding; fails if nothing
// convertible was accumulated or the value overflows to +-inf.
bool scan_double(const char*& p, const char* e, double& out) {
    const char* q = skip_ws(p, e);
    const char* s = q;
    if (q < e && (*q == '+' || *q == '-')) ++q;
    bool mant = false, dot = false, sci = false, expdig = false;
    while (q < e) {
        const char c = *q;
        if (c >= '0' && c <= '9') {
            if (sci) expdig = true;
            else mant = true;
        } else if (c == '.' && !dot && !sci) {
            dot = true;
        } else if ((c == 'e' || c == 'E') && !sci && mant) {
            sci = true;
            if (q + 1 < e && (q[1] == '+' || q[1] == '-')) ++q;
        } else {
            break;
        }
        ++q;
    }
    p = q;
    if (!mant || (sci && !expdig)) return false;
    const char* a = (*s == '+') ? s + 1 : s;
    double v = 0.0;
    auto r = std::from_chars(a, q, v, std::chars_format::general);
    if (r.ec != std::errc() || r.ptr != q) {  // underflow / rare forms: strtod decides
        std::string tmp(a, q);
        char* endp = nullptr;
        v = std::strtod(tmp.c_str(), &endp);
        if (endp != tmp.c_str() + tmp.size()) return false;
    }
    if (std::isinf(v)) return false;
    out = v;
    return true;
}

// --------------------------------------------------------------- line cursor
// std::getline semantics: a line ends at '\n'; a final unterminated segment is
// a line iff it is non-empty.
struct Lines {
    const char* p;
    const char* e;
    bool next(const char*& ls, const char*& le) {
        if (p >= e) return false;
        ls = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
        if (nl) {
            le = nl;
            p = nl + 1;
        } else {
            le = e;
            p = e;
        }
        return true;
    }
};

std::string lower(std::string s) {
    for (auto& c : s)
        if (c >= 'A' && c <= 'Z') c = static_cast<char>(c - 'A' + 'a');
    return s;
}

Error parse_error(int64_t line_no, const std::string& what) {
    return {MCMI_EPARSE, "matrix market: line " + std::to_string(line_no) + ": " + what};
}

struct Chunk {  // one thread's share of the coordinate entry lines
    const char* p;
    const char* e;
    int64_t lines = 0;  // lines scanned before stopping
    std::vector<int64_t> r, c;
    std::vector<double> v;
    int64_t entries = 0;     // entry lines parsed successfully (before err)
    int64_t err_line = -1;   // local line index (0-based) of the first bad entry line
    std::string err_what;
};

void parse_chunk(Chunk& ch, int64_t n, bool sym, bool skew, int64_t budget) {
    const size_t guess = static_cast<size_t>((ch.e - ch.p) / 12 + 16) * ((sym || skew) ? 2 : 1);
    ch.r.reserve(guess);
    ch.c.reserve(guess);
    ch.v.reserve(guess);
    Lines L{ch.p, ch.e};
    const char *ls, *le;
    while (ch.entries < budget && L.next(ls, le)) {
        ++ch.lines;
        if (ls == le || *ls == '%') continue;
        const char* q = ls;
        int64_t i = 0, j = 0;
        double v = 0.0;
        if (!scan_int(q, le, i) || !scan_int(q, le, j) || !scan_double(q, le, v)) {
            ch.err_line = ch.lines - 1;
            ch.err_what = "malformed entry";
            return;
        }
        if (i < 1 || i > n || j < 1 || j > n) {
            ch.err_line = ch.lines - 1;
            ch.err_what = "index out of range";
            return;
        }
        ch.r.push_back(i - 1);
        ch.c.push_back(j - 1);
        ch.v.push_back(v);
        if ((sym || skew) && i != j) {
            ch.r.push_back(j - 1);
            ch.c.push_back(i - 1);
            ch.v.push_back(skew ? -v : v);
        }
        ++ch.entries;
    }
}

Error parse(const char* text, size_t len, mcmi_host_csr* out) {
    Lines L{text, text + len};
    const char *ls, *le;
    int64_t line_no = 1;
    if (!L.next(ls, le)) return parse_error(line_no, "empty input");
    std::string banner, object, format, field, symmetry;
    {
        const char* q = ls;
        q = scan_word(q, le, banner);
        q = scan_word(q, le, object);
        q = scan_word(q, le, format);
        q = scan_word(q, le, field);
        scan_word(q, le, symmetry);
    }
    if (banner != "%%MatrixMarket") return parse_error(line_no, "missing %%MatrixMarket banner");
    object = lower(object);
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (object != "matrix") return parse_error(line_no, "object must be 'matrix'");
    if (format != "coordinate" && format != "array")
        return parse_error(line_no, "format must be 'coordinate' or 'array'");
    if (field == "complex") return parse_error(line_no, "complex field is not supported");
    if (field != "real" && field != "integer" && field != "double" && field != "pattern")
        return parse_error(line_no, "unsupported field '" + field + "'");
    if (field == "pattern") return parse_error(line_no, "pattern field is not supported");
    const bool sym = symmetry == "symmetric";
    const bool skew = symmetry == "skew-symmetric";
    if (!sym && !skew && symmetry != "general")
        return parse_error(line_no, "unsupported symmetry '" + symmetry + "'");

    // comments (and empty lines) up to the size line
    bool have = false;
    while (L.next(ls, le)) {
        ++line_no;
        if (ls != le && *ls != '%') {
            have = true;
            break;
        }
    }
    if (!have) return parse_error(line_no, "missing size line");
    const char* q = ls;
    int64_t n_rows = 0, n_cols = 0;
    if (!scan_int(q, le, n_rows) || !scan_int(q, le, n_cols)) return parse_error(line_no, "malformed size line");
    if (n_rows != n_cols)
        return parse_error(line_no, "matrix is not square (" + std::to_string(n_rows) + "x" +
                                        std::to_string(n_cols) + ")");
    const int64_t n = n_rows;
    std::vector<int64_t> rows, cols;
    std::vector<double> vals;

    if (format == "coordinate") {
        int64_t declared = 0;
        if (!scan_int(q, le, declared)) return parse_error(line_no, "missing nnz count");
        if (declared < 0) return {MCMI_EINVAL, "vector::reserve"};  // rows.reserve(declared) throws
        // split the rest at line boundaries, one chunk per thread
        const char* body = L.p;
        const char* end = text + len;
        const int64_t bytes = end - body;
        const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(io_threads(), bytes / (1 << 20))));
        std::vector<Chunk> ch(T);
        const char* cur = body;
        for (int t = 0; t < T; ++t) {
            const char* stop = t + 1 == T ? end : body + bytes * (t + 1) / T;
            if (stop < cur) stop = cur;
            if (t + 1 < T && stop < end) {
                const char* nl = static_cast<const char*>(std::memchr(stop, '\n', static_cast<size_t>(end - stop)));
                stop = nl ? nl + 1 : end;
            }
            ch[t].p = cur;
            ch[t].e = stop;
            cur = stop;
        }
        Trace tr;
        parallel(T, [&](int t) { parse_chunk(ch[t], n, sym, skew, declared); });
        tr.mark("parse chunks");
        // merge in file order: the first `declared` entry lines count
        int64_t seen = 0, lines = line_no;
        std::vector<Seg> segs;
        for (int t = 0; t < T && seen < declared; ++t) {
            const Chunk& c = ch[t];
            if (c.err_line >= 0 && seen + c.entries < declared)
                return parse_error(lines + c.err_line + 1, c.err_what);
            const int64_t take = std::min<int64_t>(c.entries, declared - seen);
            // entries map to 1 or 2 triplets; keep those of the first `take` entries
            int64_t trip = 0;
            if (take == c.entries) {
                trip = static_cast<int64_t>(c.r.size());
            } else {
                for (int64_t k = 0, e = 0; e < take; ++e) {
                    const bool two = (sym || skew) && c.r[k] != c.c[k];
                    k += two ? 2 : 1;
                    trip = k;
                }
            }
            segs.push_back(Seg{c.r.data(), c.c.data(), c.v.data(), trip});
            seen += take;
            lines += c.lines;
        }
        if (seen < declared) return parse_error(lines + 1, "unexpected end of file");
        Error e = from_triplets(n, segs, out);
        tr.mark("from_triplets");
        return e;
    } else {  // array: column-major dense listing (matrix_market.cpp:101-143)
        const int64_t total = (sym || skew) ? n * (n + 1) / 2 : n * n;
        int64_t seen = 0, col = 0, row_in_col = 0;
        while (seen < total) {
            if (!L.next(ls, le)) return parse_error(line_no + 1, "unexpected end of file");
            ++line_no;
            if (ls == le || *ls == '%') continue;
            const char* p = ls;
            double v;
            while (scan_double(p, le, v)) {
                int64_t i, j;
                if (sym || skew) {
                    j = col;
                    i = col + row_in_col;
                } else {
                    j = col;
                    i = row_in_col;
                }
                if (v != 0.0) {
                    rows.push_back(i);
                    cols.push_back(j);
                    vals.push_back(v);
                    if ((sym || skew) && i != j) {
                        rows.push_back(j);
                        cols.push_back(i);
                        vals.push_back(skew ? -v : v);
                    }
                }
                ++seen;
                ++row_in_col;
                const int64_t col_len = (sym || skew) ? n - col : n;
                if (row_in_col == col_len) {
                    row_in_col = 0;
                    ++col;
                }
                if (seen == total) break;
            }
        }
    }
    return from_triplets(n, {Seg{rows.data(), cols.data(), vals.data(), static_cast<int64_t>(rows.size())}}, out);
}

// --------------------------------------------------------------- formatting
inline char* put_i64(char* p, long long v) {
    return std::to_chars(p, p + 24, v).ptr;
}

inline char* put_line(char* p, int64_t i, int64_t c, double v) {  // "%lld %lld %.17g\n"
    p = put_i64(p, static_cast<long long>(i + 1));
    *p++ = ' ';
    p = put_i64(p, static_cast<long long>(c + 1));
    *p++ = ' ';
    p = std::to_chars(p, p + 32, v, std::chars_format::general, 17).ptr;
    *p++ = '\n';
    return p;
}

constexpr size_t kMaxLine = 24 + 1 + 24 + 1 + 32 + 1;

std::string header(const mcmi_csr_view& m) {
    const int64_t nnz = m.n > 0 ? m.row_ptr[m.n] : 0;
    return "%%MatrixMarket matrix coordinate real general\n" + std::to_string(m.n) + " " +
           std::to_string(m.n) + " " + std::to_string(nnz) + "\n";
}

Error check_view(const mcmi_csr_view* m) {
    if (!m || m->n < 0) return {MCMI_EINVAL, "invalid CSR view"};
    if (m->n == 0) return {MCMI_OK, {}};
    if (!m->row_ptr) return {MCMI_EINVAL, "invalid CSR view"};
    if (m->row_ptr[0] != 0) return {MCMI_EINVAL, "row_ptr[0] must be 0"};
    for (int64_t i = 0; i < m->n; ++i)
        if (m->row_ptr[i + 1] < m->row_ptr[i]) return {MCMI_EINVAL, "row_ptr is not non-decreasing"};
    if (m->row_ptr[m->n] > 0 && (!m->col_idx || !m->values)) return {MCMI_EINVAL, "invalid CSR view"};
    return {MCMI_OK, {}};
}

// Formats rows in T slices balanced by entries; slice t's text goes to parts[t].
void format_rows(const mcmi_csr_view& m, std::vector<std::string>& parts) {
    parts.clear();
    if (m.n <= 0) return;
    const int64_t nnz = m.row_ptr[m.n];
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(io_threads(), nnz / 65536)));
    parts.assign(T, std::string());
    auto first_row = [&](int t) -> int64_t {  // first row whose entries start at or after slice t's share
        if (t == 0) return 0;
        if (t == T) return m.n;
        const int64_t k = nnz * t / T;
        return std::min<int64_t>(m.n, std::lower_bound(m.row_ptr, m.row_ptr + m.n + 1, k) - m.row_ptr);
    };
    parallel(T, [&](int t) {
        const int64_t r0 = first_row(t), r1 = std::max(r0, first_row(t + 1));
        if (r1 <= r0) return;
        std::string& s = parts[t];
        s.reserve(static_cast<size_t>(m.row_ptr[r1] - m.row_ptr[r0]) * 40);
        char stage[1 << 16];
        char* p = stage;
        for (int64_t i = r0; i < r1; ++i)
            for (int64_t k = m.row_ptr[i]; k < m.row_ptr[i + 1]; ++k) {
                if (p + kMaxLine > stage + sizeof stage) {
                    s.append(stage, static_cast<size_t>(p - stage));
                    p = stage;
                }
                p = put_line(p, i, m.col_idx[k], m.values[k]);
            }
        s.append(stage, static_cast<size_t>(p - stage));
    });
}

int report(const Error& e, char* err, size_t errlen) {
    if (e.code != MCMI_OK && err && errlen) {
        std::strncpy(err, e.msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return e.code;
}

template <class F>
int guarded(F&& f, char* err, size_t errlen) {
    try {
        return report(f(), err, errlen);
    } catch (const std::bad_alloc&) {
        return report({MCMI_ENOMEM, "out of host memory"}, err, errlen);
    } catch (const std::exception& ex) {
        return report({MCMI_EINVAL, ex.what()}, err, errlen);
    }
}

}  // namespace
}  // namespace mmio
}  // namespace mcmi

using namespace mcmi::mmio;

extern "C" {

int mcmi_from_triplets(int64_t n, const int64_t* rows, const int64_t* cols, const double* vals, int64_t count,
                       mcmi_host_csr** out, char* err, size_t errlen) {
    if (!out || count < 0 || (count > 0 && (!rows || !cols || !vals)))
        return report({MCMI_EINVAL, "null argument"}, err, errlen);
    *out = nullptr;
    return guarded(
        [&]() -> Error {
            auto* m = new mcmi_host_csr();
            Error e = from_triplets(n, {Seg{rows, cols, vals, count}}, m);
            if (e.code) delete m;
            else *out = m;
            return e;
        },
        err, errlen);
}

int mcmi_mm_parse(const char* text, size_t len, mcmi_host_csr** out, char* err, size_t errlen) {
    if (!out || (len > 0 && !text)) return report({MCMI_EINVAL, "null argument"}, err, errlen);
    *out = nullptr;
    return guarded(
        [&]() -> Error {
            auto* m = new mcmi_host_csr();
            Error e = parse(text, len, m);
            if (e.code) delete m;
            else *out = m;
            return e;
        },
        err, errlen);
}

int mcmi_mm_read_file(const char* path, mcmi_host_csr** out, char* err, size_t errlen) {
    if (!out || !path) return report({MCMI_EINVAL, "null argument"}, err, errlen);
    *out = nullptr;
    return guarded(
        [&]() -> Error {
            FILE* f = std::fopen(path, "rb");
            if (!f) return {MCMI_EPARSE, std::string("cannot open '") + path + "'"};  // ParseError (:151)
            Trace tr;
            std::unique_ptr<char[]> whole;  // uninitialised: the file fills it
            size_t size = 0;
            std::string rest;
            if (std::fseek(f, 0, SEEK_END) == 0) {
                const long sz = std::ftell(f);
                std::rewind(f);
                if (sz > 0) {
                    whole.reset(new char[static_cast<size_t>(sz)]);
                    size = std::fread(whole.get(), 1, static_cast<size_t>(sz), f);
                }
            }
            char tmp[1 << 16];  // non-seekable input (pipes) or a file that grew: read to the end
            for (size_t got; (got = std::fread(tmp, 1, sizeof tmp, f)) > 0;) rest.append(tmp, got);
            std::fclose(f);
            if (!rest.empty()) {
                rest.insert(0, whole.get(), size);
                whole.reset();
                size = 0;
            }
            const char* text = rest.empty() ? whole.get() : rest.data();
            const size_t len = rest.empty() ? size : rest.size();
            tr.mark("read file");
            auto* m = new mcmi_host_csr();
            Error e = parse(text, len, m);
            if (e.code) delete m;
            else *out = m;
            return e;
        },
        err, errlen);
}

void mcmi_host_csr_get(const mcmi_host_csr* m, mcmi_csr_view* view) {
    view->n = m->n;
    view->row_ptr = const_cast<int64_t*>(m->row_ptr.data());  // n + 1 entries
    view->col_idx = const_cast<int64_t*>(m->col_idx.data());
    view->values = const_cast<double*>(m->values.data());
}

void mcmi_host_csr_free(mcmi_host_csr* m) { delete m; }

int mcmi_mm_format(const mcmi_csr_view* m, char* buf, size_t cap, size_t* len, char* err, size_t errlen) {
    if (!len) return report({MCMI_EINVAL, "null argument"}, err, errlen);
    return guarded(
        [&]() -> Error {
            Error e = check_view(m);
            if (e.code) return e;
            const std::string h = header(*m);
            std::vector<std::string> parts;
            format_rows(*m, parts);
            size_t total = h.size();
            for (const auto& p : parts) total += p.size();
            *len = total;
            if (!buf) return {MCMI_OK, {}};
            if (cap < total) return {MCMI_ENOMEM, "buffer too small"};
            char* p = buf;
            std::memcpy(p, h.data(), h.size());
            p += h.size();
            for (const auto& s : parts) {
                std::memcpy(p, s.data(), s.size());
                p += s.size();
            }
            return {MCMI_OK, {}};
        },
        err, errlen);
}

int mcmi_mm_write_file(const mcmi_csr_view* m, const char* path, char* err, size_t errlen) {
    if (!path) return report({MCMI_EINVAL, "null argument"}, err, errlen);
    return guarded(
        [&]() -> Error {
            Error e = check_view(m);
            if (e.code) return e;
            FILE* f = std::fopen(path, "wb");
            if (!f) return {MCMI_EIO, std::string("cannot open '") + path + "' for writing"};  // :173
            const std::string h = header(*m);
            std::vector<std::string> parts;
            format_rows(*m, parts);
            bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size();
            for (const auto& s : parts) ok = ok && std::fwrite(s.data(), 1, s.size(), f) == s.size();
            ok = (std::fclose(f) == 0) && ok;
            if (!ok) return {MCMI_EIO, std::string("write failure on '") + path + "'"};  // :176
            return {MCMI_OK, {}};
        },
        err, errlen);
}

}  // extern "C"
