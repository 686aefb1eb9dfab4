// io.cpp -- native text edge-list parser (reference load_edge_list,
// graph.py:273-330).
//
// Same result as the reference's Python loop, byte for byte of the CSR it
// feeds: "#"-comment and blank lines skipped; 2 or 3 whitespace-separated
// fields (u, v, optional weight, default 1.0); self-loops dropped before
// their ids are registered; vertex ids compacted 0..n-1 in order of first
// appearance; duplicate undirected edges collapse to the first occurrence
// (its weight wins).  Python's lexical rules are followed for the fields
// (int(): optional sign, digits, single underscores between digits; float():
// the same plus '.', exponent, inf/infinity/nan, no hex), as are its line
// splitting (\n, \r\n, lone \r) and ASCII whitespace set (incl. \x1c-\x1f).
// Errors report the reference's kind and line number; the Python layer
// formats the reference's message text.
#include <cerrno>
#include <climits>
#include <strings.h>
#include <algorithm>
#include <charconv>
#include <system_error>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/infuser_b200.h"

namespace {

inline bool is_ws(unsigned char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

// Python int(): [+-]digits with single underscores between digits.
// 0 ok, 1 not a number, 2 out of int64 range
int parse_int(const char *s, size_t n, int64_t *out) {
    size_t i = 0;
    bool neg = false;
    if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
    if (i >= n || !is_digit(s[i])) return 1;
    unsigned long long v = 0;
    bool over = false;
    for (; i < n; ++i) {
        const char c = s[i];
        if (c == '_') {
            if (i + 1 >= n || !is_digit(s[i + 1]) || !is_digit(s[i - 1])) return 1;
            continue;
        }
        if (!is_digit(c)) return 1;
        const unsigned d = (unsigned)(c - '0');
        if (v > (ULLONG_MAX - d) / 10) over = true;
        else v = v * 10 + d;
    }
    const unsigned long long lim = neg ? (1ull << 63) : (1ull << 63) - 1;
    if (over || v > lim) return 2;
    *out = neg ? (int64_t)(0 - v) : (int64_t)v;
    return 0;
}

// Python float(): decimal / exponent / inf / infinity / nan with an optional
// sign, underscores only between digits, no hex.  0 ok, 1 not a number.
int parse_float_slow(const char *s, size_t n, double *out);

int parse_float(const char *s, size_t n, double *out) {
    // fast path (no underscores): std::from_chars is correctly rounded like
    // strtod / Python; it takes no leading '+', and Python takes no "+-"
    if (!memchr(s, '_', n)) {
        if (memchr(s, '(', n) || memchr(s, 'x', n) || memchr(s, 'X', n)) return 1;
        const char *b = s, *e = s + n;
        if (b < e && *b == '+') {
            ++b;
            if (b < e && (*b == '-' || *b == '+')) return 1;
        }
        if (b == e) return 1;
        double v;
        const auto r = std::from_chars(b, e, v, std::chars_format::general);
        if (r.ec == std::errc::result_out_of_range) return parse_float_slow(s, n, out);   // +-inf / 0 like Python
        if (r.ec != std::errc() || r.ptr != e) return 1;
        *out = v;
        return 0;
    }
    return parse_float_slow(s, n, out);
}

int parse_float_slow(const char *s, size_t n, double *out) {
    std::string t;
    t.reserve(n);
    for (size_t i = 0; i < n; ++i) {
        const char c = s[i];
        if (c == '_') {
            if (i == 0 || i + 1 >= n || !is_digit(s[i - 1]) || !is_digit(s[i + 1])) return 1;
            continue;
        }
        if (c == 'x' || c == 'X' || c == '(' || c == ')' || c == 'p' || c == 'P') return 1;
        t.push_back(c);
    }
    if (t.empty()) return 1;
    // strtod also accepts forms Python rejects: "infin", "nanxyz" are caught by
    // the full-consumption test; a bare sign / "." / "e5" by the digit check
    {
        size_t j = (t[0] == '+' || t[0] == '-') ? 1 : 0;
        const char *w = t.c_str() + j;
        const bool word = !strcasecmp(w, "inf") || !strcasecmp(w, "infinity") || !strcasecmp(w, "nan");
        if (!word) {
            bool digit = false;
            for (size_t k = j; k < t.size() && t[k] != 'e' && t[k] != 'E'; ++k) digit |= is_digit(t[k]);
            if (!digit) return 1;
        }
    }
    errno = 0;
    char *end = nullptr;
    const double v = strtod(t.c_str(), &end);
    if (end != t.c_str() + t.size()) return 1;
    *out = v;       // overflow gives +-inf like Python's float("1e999")
    return 0;
}

// open-addressing int64 -> int32 map (first-appearance ids); one slot =
// key + value + used flag in 16 bytes, so a probe is one cache line
struct IdMap {
    struct Slot {
        int64_t key;
        int32_t val;
        int32_t used;
    };
    std::vector<Slot> slots;
    size_t count = 0, mask = 0;
    IdMap() { rehash(1 << 16); }
    static uint64_t mix(uint64_t x) {
        x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
        return x;
    }
    void rehash(size_t cap) {
        std::vector<Slot> old;
        old.swap(slots);
        slots.assign(cap, Slot{0, 0, 0});
        mask = cap - 1;
        for (const Slot &o : old)
            if (o.used) {
                size_t h = mix((uint64_t)o.key) & mask;
                while (slots[h].used) h = (h + 1) & mask;
                slots[h] = o;
            }
    }
    int32_t get_or_add(int64_t k, std::vector<int64_t> &orig) {
        size_t h = mix((uint64_t)k) & mask;
        while (slots[h].used) {
            if (slots[h].key == k) return slots[h].val;
            h = (h + 1) & mask;
        }
        const int32_t v = (int32_t)orig.size();
        slots[h] = Slot{k, v, 1};
        orig.push_back(k);
        if (++count * 2 > mask + 1) rehash((mask + 1) * 2);
        return v;
    }
};

// open-addressing set of undirected pair keys
struct PairSet {
    std::vector<uint64_t> keys;   // 0 = empty; stored as key + 1
    size_t count = 0, mask = 0;
    PairSet() { keys.assign(1 << 16, 0); mask = keys.size() - 1; }
    bool insert(uint64_t k) {     // true if new
        const uint64_t kk = k + 1;
        size_t h = IdMap::mix(k) & mask;
        while (keys[h]) {
            if (keys[h] == kk) return false;
            h = (h + 1) & mask;
        }
        keys[h] = kk;
        if (++count * 2 > mask + 1) grow();
        return true;
    }
    void grow() {
        std::vector<uint64_t> old;
        old.swap(keys);
        keys.assign(old.size() * 2, 0);
        mask = keys.size() - 1;
        for (uint64_t kk : old)
            if (kk) {
                size_t h = IdMap::mix(kk - 1) & mask;
                while (keys[h]) h = (h + 1) & mask;
                keys[h] = kk;
            }
    }
};

}  // namespace

struct imx_edge_list {
    std::vector<int64_t> orig;     // compact id -> original id
    std::vector<int64_t> edges;    // 2 per edge, compact ids
    std::vector<double> weights;
};

namespace {

// one parsed line that survives to the compaction pass
struct Rec {
    int64_t u, v;
    double w;
};

// per-chunk result of the parallel pass
struct Chunk {
    const char *begin = nullptr, *end = nullptr;
    std::vector<Rec> recs;
    int64_t lines = 0;
    int err_kind = 0;           // first error of the chunk (0: none)
    int64_t err_line = 0, err_aux = 0;
    const char *err_txt = nullptr;
    size_t err_len = 0;
};

// next line start after position p (\n, \r\n or a lone \r ends a line)
const char *next_line(const char *p, const char *end) {
    while (p < end && *p != '\n' && *p != '\r') ++p;
    if (p < end) {
        if (*p == '\r' && p + 1 < end && p[1] == '\n') p += 2;
        else ++p;
    }
    return p;
}

void parse_chunk(Chunk &c) {
    const char *p = c.begin, *end = c.end;
    c.recs.reserve((size_t)((end - p) / 16));
    while (p < end) {
        const char *ls = p, *le = p;
        while (le < end && *le != '\n' && *le != '\r') ++le;
        p = next_line(le, end);
        ++c.lines;
        const char *a = ls, *b = le;
        while (a < b && is_ws((unsigned char)*a)) ++a;
        while (b > a && is_ws((unsigned char)b[-1])) --b;
        if (a == b || *a == '#') continue;
        const char *fs[4];
        size_t fl[4];
        int nf = 0;
        for (const char *q = a; q < b;) {
            while (q < b && is_ws((unsigned char)*q)) ++q;
            if (q >= b) break;
            const char *st = q;
            while (q < b && !is_ws((unsigned char)*q)) ++q;
            if (nf < 4) { fs[nf] = st; fl[nf] = (size_t)(q - st); }
            ++nf;
        }
        auto err = [&](int kind, int64_t aux, const char *t, size_t n) {
            c.err_kind = kind; c.err_line = c.lines; c.err_aux = aux; c.err_txt = t; c.err_len = n;
        };
        if (nf != 2 && nf != 3) { err(1, nf, a, (size_t)(b - a)); return; }
        int64_t u = 0, v = 0;
        double w = 1.0;
        const int ru = parse_int(fs[0], fl[0], &u), rv = ru ? 0 : parse_int(fs[1], fl[1], &v);
        if (ru == 2 || rv == 2) { err(6, 0, a, (size_t)(b - a)); return; }     // beyond int64 (OverflowError)
        if (ru || rv || (nf == 3 && parse_float(fs[2], fl[2], &w))) { err(2, 0, a, (size_t)(b - a)); return; }
        if (!(w >= 0.0 && w <= 1.0)) { err(3, 0, fs[2], fl[2]); return; }
        if (u == v) continue;                 // self-loops register no ids
        c.recs.push_back(Rec{u, v, w});
    }
}

}  // namespace

// Two passes: the lines are split into chunks at line boundaries and parsed
// (fields, numbers, validation) by host threads; the first-appearance id
// compaction and the first-occurrence dedupe then run in file order.
extern "C" int imx_edge_list_parse(const char *path, imx_edge_list **out, int64_t *err_line, int32_t *err_kind,
                                   int64_t *err_aux, char *err_text, int64_t err_text_cap) {
    if (!path || !out) return IMX_EINVAL;
    *out = nullptr;
    auto fail = [&](int kind, int64_t line, int64_t aux, const char *txt, size_t len) {
        if (err_kind) *err_kind = kind;
        if (err_line) *err_line = line;
        if (err_aux) *err_aux = aux;
        if (err_text && err_text_cap > 0) {
            const size_t m = std::min<size_t>(len, (size_t)err_text_cap - 1);
            if (txt && m) memcpy(err_text, txt, m);
            err_text[m] = 0;
        }
        return IMX_EFORMAT;
    };
    FILE *f = fopen(path, "rb");
    if (!f) return fail(5, 0, errno, nullptr, 0);
    std::vector<char> buf;
    if (fseek(f, 0, SEEK_END) == 0) {
        const long sz = ftell(f);
        if (sz > 0) buf.resize((size_t)sz);
        fseek(f, 0, SEEK_SET);
        if (!buf.empty() && fread(buf.data(), 1, buf.size(), f) != buf.size()) buf.clear();
    }
    if (buf.empty()) {                        // unseekable or short read: stream it
        char tmp[1 << 16];
        size_t r;
        fseek(f, 0, SEEK_SET);
        while ((r = fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + r);
    }
    fclose(f);
    const bool prof = getenv("IMX_PARSE_PROFILE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    const char *base = buf.data(), *end = base + buf.size();
    unsigned hw = std::thread::hardware_concurrency();
    int nt = (int)std::min<size_t>(std::max(1u, std::min(hw, 16u)), std::max<size_t>(1, buf.size() >> 20));
    if (const char *e = getenv("IMX_PARSE_THREADS")) nt = std::max(1, atoi(e));
    std::vector<Chunk> ch(nt);
    const char *cur = base;
    for (int i = 0; i < nt; ++i) {
        const char *stop = i + 1 == nt ? end : base + (buf.size() * (size_t)(i + 1)) / nt;
        if (stop < cur) stop = cur;
        if (stop > base && stop < end && stop[-1] == '\r' && *stop == '\n') ++stop;       // keep \r\n together
        else if (stop > base && stop < end && stop[-1] != '\n' && stop[-1] != '\r') stop = next_line(stop, end);
        ch[i].begin = cur;
        ch[i].end = stop;
        cur = stop;
    }
    {
        std::vector<std::thread> th;
        for (int i = 1; i < nt; ++i) th.emplace_back(parse_chunk, std::ref(ch[i]));
        parse_chunk(ch[0]);
        for (auto &t : th) t.join();
    }
    auto t1 = now();
    int64_t lines_before = 0;
    for (int i = 0; i < nt; ++i) {
        if (ch[i].err_kind)
            return fail(ch[i].err_kind, lines_before + ch[i].err_line, ch[i].err_aux, ch[i].err_txt, ch[i].err_len);
        lines_before += ch[i].lines;
    }
    imx_edge_list *el = new imx_edge_list();
    IdMap ids;
    PairSet seen;
    size_t total = 0;
    for (auto &c : ch) total += c.recs.size();
    el->edges.reserve(2 * total);
    el->weights.reserve(total);
    for (auto &c : ch) {
        for (const Rec &r : c.recs) {
            const int32_t cu = ids.get_or_add(r.u, el->orig);
            const int32_t cv = ids.get_or_add(r.v, el->orig);
            if (el->orig.size() >= ((size_t)1 << 31) - 1) {
                delete el;
                return fail(7, lines_before, 0, nullptr, 0);      // id space exhausted
            }
            const uint32_t lo = (uint32_t)(cu < cv ? cu : cv), hi = (uint32_t)(cu < cv ? cv : cu);
            if (!seen.insert(((uint64_t)lo << 32) | hi)) continue;
            el->edges.push_back(cu);
            el->edges.push_back(cv);
            el->weights.push_back(r.w);
        }
        std::vector<Rec>().swap(c.recs);
    }
    if (prof)
        fprintf(stderr, "[parse] %d threads: fields+numbers %.1f ms, compaction+dedupe %.1f ms\n", nt,
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(now() - t1).count());
    if (el->weights.empty()) {
        delete el;
        return fail(4, lines_before, 0, nullptr, 0);
    }
    *out = el;
    return IMX_OK;
}

extern "C" int imx_edge_list_dims(const imx_edge_list *e, int64_t *n_vertices, int64_t *n_edges) {
    if (!e) return IMX_EINVAL;
    if (n_vertices) *n_vertices = (int64_t)e->orig.size();
    if (n_edges) *n_edges = (int64_t)e->weights.size();
    return IMX_OK;
}

extern "C" int imx_edge_list_copy(const imx_edge_list *e, int64_t *edges, double *weights, int64_t *orig_ids) {
    if (!e) return IMX_EINVAL;
    if (edges) memcpy(edges, e->edges.data(), sizeof(int64_t) * e->edges.size());
    if (weights) memcpy(weights, e->weights.data(), sizeof(double) * e->weights.size());
    if (orig_ids) memcpy(orig_ids, e->orig.data(), sizeof(int64_t) * e->orig.size());
    return IMX_OK;
}

extern "C" void imx_edge_list_free(imx_edge_list *e) { delete e; }
