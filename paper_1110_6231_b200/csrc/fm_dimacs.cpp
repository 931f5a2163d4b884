// fm_dimacs.cpp -- DIMACS max-flow / assignment ingest.
//
// Parses the same formats as the reference's parse_dimacs_max / parse_dimacs_asn
// (dimacs.py:123-248) with the same validation and the same line-numbered error
// messages, in one pass over the bytes.  Two-call protocol: call with null arrays to
// learn the counts, then with arrays of at least that size.
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "flowmatch_b200.h"

void fm_set_error(const char *fmt, ...);

namespace {

struct Tok {
    const char *p;
    int n;
    std::string str() const { return std::string(p, (size_t)n); }
};

// split one line into whitespace tokens (at most `cap`)
int split(const char *b, const char *e, Tok *out, int cap) {
    int k = 0;
    while (b < e) {
        while (b < e && (*b == ' ' || *b == '\t' || *b == '\r' || *b == '\f' || *b == '\v')) b++;
        if (b >= e) break;
        const char *s = b;
        while (b < e && !(*b == ' ' || *b == '\t' || *b == '\r' || *b == '\f' || *b == '\v')) b++;
        if (k < cap) out[k] = Tok{s, (int)(b - s)};
        k++;
    }
    return k;
}

bool to_int(const Tok &t, long long *v) {
    if (t.n == 0 || t.n > 19) return false;
    int i = 0;
    bool neg = false;
    if (t.p[0] == '+' || t.p[0] == '-') { neg = t.p[0] == '-'; i = 1; if (t.n == 1) return false; }
    long long x = 0;
    for (; i < t.n; i++) {
        if (t.p[i] < '0' || t.p[i] > '9') return false;
        const int d = t.p[i] - '0';
        if (x > (INT64_MAX - d) / 10) return false;   // does not fit in int64
        x = x * 10 + d;
    }
    *v = neg ? -x : x;
    return true;
}

#define PERR(...) do { fm_set_error(__VA_ARGS__); return FM_INVALID_ARG; } while (0)

int int_tok(const Tok &t, long long lineno, long long *v) {
    if (!to_int(t, v)) {
        fm_set_error("line %lld: expected integer, got '%s'", lineno, t.str().c_str());
        return FM_INVALID_ARG;
    }
    return FM_OK;
}

int node_tok(const Tok &t, long long lineno, long long n, long long *v) {
    if (int_tok(t, lineno, v)) return FM_INVALID_ARG;
    if (*v < 1 || *v > n) {
        fm_set_error("line %lld: node id %lld out of range 1..%lld", lineno, *v, n);
        return FM_INVALID_ARG;
    }
    *v -= 1;
    return FM_OK;
}

int problem_line(Tok *t, int k, long long lineno, const char *expected, bool seen,
                 long long *count, long long *declared) {
    if (seen) PERR("line %lld: duplicate problem line", lineno);
    if (k != 4) PERR("line %lld: malformed problem line", lineno);
    if (t[1].str() != expected)
        PERR("line %lld: expected problem type '%s', got '%s'", lineno, expected, t[1].str().c_str());
    if (int_tok(t[2], lineno, count) || int_tok(t[3], lineno, declared)) return FM_INVALID_ARG;
    if (*count < 0 || *declared < 0) PERR("line %lld: negative count on problem line", lineno);
    return FM_OK;
}

}  // namespace

// out_nst = {node_count, source, sink}; *out_m = arcs.  tails/heads/caps may be null
// (count only) or hold at least *out_m (from a previous call) entries.
namespace {
int parse_max(const char *text, int64_t len, int32_t *out_nst, int64_t *out_m,
              int32_t *tails, int32_t *heads, int64_t *caps, int64_t cap_arcs) {
    if (!text || len < 0 || !out_nst || !out_m) PERR("fm_dimacs_parse_max: invalid argument");
    long long n = -1, declared = 0, source = -1, sink = -1, m = 0;
    const char *p = text, *end = text + len;
    long long lineno = 0;
    Tok t[8];
    while (p < end) {
        const char *eol = (const char *)memchr(p, '\n', (size_t)(end - p));
        if (!eol) eol = end;
        lineno++;
        const int k = split(p, eol, t, 8);
        p = eol + 1;
        if (k == 0 || t[0].str() == "c") continue;
        const std::string tag = t[0].str();
        if (tag == "p") {
            if (problem_line(t, k, lineno, "max", n >= 0, &n, &declared)) return FM_INVALID_ARG;
            continue;
        }
        if (n < 0) PERR("line %lld: '%s' line before problem line", lineno, tag.c_str());
        if (tag == "n") {
            if (k != 3) PERR("line %lld: malformed node designator", lineno);
            long long node;
            if (node_tok(t[1], lineno, n, &node)) return FM_INVALID_ARG;
            const std::string which = t[2].str();
            if (which == "s") {
                if (source >= 0) PERR("line %lld: duplicate source designator", lineno);
                source = node;
            } else if (which == "t") {
                if (sink >= 0) PERR("line %lld: duplicate sink designator", lineno);
                sink = node;
            } else {
                PERR("line %lld: node designator must be 's' or 't', got '%s'", lineno, which.c_str());
            }
            if (source >= 0 && source == sink) PERR("line %lld: source and sink are the same node", lineno);
        } else if (tag == "a") {
            if (k != 4) PERR("line %lld: malformed arc line", lineno);
            long long a, b, c;
            if (node_tok(t[1], lineno, n, &a) || node_tok(t[2], lineno, n, &b) || int_tok(t[3], lineno, &c))
                return FM_INVALID_ARG;
            if (c < 0) PERR("line %lld: negative capacity %lld", lineno, c);
            if (tails && m < cap_arcs) { tails[m] = (int32_t)a; heads[m] = (int32_t)b; caps[m] = c; }
            m++;
        } else {
            PERR("line %lld: unrecognized line type '%s'", lineno, tag.c_str());
        }
    }
    if (n < 0) PERR("missing problem line");
    if (source < 0) PERR("missing source designator");
    if (sink < 0) PERR("missing sink designator");
    if (m != declared) PERR("arc count mismatch: problem line declares %lld, file has %lld", declared, m);
    if (n > INT32_MAX) PERR("node count %lld exceeds int32", n);
    out_nst[0] = (int32_t)n;
    out_nst[1] = (int32_t)source;
    out_nst[2] = (int32_t)sink;
    *out_m = m;
    if (tails && cap_arcs < m) PERR("fm_dimacs_parse_max: arrays hold %lld arcs, file has %lld",
                                    (long long)cap_arcs, m);
    return FM_OK;
}
}  // namespace

extern "C" int fm_dimacs_parse_max(const char *text, int64_t len, int32_t *out_nst, int64_t *out_m,
                                   int32_t *tails, int32_t *heads, int64_t *caps, int64_t cap_arcs) {
    try {
        return parse_max(text, len, out_nst, out_m, tails, heads, caps, cap_arcs);
    } catch (const std::bad_alloc &) {
        PERR("fm_dimacs_parse_max: out of memory");
    } catch (...) {
        PERR("fm_dimacs_parse_max: internal error");
    }
}

// Assignment: out_nm = {n (per side)}; *out_m = edges; xs/ys/ws in file order with
// X / Y ids mapped to 0..n-1 in sorted order (dimacs.py:187-248).
namespace {

int parse_asn(const char *text, int64_t len, int32_t *out_n, int64_t *out_m,
              int32_t *xs, int32_t *ys, int64_t *ws, int64_t cap_edges) {
    if (!text || len < 0 || !out_n || !out_m) PERR("fm_dimacs_parse_asn: invalid argument");
    long long n = -1, declared = 0;
    std::vector<long long> xmarks;   // designated X ids (no O(n) allocation from the header)
    struct E { long long u, v, w, line; };
    std::vector<E> raw;
    const char *p = text, *end = text + len;
    long long lineno = 0;
    Tok t[8];
    while (p < end) {
        const char *eol = (const char *)memchr(p, '\n', (size_t)(end - p));
        if (!eol) eol = end;
        lineno++;
        const int k = split(p, eol, t, 8);
        p = eol + 1;
        if (k == 0 || t[0].str() == "c") continue;
        const std::string tag = t[0].str();
        if (tag == "p") {
            if (problem_line(t, k, lineno, "asn", n >= 0, &n, &declared)) return FM_INVALID_ARG;
            continue;
        }
        if (n < 0) PERR("line %lld: '%s' line before problem line", lineno, tag.c_str());
        if (tag == "n") {
            if (k != 2) PERR("line %lld: malformed node designator", lineno);
            long long node;
            if (node_tok(t[1], lineno, n, &node)) return FM_INVALID_ARG;
            xmarks.push_back(node);
        } else if (tag == "a") {
            if (k != 4) PERR("line %lld: malformed edge line", lineno);
            long long u, v, w;
            if (node_tok(t[1], lineno, n, &u) || node_tok(t[2], lineno, n, &v) || int_tok(t[3], lineno, &w))
                return FM_INVALID_ARG;
            raw.push_back(E{u, v, w, lineno});
        } else {
            PERR("line %lld: unrecognized line type '%s'", lineno, tag.c_str());
        }
    }
    if (n < 0) PERR("missing problem line");
    std::sort(xmarks.begin(), xmarks.end());
    xmarks.erase(std::unique(xmarks.begin(), xmarks.end()), xmarks.end());
    const long long nx = (long long)xmarks.size(), ny = n - nx;
    if (nx != ny)
        PERR("X side has %lld nodes, Y side has %lld: sides must be the same size", nx, ny);
    if ((long long)raw.size() != declared)
        PERR("edge count mismatch: problem line declares %lld, file has %lld", declared, (long long)raw.size());
    if (nx < 1) PERR("n must be at least 1, got 0");
    if (nx > INT32_MAX) PERR("n = %lld exceeds int32", nx);
    *out_n = (int32_t)nx;
    *out_m = (int64_t)raw.size();
    if (!xs) return FM_OK;
    if (cap_edges < (int64_t)raw.size()) PERR("fm_dimacs_parse_asn: arrays too small");
    // X ids map to their rank among the designated ids, Y ids to their rank among the
    // rest (dimacs.py:231-247); every same-side edge is reported before duplicates
    // (the reference maps all edges, then AssignmentInstance.build checks them)
    const auto xrank = [&](long long v) -> long long {
        const auto it = std::lower_bound(xmarks.begin(), xmarks.end(), v);
        return (it != xmarks.end() && *it == v) ? (long long)(it - xmarks.begin()) : -1;
    };
    const auto yrank = [&](long long v) -> long long {
        return v - (long long)(std::lower_bound(xmarks.begin(), xmarks.end(), v) - xmarks.begin());
    };
    std::vector<unsigned long long> key(raw.size());
    for (size_t i = 0; i < raw.size(); i++) {
        const E &e = raw[i];
        long long x, y;
        const long long xu = xrank(e.u), xv = xrank(e.v);
        if (xu >= 0 && xv < 0) { x = xu; y = yrank(e.v); }
        else if (xu < 0 && xv >= 0) { x = xv; y = yrank(e.u); }
        else PERR("line %lld: edge endpoints on the same side", e.line);
        xs[i] = (int32_t)x;
        ys[i] = (int32_t)y;
        ws[i] = e.w;
        key[i] = ((unsigned long long)x << 32) | (unsigned long long)y;
    }
    // duplicates: the first repeated (x, y) in file order (AssignmentInstance.build)
    std::vector<uint32_t> order(raw.size());
    for (size_t i = 0; i < order.size(); i++) order[i] = (uint32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
    size_t first_dup = raw.size();
    for (size_t j = 1; j < order.size(); j++)
        if (key[order[j]] == key[order[j - 1]] && (j < 2 || key[order[j - 2]] != key[order[j]]))
            first_dup = std::min(first_dup, (size_t)order[j]);
    if (first_dup < raw.size()) PERR("duplicate edge (%d,%d)", xs[first_dup], ys[first_dup]);
    return FM_OK;
}

}  // namespace

// Assignment: *out_n = nodes per side; *out_m = edges; xs/ys/ws in file order with
// X / Y ids mapped to 0..n-1 in sorted order (dimacs.py:187-248).
extern "C" int fm_dimacs_parse_asn(const char *text, int64_t len, int32_t *out_n, int64_t *out_m,
                                   int32_t *xs, int32_t *ys, int64_t *ws, int64_t cap_edges) {
    try {
        return parse_asn(text, len, out_n, out_m, xs, ys, ws, cap_edges);
    } catch (const std::bad_alloc &) {
        PERR("fm_dimacs_parse_asn: out of memory");
    } catch (...) {
        PERR("fm_dimacs_parse_asn: internal error");
    }
}
