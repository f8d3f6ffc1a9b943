// Float-hex text I/O for snapshots and element records, host side.
//
// The reference writes every embedding component with Python's float.hex
// (pkg/src/semcache/index.py:343-346 snapshot lines, model.py:237 element
// records) and reads it back with float.fromhex (index.py:370, model.py:263).
// These routines produce byte-identical text (CPython float_hex:
// "[-]0x1.<13 hex digits>p[+-]e", "0x0.<13>p-1022" for subnormals,
// "0x0.0p+0" for zero, repr for inf/nan) and parse it bit-exactly, split
// across host threads.  Non-canonical tokens (other hex layouts, decimal,
// inf/nan spellings) fall back to strtod, which reads hex floats exactly.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace sine {
namespace hexio {

constexpr int kMaxTok = 24;   // "-0x1.fffffffffffffp-1022"
constexpr int kMaxId = 21;    // int64 + separator

inline int fmt_double(double x, char* o) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    const bool neg = (b >> 63) != 0;
    const int be = static_cast<int>((b >> 52) & 0x7ff);
    const uint64_t mant = b & ((1ull << 52) - 1);
    char* p = o;
    if (be == 0x7ff) {  // repr(): 'nan' never carries a sign
        const char* s = mant ? "nan" : (neg ? "-inf" : "inf");
        const size_t n = std::strlen(s);
        std::memcpy(p, s, n);
        return static_cast<int>(n);
    }
    if (neg) *p++ = '-';
    if (be == 0 && mant == 0) {
        std::memcpy(p, "0x0.0p+0", 8);
        return static_cast<int>(p - o) + 8;
    }
    *p++ = '0';
    *p++ = 'x';
    *p++ = be ? '1' : '0';
    *p++ = '.';
    static const char* hx = "0123456789abcdef";
    for (int i = 12; i >= 0; --i) *p++ = hx[(mant >> (4 * i)) & 0xf];
    *p++ = 'p';
    int e = be ? be - 1023 : -1022;
    *p++ = e < 0 ? '-' : '+';
    if (e < 0) e = -e;
    char d[8];
    int nd = 0;
    do {
        d[nd++] = static_cast<char>('0' + e % 10);
        e /= 10;
    } while (e);
    while (nd) *p++ = d[--nd];
    return static_cast<int>(p - o);
}

inline int fmt_i64(int64_t v, char* o) {
    char d[24];
    int nd = 0;
    uint64_t u = v < 0 ? static_cast<uint64_t>(-(v + 1)) + 1 : static_cast<uint64_t>(v);
    do {
        d[nd++] = static_cast<char>('0' + u % 10);
        u /= 10;
    } while (u);
    char* p = o;
    if (v < 0) *p++ = '-';
    while (nd) *p++ = d[--nd];
    return static_cast<int>(p - o);
}

inline int hexval(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    return -1;
}

// Parse one token [s, e); false if it is not a float.
inline bool parse_double(const char* s, const char* e, double* out) {
    const char* p = s;
    bool neg = false;
    if (p < e && (*p == '-' || *p == '+')) neg = *p++ == '-';
    // canonical normal: 0x1.<13 hex>p<sign><digits>
    if (e - p >= 20 && p[0] == '0' && (p[1] == 'x' || p[1] == 'X') && p[2] == '1' && p[3] == '.' && p[17] == 'p') {
        uint64_t mant = 0;
        bool ok = true;
        for (int i = 0; i < 13; ++i) {
            const int v = hexval(p[4 + i]);
            ok &= v >= 0;
            mant = (mant << 4) | static_cast<uint64_t>(v < 0 ? 0 : v);
        }
        const char* q = p + 18;
        bool eneg = false;
        if (q < e && (*q == '+' || *q == '-')) eneg = *q++ == '-';
        int ex = 0, nd = 0;
        while (q < e && *q >= '0' && *q <= '9' && nd < 6) ex = ex * 10 + (*q++ - '0'), ++nd;
        if (ok && nd && q == e) {
            const int be = (eneg ? -ex : ex) + 1023;
            if (be >= 1 && be <= 2046) {
                const uint64_t b = (static_cast<uint64_t>(neg) << 63) | (static_cast<uint64_t>(be) << 52) | mant;
                std::memcpy(out, &b, 8);
                return true;
            }
        }
    }
    // anything else (zero, subnormals, other layouts, inf/nan): strtod
    std::string tok(s, e);
    char* end = nullptr;
    const double v = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size() || tok.empty()) return false;
    *out = v;
    return true;
}

template <typename F>
inline void parallel_for_n(int64_t nt, F&& f) {
    if (nt <= 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t) th.emplace_back([&, t] { f(t); });
    for (auto& x : th) x.join();
}

template <typename F>
inline void parallel_for(int64_t n, F&& f) {
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 256));
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt); });
    for (auto& x : th) x.join();
}

inline int tok_len(double x) {
    char tmp[kMaxTok + 1];
    return fmt_double(x, tmp);
}

inline int i64_len(int64_t v) {
    char tmp[24];
    return fmt_i64(v, tmp);
}

// Lines "[<id> ]<hex> <hex> ...\n" for n rows of d doubles, written in
// place: per-row lengths, a prefix sum, then every thread formats its rows
// straight into `out` (one pass over the output, no staging copies).
// Returns the byte count; out must hold n * (kMaxId + d * (kMaxTok + 1) + 1).
inline int64_t format_rows(const int64_t* ids, const double* rows, int64_t n, int64_t d, char* out) {
    std::vector<int64_t> off(static_cast<size_t>(n) + 1, 0);
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            int64_t L = ids ? i64_len(ids[i]) + 1 : 0;
            for (int64_t j = 0; j < d; ++j) L += tok_len(rows[i * d + j]) + 1;  // separators + '\n'
            off[i + 1] = L;
        }
    });
    for (int64_t i = 0; i < n; ++i) off[i + 1] += off[i];
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            char* p = out + off[i];
            if (ids) {
                p += fmt_i64(ids[i], p);
                *p++ = ' ';
            }
            for (int64_t j = 0; j < d; ++j) {
                if (j) *p++ = ' ';
                p += fmt_double(rows[i * d + j], p);
            }
            *p++ = '\n';
        }
    });
    return off[n];
}

// Parse n lines of ("<id> " if ids) + d space-separated floats; lines end
// with '\n' (the last may end at len).  Returns "" or an error message.
inline std::string parse_rows(const char* text, int64_t len, int64_t n, int64_t d, int64_t* ids, double* rows) {
    // line starts: newline counts per text chunk (parallel), prefix, then
    // each chunk records its starts at the global line index
    std::vector<int64_t> start(static_cast<size_t>(n) + 1);
    {
        const int64_t nc = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), len >> 20));
        std::vector<int64_t> cnt(nc + 1, 0);
        auto chunk = [&](int64_t c, int64_t& a, int64_t& b) {
            a = len * c / nc;
            b = len * (c + 1) / nc;
        };
        parallel_for_n(nc, [&](int64_t c) {
            int64_t a, b, k = 0;
            chunk(c, a, b);
            for (const char* p = text + a; (p = static_cast<const char*>(std::memchr(p, '\n', text + b - p)));
                 ++p)
                ++k;
            cnt[c + 1] = k;
        });
        for (int64_t c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
        const int64_t nl = cnt[nc];
        const bool tail = len > 0 && text[len - 1] != '\n';  // last line without a newline
        if (nl + (tail ? 1 : 0) < n)
            return "expected " + std::to_string(n) + " lines, got " + std::to_string(nl + (tail ? 1 : 0));
        start[0] = 0;
        parallel_for_n(nc, [&](int64_t c) {
            int64_t a, b, k = cnt[c];
            chunk(c, a, b);
            for (const char* p = text + a; k < n && (p = static_cast<const char*>(std::memchr(p, '\n', text + b - p)));
                 ++p)
                start[++k] = (p - text) + 1;
        });
        if (nl < n) start[n] = len + 1;  // the unterminated last line
    }
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 256));
    std::vector<int64_t> badat(nt, -1);
    std::vector<std::string> badmsg(nt);
    auto work = [&](int64_t t) {
        const int64_t a = n * t / nt, b = n * (t + 1) / nt;
        for (int64_t i = a; i < b; ++i) {
            const char* s = text + start[i];
            const char* e = text + start[i + 1] - 1;  // excludes '\n' (or the end)
            if (e > text + len) e = text + len;
            int64_t tok = 0;
            const int64_t want = d + (ids ? 1 : 0);
            const char* p = s;
            while (true) {
                const char* q = static_cast<const char*>(std::memchr(p, ' ', static_cast<size_t>(e - p)));
                const char* te = q ? q : e;
                if (tok >= want) {
                    badat[t] = i, badmsg[t] = "too many fields";
                    return;
                }
                if (ids && tok == 0) {
                    char* end = nullptr;
                    std::string v(p, te);
                    ids[i] = std::strtoll(v.c_str(), &end, 10);
                    if (v.empty() || end != v.c_str() + v.size()) {
                        badat[t] = i, badmsg[t] = "malformed id '" + v + "'";
                        return;
                    }
                } else if (!parse_double(p, te, rows + i * d + (tok - (ids ? 1 : 0)))) {
                    badat[t] = i, badmsg[t] = "malformed float '" + std::string(p, te) + "'";
                    return;
                }
                ++tok;
                if (!q) break;
                p = q + 1;
            }
            if (tok != want) {
                badat[t] = i, badmsg[t] = "expected " + std::to_string(want) + " fields, got " + std::to_string(tok);
                return;
            }
        }
    };
    if (nt == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int64_t t = 0; t < nt; ++t) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }
    for (int64_t t = 0; t < nt; ++t)
        if (badat[t] >= 0) return "line " + std::to_string(badat[t] + 1) + ": " + badmsg[t];
    return "";
}

}  // namespace hexio
}  // namespace sine
