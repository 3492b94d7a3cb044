// genasm_io.cpp -- pair-list TSV in, `bitalign align` rows out (genasm_io.h).
//
// The parser reads a whole file image in parallel: the buffer is cut after
// '\n' bytes into one chunk per thread (a '\n' always ends a line, alone or
// as part of "\r\n"), pass 1 counts lines, pairs, symbols and id bytes per
// chunk and records the chunk's first malformed row, pass 2 writes codes,
// offsets and ids at the chunks' prefix sums.  Row rules follow
// io.read_pairs (pkg/src/bitalign/io.py:98-113) under Python's universal
// newlines; ASCII only (anything else is GA_IO_NONASCII, see the header).
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/genasm.h"
#include "../../include/genasm_io.h"

namespace {

// str.isspace() over ASCII (Python: \t \n \v \f \r, \x1c-\x1f, space)
inline bool py_space(unsigned char c) { return (c >= 9 && c <= 13) || (c >= 28 && c <= 32); }

struct CodeLut {
    uint8_t v[256];
    CodeLut() {
        memset(v, 4, sizeof v);
        v['A'] = v['a'] = 0;  // str.upper() then build_masks (distance.py:70-79)
        v['C'] = v['c'] = 1;
        v['G'] = v['g'] = 2;
        v['T'] = v['t'] = 3;
    }
};
const CodeLut kLut;

// symbol ids: a bijection of the upper-cased bytes with ACGT at 0..3
struct SymLut {
    uint8_t v[256];
    SymLut() {
        for (int b = 0; b < 256; ++b) v[b] = (uint8_t)((b >= 'a' && b <= 'z') ? b - 32 : b);
        const uint8_t acgt[4] = {'A', 'C', 'G', 'T'};
        for (int c = 0; c < 4; ++c) {
            v[c] = acgt[c];
            v[acgt[c]] = v[acgt[c] + 32] = (uint8_t)c;
        }
    }
};
const SymLut kSym;

struct Line {
    int64_t s, e;  // content [s, e), terminator excluded
    int64_t next;  // start of the next line
};

// the line starting at s (s < end)
inline Line next_line(const char* d, int64_t s, int64_t end) {
    int64_t p = s;
    while (p < end && d[p] != '\n' && d[p] != '\r') ++p;
    Line l{s, p, p};
    if (p < end) l.next = (d[p] == '\r' && p + 1 < end && d[p + 1] == '\n') ? p + 2 : p + 1;
    return l;
}

enum RowKind { ROW_SKIP, ROW_PAIR, ROW_BAD_COLS, ROW_EMPTY_PAT };

struct Row {
    RowKind kind;
    int64_t t1, t2;  // the two tabs of a pair row
    int cols;
};

inline Row classify(const char* d, const Line& l) {
    Row r{ROW_SKIP, -1, -1, 1};
    int64_t first = -1;
    for (int64_t p = l.s; p < l.e; ++p) {
        const unsigned char c = (unsigned char)d[p];
        if (first < 0 && !py_space(c)) first = p;
        if (c == '\t') {
            if (r.cols == 1) r.t1 = p;
            else if (r.cols == 2) r.t2 = p;
            ++r.cols;
        }
    }
    if (first < 0 || d[first] == '#') return r;  // blank or comment
    if (r.cols != 3) r.kind = ROW_BAD_COLS;
    else if (r.t2 == r.t1 + 1) r.kind = ROW_EMPTY_PAT;
    else r.kind = ROW_PAIR;
    return r;
}

struct ChunkCount {
    int64_t lines = 0, pairs = 0, symbols = 0, id_bytes = 0;
    int64_t bad_line = -1;  // line index within the chunk of the first bad row
    Row bad{};
    bool too_long = false;
    bool nonascii = false;
};

struct PairsImpl {
    ga_pairs view{};
    std::vector<uint8_t> codes, syms;
    std::vector<int64_t> pat_off, txt_off, id_off;
    std::vector<int32_t> pat_len, txt_len;
    std::vector<char> ids;
};

int resolve_threads(int nthreads) {
    if (nthreads > 0) return nthreads;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? (int)h : 1;
}

template <class F>
void parallel(int nt, F&& f) {
    if (nt <= 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt);
    for (int t = 0; t < nt; ++t) th.emplace_back([&f, t] { f(t); });
    for (auto& x : th) x.join();
}

void put_err(char* err, int64_t cap, const std::string& msg) {
    if (!err || cap <= 0) return;
    const size_t n = std::min<size_t>(msg.size(), (size_t)cap - 1);
    memcpy(err, msg.data(), n);
    err[n] = 0;
}

}  // namespace

extern "C" {

int ga_parse_pairs_tsv(const char* data, int64_t len, int nthreads, int32_t flags,
                       ga_pairs** out, char* err, int64_t err_cap) {
    const bool want_syms = flags & GA_PARSE_SYMBOLS;
    *out = nullptr;
    if (len < 0) len = 0;
    int nt = resolve_threads(nthreads);
    if (len < (int64_t)nt * (1 << 20)) nt = (int)std::max<int64_t>(1, len >> 20);
    // chunk starts: after the first '\n' at or beyond each even cut
    std::vector<int64_t> cut(nt + 1, len);
    cut[0] = 0;
    for (int t = 1; t < nt; ++t) {
        int64_t x = std::max(len * t / nt, cut[t - 1]);
        const void* q = x < len ? memchr(data + x, '\n', (size_t)(len - x)) : nullptr;
        cut[t] = q ? (const char*)q - data + 1 : len;
    }
    std::vector<ChunkCount> cc(nt);
    parallel(nt, [&](int t) {
        ChunkCount& c = cc[t];
        for (int64_t p = cut[t]; p < cut[t + 1]; ++p)
            if ((unsigned char)data[p] >= 0x80) {
                c.nonascii = true;
                return;
            }
        for (int64_t s = cut[t]; s < cut[t + 1];) {
            const Line l = next_line(data, s, cut[t + 1]);
            const Row r = classify(data, l);
            if (r.kind == ROW_PAIR) {
                const int64_t lp = r.t2 - r.t1 - 1, lt = l.e - r.t2 - 1;
                if (lp > INT32_MAX || lt > INT32_MAX) c.too_long = true;
                ++c.pairs;
                c.symbols += lp + lt;
                c.id_bytes += r.t1 - l.s;
            } else if (r.kind != ROW_SKIP && c.bad_line < 0) {
                c.bad_line = c.lines;
                c.bad = r;
            }
            ++c.lines;
            s = l.next;
        }
    });
    int64_t lines = 0;
    for (int t = 0; t < nt; ++t) {
        const ChunkCount& c = cc[t];
        if (c.nonascii) {
            put_err(err, err_cap, "non-ASCII input");
            return GA_IO_NONASCII;
        }
        if (c.bad_line >= 0) {
            const int64_t line_no = lines + c.bad_line + 1;
            std::string msg = "line " + std::to_string(line_no) + ": ";
            if (c.bad.kind == ROW_BAD_COLS)
                msg += "expected 3 tab-separated columns, got " + std::to_string(c.bad.cols);
            else
                msg += "empty pattern column";
            put_err(err, err_cap, msg);
            return GA_IO_PARSE;
        }
        if (c.too_long) {
            put_err(err, err_cap, "sequence longer than 2^31-1 symbols");
            return GA_IO_PARSE;
        }
        lines += c.lines;
    }
    PairsImpl* P = new (std::nothrow) PairsImpl;
    if (!P) return GA_IO_NOMEM;
    std::vector<int64_t> pair0(nt + 1, 0), sym0(nt + 1, 0), id0(nt + 1, 0);
    for (int t = 0; t < nt; ++t) {
        pair0[t + 1] = pair0[t] + cc[t].pairs;
        sym0[t + 1] = sym0[t] + cc[t].symbols;
        id0[t + 1] = id0[t] + cc[t].id_bytes;
    }
    const int64_t n = pair0[nt];
    try {
        P->codes.resize((size_t)std::max<int64_t>(sym0[nt], 1));
        if (want_syms) P->syms.resize((size_t)std::max<int64_t>(sym0[nt], 1));
        P->pat_off.resize((size_t)n);
        P->txt_off.resize((size_t)n);
        P->pat_len.resize((size_t)n);
        P->txt_len.resize((size_t)n);
        P->id_off.resize((size_t)n + 1);
        P->ids.resize((size_t)std::max<int64_t>(id0[nt], 1));
    } catch (const std::bad_alloc&) {
        delete P;
        put_err(err, err_cap, "out of host memory");
        return GA_IO_NOMEM;
    }
    parallel(nt, [&](int t) {
        int64_t q = pair0[t], sym = sym0[t], idb = id0[t];
        uint8_t* codes = P->codes.data();
        for (int64_t s = cut[t]; s < cut[t + 1];) {
            const Line l = next_line(data, s, cut[t + 1]);
            const Row r = classify(data, l);
            s = l.next;
            if (r.kind != ROW_PAIR) continue;
            const int64_t lid = r.t1 - l.s, lp = r.t2 - r.t1 - 1, lt = l.e - r.t2 - 1;
            memcpy(P->ids.data() + idb, data + l.s, (size_t)lid);
            P->id_off[q] = idb;
            idb += lid;
            P->pat_off[q] = sym;
            P->pat_len[q] = (int32_t)lp;
            for (int64_t x = 0; x < lp; ++x) codes[sym + x] = kLut.v[(unsigned char)data[r.t1 + 1 + x]];
            if (want_syms)
                for (int64_t x = 0; x < lp; ++x)
                    P->syms[sym + x] = kSym.v[(unsigned char)data[r.t1 + 1 + x]];
            sym += lp;
            P->txt_off[q] = sym;
            P->txt_len[q] = (int32_t)lt;
            for (int64_t x = 0; x < lt; ++x) codes[sym + x] = kLut.v[(unsigned char)data[r.t2 + 1 + x]];
            if (want_syms)
                for (int64_t x = 0; x < lt; ++x)
                    P->syms[sym + x] = kSym.v[(unsigned char)data[r.t2 + 1 + x]];
            sym += lt;
            ++q;
        }
    });
    P->id_off[n] = id0[nt];
    ga_pairs& v = P->view;
    v.n_pairs = n;
    v.codes = P->codes.data();
    v.codes_len = sym0[nt];
    v.pat_off = P->pat_off.data();
    v.pat_len = P->pat_len.data();
    v.txt_off = P->txt_off.data();
    v.txt_len = P->txt_len.data();
    v.ids = P->ids.data();
    v.id_off = P->id_off.data();
    v.syms = want_syms ? P->syms.data() : nullptr;
    v.impl = P;
    *out = &P->view;
    return GA_IO_OK;
}

void ga_pairs_free(ga_pairs* pairs) {
    if (pairs) delete static_cast<PairsImpl*>(pairs->impl);
}

int64_t ga_format_align_rows(int64_t n, const char* ids, const int64_t* id_off, const void* results,
                             const uint8_t* ops, const int64_t* ops_off, int32_t ops2, int32_t k,
                             int32_t flags, int nthreads, char* buf, int64_t cap) {
    const ga_pair_result* R = static_cast<const ga_pair_result*>(results);
    for (int64_t q = 0; q < n; ++q)
        if (R[q].status == GA_STUCK) return -2;
    int nt = resolve_threads(nthreads);
    if (n < (int64_t)nt * 256) nt = (int)std::max<int64_t>(1, n / 256);
    const bool collapse = flags & GA_ROWS_COLLAPSE_M, stats = flags & GA_ROWS_STATS;
    std::vector<std::string> part(nt);
    parallel(nt, [&](int t) {
        std::string& o = part[t];
        char num[24];
        auto put_num = [&](int64_t v) {
            const auto r = std::to_chars(num, num + sizeof num, v);
            o.append(num, r.ptr);
        };
        const int64_t q0 = n * t / nt, q1 = n * (t + 1) / nt;
        for (int64_t q = q0; q < q1; ++q) {
            const ga_pair_result& r = R[q];
            o.append(ids + id_off[q], (size_t)(id_off[q + 1] - id_off[q]));
            o.push_back('\t');
            if (r.status == GA_WINDOW_FAILED) {
                o += "ERROR WindowFailed: window ";
                put_num(r.fail_window);
                o += " found no alignment within k=";
                put_num(k);
                o.push_back('\n');
                continue;
            }
            if (r.status == GA_EMPTY_PATTERN) {
                o += "ERROR EmptyPattern: pattern must not be empty\n";
                continue;
            }
            put_num(r.cost);
            o.push_back('\t');
            put_num(r.text_consumed);
            o.push_back('\t');
            // run-length CIGAR (io.py:121-147); '='/'X' fold into 'M' when collapsing
            static const char kOps[4] = {'=', 'X', 'I', 'D'};
            const int64_t a = ops_off[q];
            char run = 0;
            int64_t run_len = 0;
            for (int64_t x = 0; x < r.ops_len; ++x) {
                char c = ops2 ? kOps[(ops[(a + x) >> 2] >> (2 * ((a + x) & 3))) & 3]
                              : (char)ops[a + x];
                if (collapse && (c == '=' || c == 'X')) c = 'M';
                if (c == run) {
                    ++run_len;
                    continue;
                }
                if (run_len) {
                    put_num(run_len);
                    o.push_back(run);
                }
                run = c;
                run_len = 1;
            }
            if (run_len) {
                put_num(run_len);
                o.push_back(run);
            }
            if (stats) {
                for (int64_t v : {r.rows_computed, r.entry_reads, r.entry_writes, r.words_allocated}) {
                    o.push_back('\t');
                    put_num(v);
                }
            }
            o.push_back('\n');
        }
    });
    int64_t total = 0;
    for (const auto& s : part) total += (int64_t)s.size();
    if (total > cap) return -1;
    int64_t at = 0;
    for (const auto& s : part) {
        memcpy(buf + at, s.data(), s.size());
        at += (int64_t)s.size();
    }
    return total;
}

}  // extern "C"

// ACGT -> 0..3, everything else 4 (the reference's masks cover exactly the
// uppercase alphabet, pkg/src/bitalign/distance.py:70-79)
static const struct AsciiLut {
    uint8_t v[256];
    AsciiLut() {
        memset(v, 4, sizeof v);
        v[(unsigned char)'A'] = 0;
        v[(unsigned char)'C'] = 1;
        v[(unsigned char)'G'] = 2;
        v[(unsigned char)'T'] = 3;
    }
} kAsciiLut;

extern "C" void ga_encode_ascii_gather(const uint64_t* ptrs, const int64_t* lens, int64_t n_seqs,
                                       uint8_t* out, int32_t threads) {
    // sequence s starts at the sum of the lengths before it; threads take
    // equal byte ranges of the output (a sequence may span two of them)
    std::vector<int64_t> start((size_t)n_seqs + 1, 0);
    for (int64_t q = 0; q < n_seqs; ++q) start[(size_t)q + 1] = start[(size_t)q] + lens[q];
    const int64_t total = start[(size_t)n_seqs];
    int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (t < 1) t = 1;
    if (total < (int64_t)1 << 20) t = 1;
    const int64_t per = (total + t - 1) / t;
    auto work = [&](int64_t a, int64_t b) {  // output bytes [a, b)
        if (a >= b) return;
        int64_t q = std::upper_bound(start.begin(), start.end(), a) - start.begin() - 1;
        for (int64_t i = a; i < b; ++q) {
            const int64_t e = std::min(b, start[(size_t)q + 1]);
            const char* src = reinterpret_cast<const char*>(ptrs[q]) + (i - start[(size_t)q]);
            for (int64_t x = i; x < e; ++x) out[x] = kAsciiLut.v[(unsigned char)src[x - i]];
            i = std::max(i, e);  // (an empty sequence leaves i where it is)
        }
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < t; ++k) pool.emplace_back(work, k * per, std::min(total, (k + 1) * per));
    work(0, std::min(total, per));
    for (auto& th : pool) th.join();
}

extern "C" void ga_encode_ascii_mt(const char* seq, int64_t n, uint8_t* out, int32_t threads) {
    const AsciiLut& lut = kAsciiLut;
    int t = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
    if (t < 1) t = 1;
    if (n < (int64_t)1 << 20) t = 1;
    const int64_t per = (n + t - 1) / t;
    auto work = [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) out[i] = lut.v[(unsigned char)seq[i]];
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < t; ++k) {
        const int64_t a = k * per, b = std::min(n, a + per);
        if (a < b) pool.emplace_back(work, a, b);
    }
    work(0, std::min(n, per));
    for (auto& th : pool) th.join();
}
