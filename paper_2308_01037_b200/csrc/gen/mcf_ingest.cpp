// Graph-file parsers for load_graph (reference sparsemat.py:165-245): edge
// lists and coordinate Matrix Market files read in one pass into edge arrays.
// Host code -- text parsing -- with the reference's accept/reject rules and
// line numbers; the filters that follow (loops, undirected expansion,
// duplicates, isolated nodes) run on the device (ingest.py).
//
// Usage from Python: h = open(path, format) parses everything and reports the
// edge count (or an error code + line); copy(h, u, v) fills int64 arrays;
// close(h) frees.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define GEN_API extern "C" __attribute__((visibility("default")))

namespace {

enum Err {
    OK = 0,
    E_FEW_COLUMNS = 1,      // edgelist: "expected at least two columns"
    E_NOT_INT = 2,          // edgelist: "node ids must be integers"
    E_NEGATIVE = 3,         // edgelist: "node ids must be non-negative"
    E_NOT_FOUND = 4,        // cannot open the file
    E_MM_HEADER = 10,       // "missing MatrixMarket header"
    E_MM_KIND = 11,         // "only 'matrix coordinate' files are supported"
    E_MM_VALUE = 12,        // "unsupported value type"
    E_MM_STORAGE = 13,      // "unsupported storage"
    E_MM_SIZE = 14,         // "size line must be 'rows cols nnz'"
    E_MM_SQUARE = 15,       // "adjacency matrix must be square"
    E_MM_COLUMNS = 16,      // "expected N columns"
    E_MM_MALFORMED = 17,    // "malformed entry"
    E_MM_RANGE = 18,        // "index out of declared range"
    E_MM_NO_SIZE = 19,      // "missing size line"
};

struct Parsed {
    std::vector<int64_t> u, v;
    int64_t err_line = 0;
    int err = OK;
    int expected_cols = 0;
};

// split a line on ASCII whitespace (Python str.split())
void split(const std::string &s, std::vector<std::string> &out) {
    out.clear();
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && isspace((unsigned char)s[i])) ++i;
        size_t j = i;
        while (j < s.size() && !isspace((unsigned char)s[j])) ++j;
        if (j > i) out.emplace_back(s, i, j - i);
        i = j;
    }
}

// Python int() on a token: optional sign, decimal digits (underscores between digits allowed)
bool parse_int(const std::string &t, int64_t &out) {
    size_t i = 0;
    bool neg = false;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
    if (i >= t.size()) return false;
    __int128 val = 0;
    bool prev_digit = false;
    for (; i < t.size(); ++i) {
        const char c = t[i];
        if (c >= '0' && c <= '9') {
            val = val * 10 + (c - '0');
            if (val > ((__int128)1 << 62)) return false;
            prev_digit = true;
        } else if (c == '_' && prev_digit && i + 1 < t.size() && t[i + 1] >= '0' && t[i + 1] <= '9') {
            prev_digit = false;
        } else {
            return false;
        }
    }
    out = (int64_t)(neg ? -val : val);
    return true;
}

// Python float() on a token (decimal / exponent / inf / nan forms)
bool parse_float(const std::string &t, double &out) {
    errno = 0;
    char *end = nullptr;
    out = strtod(t.c_str(), &end);
    return end && *end == '\0' && end != t.c_str();
}

bool read_line(FILE *f, std::string &line) {
    line.clear();
    int c;
    bool any = false;
    while ((c = fgetc(f)) != EOF) {
        any = true;
        if (c == '\n') return true;
        line.push_back((char)c);
    }
    return any;
}

std::string strip(const std::string &s) {
    size_t a = 0, b = s.size();
    while (a < b && isspace((unsigned char)s[a])) ++a;
    while (b > a && isspace((unsigned char)s[b - 1])) --b;
    return s.substr(a, b - a);
}

void parse_edgelist(FILE *f, Parsed &p) {
    std::string line;
    std::vector<std::string> parts;
    int64_t lineno = 0;
    while (read_line(f, line)) {
        ++lineno;
        const std::string s = strip(line);
        if (s.empty() || s[0] == '#' || s[0] == '%') continue;
        split(s, parts);
        if (parts.size() < 2) {
            p.err = E_FEW_COLUMNS;
            p.err_line = lineno;
            return;
        }
        int64_t a, b;
        if (!parse_int(parts[0], a) || !parse_int(parts[1], b)) {
            p.err = E_NOT_INT;
            p.err_line = lineno;
            return;
        }
        if (a < 0 || b < 0) {
            p.err = E_NEGATIVE;
            p.err_line = lineno;
            return;
        }
        p.u.push_back(a);
        p.v.push_back(b);
    }
}

std::string lower(std::string s) {
    for (auto &c : s) c = (char)tolower((unsigned char)c);
    return s;
}

void parse_mm(FILE *f, Parsed &p) {
    std::string line;
    std::vector<std::string> parts;
    if (!read_line(f, line) || line.rfind("%%MatrixMarket", 0) != 0) {
        p.err = E_MM_HEADER;
        p.err_line = 1;
        return;
    }
    split(strip(line), parts);
    if (parts.size() < 5 || lower(parts[1]) != "matrix" || lower(parts[2]) != "coordinate") {
        p.err = E_MM_KIND;
        p.err_line = 1;
        return;
    }
    const std::string vt = lower(parts[3]), st = lower(parts[4]);
    if (vt != "real" && vt != "pattern" && vt != "integer") {
        p.err = E_MM_VALUE;
        p.err_line = 1;
        return;
    }
    if (st != "general" && st != "symmetric") {
        p.err = E_MM_STORAGE;
        p.err_line = 1;
        return;
    }
    const bool pattern = vt == "pattern", symmetric = st == "symmetric";
    int64_t size = -1, lineno = 1;
    while (read_line(f, line)) {
        ++lineno;
        const std::string s = strip(line);
        if (s.empty() || s[0] == '%') continue;
        split(s, parts);
        if (size < 0) {
            int64_t nr, nc, nz;
            if (parts.size() != 3 || !parse_int(parts[0], nr) || !parse_int(parts[1], nc) || !parse_int(parts[2], nz)) {
                p.err = E_MM_SIZE;
                p.err_line = lineno;
                return;
            }
            if (nr != nc) {
                p.err = E_MM_SQUARE;
                p.err_line = lineno;
                return;
            }
            size = nr;
            continue;
        }
        const size_t want = pattern ? 2 : 3;
        if (parts.size() < want) {
            p.err = E_MM_COLUMNS;
            p.expected_cols = (int)want;
            p.err_line = lineno;
            return;
        }
        int64_t i, j;
        double value = 1.0;
        if (!parse_int(parts[0], i) || !parse_int(parts[1], j) || (!pattern && !parse_float(parts[2], value))) {
            p.err = E_MM_MALFORMED;
            p.err_line = lineno;
            return;
        }
        i -= 1;
        j -= 1;
        if (i < 0 || j < 0 || i >= size || j >= size) {
            p.err = E_MM_RANGE;
            p.err_line = lineno;
            return;
        }
        if (value == 0.0) continue;
        p.u.push_back(i);
        p.v.push_back(j);
        if (symmetric && i != j) {
            p.u.push_back(j);
            p.v.push_back(i);
        }
    }
    if (size < 0) {
        p.err = E_MM_NO_SIZE;
        p.err_line = 0;
    }
}

}  // namespace

// format 0 = edgelist, 1 = matrix market.  Returns a handle (never null);
// query it with mcfgen_parsed_info.
GEN_API void *mcfgen_parse_open(const char *path, int format) {
    Parsed *p = new Parsed();
    FILE *f = fopen(path, "rb");
    if (!f) {
        p->err = E_NOT_FOUND;
        return p;
    }
    if (format == 0)
        parse_edgelist(f, *p);
    else
        parse_mm(f, *p);
    fclose(f);
    return p;
}

// edges parsed (or -1 on error, with *err and *err_line set)
GEN_API int64_t mcfgen_parsed_info(void *h, int *err, int64_t *err_line, int *expected_cols) {
    const Parsed *p = static_cast<const Parsed *>(h);
    *err = p->err;
    *err_line = p->err_line;
    *expected_cols = p->expected_cols;
    return p->err ? -1 : (int64_t)p->u.size();
}

GEN_API void mcfgen_parsed_copy(void *h, int64_t *u, int64_t *v) {
    const Parsed *p = static_cast<const Parsed *>(h);
    memcpy(u, p->u.data(), sizeof(int64_t) * p->u.size());
    memcpy(v, p->v.data(), sizeof(int64_t) * p->v.size());
}

GEN_API void mcfgen_parse_close(void *h) { delete static_cast<Parsed *>(h); }
