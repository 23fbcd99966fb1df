// Host-side synthetic graph generators for the benchmark workloads
// (BASELINE.json configs; workload generation is outside the hot path,
// SURVEY.md §2.1 row 4).  Output: sorted, duplicate-free symmetric CSR.
#include <stdint.h>

#include <algorithm>
#include <vector>

namespace {

struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t n) { return (uint64_t)(((__uint128_t)next() * n) >> 64); }
};

void to_csr(int64_t n, const std::vector<int64_t> &u, const std::vector<int64_t> &v, int64_t *row_ptr,
            int32_t *col_ids) {
    std::vector<int64_t> deg(n + 1, 0);
    for (size_t e = 0; e < u.size(); ++e) {
        ++deg[u[e] + 1];
        ++deg[v[e] + 1];
    }
    for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
    for (int64_t i = 0; i <= n; ++i) row_ptr[i] = deg[i];
    std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
    for (size_t e = 0; e < u.size(); ++e) {
        col_ids[fill[u[e]]++] = (int32_t)v[e];
        col_ids[fill[v[e]]++] = (int32_t)u[e];
    }
    for (int64_t i = 0; i < n; ++i) std::sort(col_ids + row_ptr[i], col_ids + row_ptr[i + 1]);
}

}  // namespace

extern "C" {

// Preferential attachment (Barabasi-Albert): a star on m+1 nodes, then every
// new node attaches to m distinct targets drawn from the degree-weighted
// repeated-node list.  nnz = 2 (m + (n - m - 1) m).  Returns nnz, or -1.
__attribute__((visibility("default"))) int64_t mcfgen_ba_nnz(int64_t n, int64_t m) {
    if (m < 1 || n <= m + 1) return -1;
    return 2 * (m + (n - m - 1) * m);
}

__attribute__((visibility("default"))) int64_t mcfgen_barabasi_albert(int64_t n, int64_t m, uint64_t seed,
                                                                      int64_t *row_ptr, int32_t *col_ids) {
    if (m < 1 || n <= m + 1) return -1;
    SplitMix64 rng{seed * 0x2545F4914F6CDD1Dull + 0x1234567ull};
    std::vector<int64_t> u, v, rep;
    u.reserve((size_t)(n * m));
    v.reserve((size_t)(n * m));
    rep.reserve((size_t)(2 * n * m));
    for (int64_t j = 1; j <= m; ++j) {  // star_graph(m): center 0
        u.push_back(0);
        v.push_back(j);
        rep.push_back(0);
        rep.push_back(j);
    }
    std::vector<int64_t> tgt(m);
    for (int64_t src = m + 1; src < n; ++src) {
        int64_t got = 0;
        while (got < m) {
            int64_t t = rep[rng.below(rep.size())];
            bool dup = false;
            for (int64_t k = 0; k < got; ++k) dup |= (tgt[k] == t);
            if (!dup) tgt[got++] = t;
        }
        for (int64_t k = 0; k < m; ++k) {
            u.push_back(src);
            v.push_back(tgt[k]);
            rep.push_back(tgt[k]);
            rep.push_back(src);
        }
    }
    to_csr(n, u, v, row_ptr, col_ids);
    return (int64_t)(2 * u.size());
}

}  // extern "C"
