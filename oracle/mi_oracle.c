/*
 * CPU ORACLE -- test infrastructure only (plain C restatement).
 *
 * Restates the reference's dense hot path (arxiv 2411.19702, package
 * `mimatrix`) so the CUDA engine can be checked against it at sizes the
 * NumPy oracle (oracle/oracle.py) is too slow for, and so bench.py can time
 * the reference algorithm on the host cores ("cpu_baseline", kind "port").
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU leg load it.
 *
 * Citations: path:line relative to /root/reference/pkg/src/mimatrix/.
 *   column_sums            binmat.py:175-177
 *   gram_ones_kernel       _kernels.py:36-61  (AND + popcount, paired rows)
 *   gram_complete_opt.     gram.py:88-111     (g00 = n+g11-vi-vj, g01 = vj-g11)
 *   probabilities          engine.py:93-102   (p = count / n)
 *   mi_from_probabilities  engine.py:116-141  (cells (1,1),(1,0),(0,1),(0,0);
 *                                              p*log2(p/e); mirror; diagonal)
 *
 * Pinned against the real reference's outputs in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* binmat.py:175-177 */
void oracle_column_sums(const uint64_t *words, int64_t m, int64_t nw, uint64_t *v) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < m; ++j) {
        uint64_t s = 0;
        const uint64_t *w = words + j * nw;
        for (int64_t k = 0; k < nw; ++k) s += (uint64_t)__builtin_popcountll(w[k]);
        v[j] = s;
    }
}

static inline int64_t and_popcount(const uint64_t *a, const uint64_t *b, int64_t nw) {
    uint64_t acc = 0;
    for (int64_t k = 0; k < nw; ++k) acc += (uint64_t)__builtin_popcountll(a[k] & b[k]);
    return (int64_t)acc;
}

/* _kernels.py:36-61: rows u and m-1-u per parallel iteration, j >= i, mirrored. */
void oracle_gram_ones(const uint64_t *words, int64_t m, int64_t nw, int64_t *out) {
    int64_t half = (m + 1) / 2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t u = 0; u < half; ++u) {
        int64_t rows[2] = {u, m - 1 - u};
        int nr = (rows[1] != u) ? 2 : 1;
        for (int r = 0; r < nr; ++r) {
            int64_t i = rows[r];
            for (int64_t j = i; j < m; ++j) {
                int64_t c = and_popcount(words + i * nw, words + j * nw, nw);
                out[i * m + j] = c;
                out[j * m + i] = c;
            }
        }
    }
}

/* engine.py:105-113, applied to one cell. */
static inline double cell_term(double p, double e, int mode, double eps) {
    if (mode == 0) return (p > 0.0) ? p * log2(p / e) : 0.0;
    return p * log2((p + eps) / (e + eps));
}

/* engine.py:93-102 + 116-141 for one upper-triangle element (i <= j). */
static inline double mi_element(int64_t g, int64_t vi, int64_t vj, int64_t n,
                                int mode, double eps) {
    const double nf = (double)n;
    const double p11 = (double)g / nf;                     /* g11 / n            */
    const double p10 = (double)(vi - g) / nf;              /* g01.T = (v_i - g11) / n */
    const double p01 = (double)(vj - g) / nf;              /* g01 = (v_j - g11) / n   */
    const double p00 = (double)((n + g) - vi - vj) / nf;   /* g00 = n + g11 - vi - vj */
    const double p1i = (double)vi / nf, p1j = (double)vj / nf;
    const double p0i = (double)(n - vi) / nf, p0j = (double)(n - vj) / nf;
    double mi = 0.0;
    mi += cell_term(p11, p1i * p1j, mode, eps);
    mi += cell_term(p10, p1i * p0j, mode, eps);
    mi += cell_term(p01, p0i * p1j, mode, eps);
    mi += cell_term(p00, p0i * p0j, mode, eps);
    return mi;
}

/*
 * engine.mi_all_pairs(dense) fused: per pair count (gram_ones algorithm),
 * closed-form cells, fp64 epilogue in the reference's order, mirrored.
 * Returns 0, or 3 when a derived count leaves [0, n] (gram.py:108-110).
 */
int oracle_mi_all_pairs(const uint64_t *words, int64_t m, int64_t nw, int64_t n,
                        int mode, double eps, int include_diagonal, double *out) {
    uint64_t *v = (uint64_t *)malloc((size_t)m * sizeof(uint64_t));
    if (!v) return 1;
    oracle_column_sums(words, m, nw, v);
    int bad = 0;
    for (int64_t j = 0; j < m; ++j)
        if ((int64_t)v[j] > n) bad = 1;
    if (bad) { free(v); return 3; }
    int64_t half = (m + 1) / 2;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
    for (int64_t u = 0; u < half; ++u) {
        int64_t rows[2] = {u, m - 1 - u};
        int nr = (rows[1] != u) ? 2 : 1;
        for (int r = 0; r < nr; ++r) {
            int64_t i = rows[r];
            const uint64_t *wi = words + i * nw;
            for (int64_t j = i; j < m; ++j) {
                int64_t g = and_popcount(wi, words + j * nw, nw);
                int64_t vi = (int64_t)v[i], vj = (int64_t)v[j];
                int64_t g00 = (n + g) - vi - vj;
                if (g < 0 || g > n || vi - g < 0 || vj - g < 0 || g00 < 0 || g00 > n) bad |= 1;
                double x = mi_element(g, vi, vj, n, mode, eps);
                if (i == j && !include_diagonal) x = 0.0;
                out[i * m + j] = x;
                out[j * m + i] = x;
            }
        }
    }
    free(v);
    return bad ? 3 : 0;
}

/* MI from an existing count matrix (for cross-checking an exported G). */
int oracle_mi_from_gram(const int64_t *g11, const uint64_t *v, int64_t m, int64_t n,
                        int mode, double eps, int include_diagonal, double *out) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = i; j < m; ++j) {
            double x = mi_element(g11[i * m + j], (int64_t)v[i], (int64_t)v[j], n, mode, eps);
            if (i == j && !include_diagonal) x = 0.0;
            out[i * m + j] = x;
            out[j * m + i] = x;
        }
    }
    return 0;
}

/*
 * datagen.py:44-73 stream (draw k = r*m + c + 1, state seed + k*gamma) packed
 * straight into words, for the listed columns only (cols == NULL: all).
 * kind[c]: 0 Bernoulli(thr[c]), 1 all zero, 2 all one, 3 src[c] XOR
 * Bernoulli(flip_thr) drawn from the flip_seed stream at the target's index.
 */
static inline uint64_t splitmix64_draw(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void oracle_generate_words(uint64_t *words, int64_t n, int64_t m, uint64_t seed, const uint64_t *thr,
                           const uint8_t *kind, const int32_t *src, uint64_t flip_thr, uint64_t flip_seed,
                           const int64_t *cols, int64_t ncols_out) {
    const int64_t nw = (n + 63) / 64;
#pragma omp parallel for schedule(static)
    for (int64_t idx = 0; idx < ncols_out * nw; ++idx) {
        const int64_t k = idx / nw, w = idx % nw;
        const int64_t c = cols ? cols[k] : k;
        const int64_t r0 = w * 64;
        const int64_t nr = (n - r0) < 64 ? (n - r0) : 64;
        uint64_t out = 0;
        for (int64_t b = 0; b < nr; ++b) {
            const uint64_t row = (uint64_t)(r0 + b) * (uint64_t)m;
            uint64_t bit = 0;
            switch (kind[c]) {
            case 0: bit = splitmix64_draw(seed, row + (uint64_t)c + 1) < thr[c]; break;
            case 1: bit = 0; break;
            case 2: bit = 1; break;
            default:
                bit = (splitmix64_draw(seed, row + (uint64_t)src[c] + 1) < thr[src[c]]) ^
                      (splitmix64_draw(flip_seed, row + (uint64_t)c + 1) < flip_thr);
            }
            out |= bit << b;
        }
        words[k * nw + w] = out;
    }
}
