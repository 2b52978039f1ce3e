/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct CPU implementation of what the hot path
 * computes, written from the paper (arXiv 1303.3692, /root/reference/PAPER.md,
 * cited "P:L<line>").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg / `--impl reference` arm may load this library.  It shares
 * no code, header, table or helper with the CUDA library in
 * paper_1303_3692_b200/; the only thing both sides consume is the seeded input
 * module synth/.
 *
 * What is computed (readings A1-A16 in DESIGN.md):
 *   - text S[0..n) over a<c<g<t (Sec. III), 0-based (A1);
 *   - the suffix array: all suffix start positions in lexicographic order, a
 *     suffix that is a proper prefix of another sorting first, no sentinel
 *     (Table I; reading A2).  Built by "create an array ... and then
 *     apply a sorting algorithm": a comparison sort.
 *   - per query P (length m), with t_i = S[i .. min(i+m, n)) (A7):
 *         lo(P) = #{ i : t_i <  P }      hi(P) = #{ i : t_i <= P }
 *     so [lo, hi) is the paper's [LB, RB] as a half-open interval (P:L161,
 *     Sec. IV; A3), empty when P does not occur (A5), and the positions are
 *     SA[lo..hi) in SA order ("namely 9, 0, 5"; A15).
 *   - the textbook binary searches (Alg. 1) with virtual
 *     sentinels L=-1, R=n (A4) and the comparison direction corrected (A6):
 *     LB loop moves R when P <= t_pivot, RB loop when P < t_pivot.
 *
 * Parity pins live in tests/ (paper worked examples, brute force, closed
 * forms, invariants); see DESIGN.md "Oracle pins".
 *
 * Query layout read here (the input format of include/sa.h, produced by
 * synth/): base j of query q is 2 bits at word q*stride + j/32, bit
 * 62-2*(j%32), codes A=0 C=1 G=2 T=3.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- alphabet (Sigma = {a,c,g,t}, ordered a<c<g<t; reading A2) ---- */

/* ASCII -> codes 0..3.  Case-insensitive.  Returns -1 on success, else the
 * index of the first byte that is not A/C/G/T (reading A13). */
int64_t oracle_encode(const char *ascii, int64_t n, uint8_t *codes) {
    for (int64_t i = 0; i < n; ++i) {
        switch (ascii[i]) {
        case 'A': case 'a': codes[i] = 0; break;
        case 'C': case 'c': codes[i] = 1; break;
        case 'G': case 'g': codes[i] = 2; break;
        case 'T': case 't': codes[i] = 3; break;
        default: return i;
        }
    }
    return -1;
}

/* Query q, base j, from the packed layout. */
static inline uint8_t query_base(const uint64_t *words, uint32_t stride, int64_t q, int64_t j) {
    return (uint8_t)((words[q * (int64_t)stride + (j >> 5)] >> (62 - 2 * (j & 31))) & 3u);
}

static void decode_query(const uint64_t *words, uint32_t stride, int64_t q, int64_t m, uint8_t *P) {
    for (int64_t j = 0; j < m; ++j) P[j] = query_base(words, stride, q, j);
}

static inline int64_t query_len(const uint32_t *lens, uint32_t fixed_len, int64_t q) {
    return lens ? (int64_t)lens[q] : (int64_t)fixed_len;
}

/* ---- suffix order (Table I) ---------------------------------- */

/* Lexicographic order of the full suffixes S_i and S_j; a proper prefix sorts
 * first (Table I: "ac"(9) < "acggtacgtac"(0)). */
static int suffix_cmp(const uint8_t *S, int64_t n, int64_t i, int64_t j) {
    int64_t li = n - i, lj = n - j, l = li < lj ? li : lj;
    int c = memcmp(S + i, S + j, (size_t)l);
    if (c != 0) return c < 0 ? -1 : 1;
    if (li == lj) return 0;
    return li < lj ? -1 : 1;
}

typedef struct { const uint8_t *S; int64_t n; } sa_ctx;

static int sa_qsort_cmp(const void *a, const void *b, void *arg) {
    const sa_ctx *c = (const sa_ctx *)arg;
    return suffix_cmp(c->S, c->n, (int64_t)*(const uint32_t *)a, (int64_t)*(const uint32_t *)b);
}

/* "create an array with all the suffix elements ... and then apply a
 * sorting algorithm".  n must be < 2^32. */
void oracle_sa_naive(const uint8_t *S, int64_t n, uint32_t *sa) {
    for (int64_t i = 0; i < n; ++i) sa[i] = (uint32_t)i;
    sa_ctx c = {S, n};
    qsort_r(sa, (size_t)n, sizeof(uint32_t), sa_qsort_cmp, &c);
}

/* ---- the comparison of Sec. IV, truncated (reading A7) ----- */

/* sign(P - t_s) where t_s = S[s .. min(s+m, n)):
 *   0  : P is a prefix of S_s            (case 1)
 *  -1  : P < t_s                         (case 2)
 *  +1  : P > t_s, including the case where S_s is a proper prefix of P  (A7) */
int oracle_cmp(const uint8_t *S, int64_t n, int64_t s, const uint8_t *P, int64_t m) {
    int64_t len = n - s;
    int64_t l = m < len ? m : len;
    for (int64_t j = 0; j < l; ++j) {
        if (P[j] != S[s + j]) return P[j] < S[s + j] ? -1 : 1;
    }
    if (l < m) return 1; /* the suffix ended first: it is a proper prefix of P, so t_s < P */
    return 0;
}

/* Alg. 1 as the textbook pair of binary searches, sentinels
 * L=-1, R=n (A4), comparisons corrected (A6):
 *   LB loop: while R > L+1 { p=(L+R)>>1; if P <= t_p then R=p else L=p }  lo = R
 *   RB loop: while R > L+1 { p=(L+R)>>1; if P <  t_p then R=p else L=p }  hi = R
 * (the paper's RB = hi-1 when hi > lo; reading A3). */
void oracle_search(const uint8_t *S, int64_t n, const uint32_t *sa, const uint8_t *P, int64_t m,
                   uint64_t *lo, uint64_t *hi) {
    int64_t L = -1, R = n;
    while (R > L + 1) {
        int64_t p = (L + R) >> 1;
        if (oracle_cmp(S, n, sa[p], P, m) <= 0) R = p; else L = p;
    }
    *lo = (uint64_t)R;
    L = -1; R = n;
    while (R > L + 1) {
        int64_t p = (L + R) >> 1;
        if (oracle_cmp(S, n, sa[p], P, m) < 0) R = p; else L = p;
    }
    *hi = (uint64_t)R;
}

/* The plain definition by scanning every suffix: lo = #{t_i < P}, hi = #{t_i <= P}. */
void oracle_count(const uint8_t *S, int64_t n, const uint8_t *P, int64_t m, uint64_t *lo, uint64_t *hi) {
    uint64_t a = 0, b = 0;
    for (int64_t i = 0; i < n; ++i) {
        int c = oracle_cmp(S, n, i, P, m);
        if (c > 0) ++a;
        if (c >= 0) ++b;
    }
    *lo = a;
    *hi = b;
}

/* ---- batch drivers over packed queries ---------------------------------- */

/* Textbook search for every query; a static block partition of the queries
 * over threads (output identical for any thread count).  lohi: 2Q uint64. */
int oracle_search_batch(const uint8_t *S, int64_t n, const uint32_t *sa, const uint64_t *words, uint32_t stride,
                        const uint32_t *lens, uint32_t fixed_len, int64_t Q, uint64_t *lohi, int nthreads) {
    set_threads(nthreads);
    int64_t mmax = 0;
    for (int64_t q = 0; q < Q; ++q) { int64_t m = query_len(lens, fixed_len, q); if (m > mmax) mmax = m; }
    int err = 0;
#pragma omp parallel
    {
        uint8_t *P = (uint8_t *)malloc((size_t)mmax + 1);
        if (!P) {
#pragma omp atomic write
            err = 1;
        }
#pragma omp for schedule(static)
        for (int64_t q = 0; q < Q; ++q) {
            if (!P) continue;
            int64_t m = query_len(lens, fixed_len, q);
            decode_query(words, stride, q, m, P);
            oracle_search(S, n, sa, P, m, &lohi[2 * q], &lohi[2 * q + 1]);
        }
        free(P);
    }
    return err ? -1 : 0;
}

/* Streaming counting oracle (no suffix array): for a batch of queries compute
 * lo and hi straight from the definition with one pass over all n suffixes.
 *
 * lo(P) = #{i : S_i < P}  and  hi(P) = #{i : S_i < P+}  where S_i is the full
 * suffix and P+ stands for "P followed by a symbol larger than every base"
 * (t_i < P  <=>  S_i < P, and t_i <= P  <=>  S_i < P+, A7).  The 2Q keys
 * {P, P+} are sorted; each suffix is placed among them by binary search
 * (c(i) = first key greater than S_i); a histogram of c(i) and its prefix sum
 * give #{i : S_i < K_j} for every key K_j. */
typedef struct { const uint8_t *P; int64_t m; int plus; int64_t q; } okey;

static int key_cmp(const void *a, const void *b) {
    const okey *x = (const okey *)a, *y = (const okey *)b;
    int64_t l = x->m < y->m ? x->m : y->m;
    int c = memcmp(x->P, y->P, (size_t)l);
    if (c != 0) return c < 0 ? -1 : 1;
    if (x->m == y->m) {
        if (x->plus != y->plus) return x->plus < y->plus ? -1 : 1;
        return x->q < y->q ? -1 : (x->q > y->q);
    }
    /* one is a proper prefix of the other */
    if (x->m < y->m) return x->plus ? 1 : -1; /* x=P < anything longer; x=P+ > anything starting with P */
    return y->plus ? -1 : 1;
}

/* sign(S_i - K): S_i against a key */
static int suffix_vs_key(const uint8_t *S, int64_t n, int64_t i, const okey *k) {
    int64_t len = n - i, l = len < k->m ? len : k->m;
    int c = memcmp(S + i, k->P, (size_t)l);
    if (c != 0) return c < 0 ? -1 : 1;
    if (len < k->m) return -1;   /* S_i is a proper prefix of P: S_i < P and < P+ */
    return k->plus ? -1 : 1;     /* P is a prefix of S_i: S_i >= P (never equal to P+), S_i < P+ */
    /* (S_i == P exactly is reported as +1 = "not less than P", which is all the count uses) */
}

int oracle_count_batch(const uint8_t *S, int64_t n, const uint64_t *words, uint32_t stride, const uint32_t *lens,
                       uint32_t fixed_len, int64_t Q, uint64_t *lohi, int nthreads) {
    set_threads(nthreads);
    int64_t tot = 0;
    for (int64_t q = 0; q < Q; ++q) tot += query_len(lens, fixed_len, q);
    uint8_t *buf = (uint8_t *)malloc((size_t)tot + 1);
    okey *keys = (okey *)malloc(sizeof(okey) * (size_t)(2 * Q + 1));
    if (!buf || !keys) { free(buf); free(keys); return -1; }
    int64_t off = 0;
    for (int64_t q = 0; q < Q; ++q) {
        int64_t m = query_len(lens, fixed_len, q);
        decode_query(words, stride, q, m, buf + off);
        okey a = {buf + off, m, 0, q}, b = {buf + off, m, 1, q};
        keys[2 * q] = a;
        keys[2 * q + 1] = b;
        off += m;
    }
    int64_t K = 2 * Q;
    qsort(keys, (size_t)K, sizeof(okey), key_cmp);
    uint64_t *hist = (uint64_t *)calloc((size_t)K + 1, sizeof(uint64_t));
    int err = hist ? 0 : 1;
    if (!err) {
#pragma omp parallel
        {
            uint64_t *h = (uint64_t *)calloc((size_t)K + 1, sizeof(uint64_t));
            if (!h) {
#pragma omp atomic write
                err = 1;
            }
#pragma omp for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                if (!h) continue;
                int64_t a = 0, b = K; /* first key > S_i */
                while (a < b) {
                    int64_t mid = (a + b) >> 1;
                    if (suffix_vs_key(S, n, i, &keys[mid]) < 0) b = mid; else a = mid + 1;
                }
                h[a]++;
            }
            if (h) {
#pragma omp critical
                for (int64_t j = 0; j <= K; ++j) hist[j] += h[j];
                free(h);
            }
        }
    }
    if (!err) {
        uint64_t run = 0; /* #{i : c(i) <= j} = #{i : S_i < K_j} */
        for (int64_t j = 0; j < K; ++j) {
            run += hist[j];
            lohi[2 * keys[j].q + (keys[j].plus ? 1 : 0)] = run;
        }
    }
    free(hist);
    free(keys);
    free(buf);
    return err ? -1 : 0;
}

/* ---- checks that hold at any size -------------------------------------- */

/* A suffix array is exactly a permutation of [0,n) whose adjacent entries are
 * strictly increasing suffixes ("lexicographically ordered").  Returns
 * -1 if sa is the suffix array of S; otherwise an index r (the first bad
 * adjacent pair found, or the first repeated / out-of-range entry). */
int64_t oracle_check_sa(const uint8_t *S, int64_t n, const uint32_t *sa, int nthreads) {
    set_threads(nthreads);
    uint8_t *seen = (uint8_t *)calloc((size_t)(n / 8 + 1), 1);
    if (!seen) return -2;
    for (int64_t r = 0; r < n; ++r) {
        uint32_t v = sa[r];
        if ((int64_t)v >= n || (seen[v >> 3] >> (v & 7)) & 1) { free(seen); return r; }
        seen[v >> 3] |= (uint8_t)(1u << (v & 7));
    }
    free(seen);
    int64_t bad = n; /* min over threads */
#pragma omp parallel for schedule(dynamic, 65536) reduction(min : bad)
    for (int64_t r = 0; r < n - 1; ++r) {
        if (suffix_cmp(S, n, sa[r], sa[r + 1]) >= 0 && r < bad) bad = r;
    }
    return bad == n ? -1 : bad;
}

/* Certificate for one interval, given a verified suffix array:
 *   0 <= lo <= hi <= n
 *   lo < hi  =>  P is a prefix of S_SA[lo] and of S_SA[hi-1]
 *   lo > 0   =>  t_SA[lo-1] < P
 *   hi < n   =>  t_SA[hi]   > P
 * Because t_SA[r] is non-decreasing in r, these fix lo and hi uniquely.
 * Returns the number of failing queries; *first_bad = first failing q or -1. */
int64_t oracle_certificate(const uint8_t *S, int64_t n, const uint32_t *sa, const uint64_t *words, uint32_t stride,
                           const uint32_t *lens, uint32_t fixed_len, int64_t Q, const uint32_t *lohi,
                           int64_t *first_bad, int nthreads) {
    set_threads(nthreads);
    int64_t mmax = 0;
    for (int64_t q = 0; q < Q; ++q) { int64_t m = query_len(lens, fixed_len, q); if (m > mmax) mmax = m; }
    int64_t nbad = 0, fb = Q;
#pragma omp parallel reduction(+ : nbad) reduction(min : fb)
    {
        uint8_t *P = (uint8_t *)malloc((size_t)mmax + 1);
#pragma omp for schedule(static)
        for (int64_t q = 0; q < Q; ++q) {
            int64_t m = query_len(lens, fixed_len, q);
            decode_query(words, stride, q, m, P);
            int64_t lo = lohi[2 * q], hi = lohi[2 * q + 1];
            int ok = 0 <= lo && lo <= hi && hi <= n;
            if (ok && lo < hi) ok = oracle_cmp(S, n, sa[lo], P, m) == 0 && oracle_cmp(S, n, sa[hi - 1], P, m) == 0;
            if (ok && lo > 0) ok = oracle_cmp(S, n, sa[lo - 1], P, m) > 0;
            if (ok && hi < n) ok = oracle_cmp(S, n, sa[hi], P, m) < 0;
            if (!ok) { nbad++; if (q < fb) fb = q; }
        }
        free(P);
    }
    if (first_bad) *first_bad = nbad ? fb : -1;
    return nbad;
}

/* ---- k-mer table (auxiliary structure of the B200 design) ------ */

/* T[x] = #{ i : trunc_k(S_i) < x } for x in [0, 4^k], x read as the k-mer
 * whose base-4 digits are x (most significant first), T[4^k] = n.  Computed as
 * the histogram of the k-mers of the suffixes of length >= k, prefix-summed,
 * plus, for each of the k-1 shorter suffixes u, the number of x with u < x
 * decided by a plain string comparison. */
void oracle_kmer_table(const uint8_t *S, int64_t n, int k, uint32_t *T) {
    uint64_t K = 1ull << (2 * k);
    uint64_t *hist = (uint64_t *)calloc((size_t)K, sizeof(uint64_t));
    for (int64_t i = 0; i + k <= n; ++i) {
        uint64_t x = 0;
        for (int j = 0; j < k; ++j) x = (x << 2) | S[i + j];
        hist[x]++;
    }
    uint64_t run = 0;
    for (uint64_t x = 0; x < K; ++x) { T[x] = (uint32_t)run; run += hist[x]; }
    T[K] = (uint32_t)n;
    free(hist);
    /* shorter suffixes u = S[i..n), n-i < k */
    uint8_t xs[32];
    for (int64_t i = n - k + 1 < 0 ? 0 : n - k + 1; i < n; ++i) {
        int64_t l = n - i;
        for (uint64_t x = 0; x < K; ++x) {
            for (int j = 0; j < k; ++j) xs[j] = (uint8_t)((x >> (2 * (k - 1 - j))) & 3u);
            /* u < x ? (u shorter than x: proper prefix sorts first) */
            int c = memcmp(S + i, xs, (size_t)l);
            if (c <= 0) T[x]++; /* c == 0: u is a proper prefix of x */
        }
    }
}
