/*
 * synth.c -- seeded synthetic inputs (reference genomes and reads).
 *
 * This module is shared by BOTH sides of the parity check (the CPU oracle in
 * oracle/ and the CUDA path in paper_1303_3692_b200/) and therefore holds none
 * of the method's arithmetic: no suffix order, no comparison, no search.  It
 * only produces bytes.  The recipes are stated in DESIGN.md ("Input recipe");
 * they stand in for the paper's NCBI data (Sec. V: the first
 * 10^7 nt of NT_167186.1 plus 1024-nt queries mixing a hit contig with a miss
 * contig), which is out of scope.
 *
 * Randomness is counter based: every background block, repeat element and read
 * draws from its own SplitMix64 stream keyed by (seed, kind, id).  Output is
 * therefore identical for any thread count, and a rank can generate only its
 * shard [q_begin, q_begin+q_count) of the reads.
 *
 * Alphabet: upper-case 'A','C','G','T' (Sec. III: Sigma={a,c,g,t}).
 * Reads are written 2 bits per base, MSB-first, in uint64 words with a fixed
 * stride (the query layout of include/sa.h): base j of read q sits in word
 * q*stride + j/32 at bits [63-2(j%32), 62-2(j%32)], codes A=0 C=1 G=2 T=3,
 * bits past the read's length are zero.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SYNTH_VERSION 1

/* ---- counter-based SplitMix64 streams ---------------------------------- */
typedef struct { uint64_t s; } rng_t;

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline rng_t rng_stream(uint64_t seed, uint64_t kind, uint64_t id) {
    rng_t r;
    r.s = mix64(mix64(seed + 0x9E3779B97F4A7C15ull * (kind + 1)) ^ (id * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull));
    return r;
}
static inline uint64_t rng_next(rng_t *r) { r->s += 0x9E3779B97F4A7C15ull; return mix64(r->s); }
static inline double rng_unif(rng_t *r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static inline uint64_t rng_below(rng_t *r, uint64_t b) {
    return (uint64_t)(((unsigned __int128)rng_next(r) * b) >> 64);
}
static inline uint64_t rng_range(rng_t *r, uint64_t lo, uint64_t hi) { /* inclusive */
    return lo + rng_below(r, hi - lo + 1);
}

static const char BASES[4] = {'A', 'C', 'G', 'T'};

/* iid base with GC content gc (P(C)=P(G)=gc/2, P(A)=P(T)=(1-gc)/2). */
static inline char base_gc(rng_t *r, double gc) {
    double u = rng_unif(r);
    if (u < gc) return (u < 0.5 * gc) ? 'C' : 'G';
    return (u - gc < 0.5 * (1.0 - gc)) ? 'A' : 'T';
}
static inline int code_of(char c) {
    switch (c) { case 'A': return 0; case 'C': return 1; case 'G': return 2; default: return 3; }
}
/* substitute with one of the other three bases */
static inline char substitute(rng_t *r, char c) {
    int k = code_of(c);
    int d = 1 + (int)rng_below(r, 3);
    return BASES[(k + d) & 3];
}

/* stream kinds */
enum { K_BG = 1, K_PLAN, K_SEG, K_ALUFAM, K_L1FAM, K_SDFAM, K_READ, K_ELEM };

enum { SYNTH_REF_UNIFORM = 0, SYNTH_REF_BACTERIAL = 1, SYNTH_REF_REPEAT = 2, SYNTH_REF_REPEAT_DUP = 3 };

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

/* ---- iid background ----------------------------------------------------- */
#define BG_BLOCK (1u << 20)
static void fill_background(char *out, uint64_t n, uint64_t seed, double gc) {
    int64_t nb = (int64_t)((n + BG_BLOCK - 1) / BG_BLOCK);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nb; ++b) {
        rng_t r = rng_stream(seed, K_BG, (uint64_t)b);
        uint64_t lo = (uint64_t)b * BG_BLOCK, hi = lo + BG_BLOCK;
        if (hi > n) hi = n;
        for (uint64_t i = lo; i < hi; ++i) out[i] = base_gc(&r, gc);
    }
}

/* ---- E. coli-like (config C2) ------------------------------------------ */
/* 5 Mbp iid at GC 50.8 %, plus 7 copies of one 5 kb "rRNA operon" at 99.9 %
 * identity and 10 copies of one 1.3 kb "IS element" at 99.5 % identity, placed
 * at sorted uniform offsets without overlap. */
static void gen_bacterial(char *out, uint64_t n, uint64_t seed) {
    fill_background(out, n, seed, 0.508);
    enum { NEL = 17 };
    uint32_t len[NEL], fam[NEL];
    double div[NEL];
    for (int j = 0; j < NEL; ++j) {
        fam[j] = j < 7 ? 0 : 1;
        len[j] = j < 7 ? 5000 : 1300;
        div[j] = j < 7 ? 0.001 : 0.005;
    }
    uint64_t total = 7ull * 5000 + 10ull * 1300;
    if (n < 2 * total) return; /* tiny test references: background only */
    rng_t pr = rng_stream(seed, K_PLAN, 0);
    /* seeded shuffle of element order, then sorted offsets in [0, n-total] */
    for (int j = NEL - 1; j > 0; --j) {
        int t = (int)rng_below(&pr, (uint64_t)j + 1);
        uint32_t a = len[j]; len[j] = len[t]; len[t] = a;
        a = fam[j]; fam[j] = fam[t]; fam[t] = a;
        double d = div[j]; div[j] = div[t]; div[t] = d;
    }
    uint64_t off[NEL];
    for (int j = 0; j < NEL; ++j) off[j] = rng_below(&pr, n - total + 1);
    for (int a = 1; a < NEL; ++a) /* insertion sort */
        for (int b = a; b > 0 && off[b - 1] > off[b]; --b) { uint64_t t = off[b]; off[b] = off[b - 1]; off[b - 1] = t; }
    uint64_t shift = 0;
    char *src = (char *)malloc(5000);
    for (int j = 0; j < NEL; ++j) {
        rng_t fr = rng_stream(seed, K_SDFAM, fam[j]);
        for (uint32_t i = 0; i < len[j]; ++i) src[i] = base_gc(&fr, 0.508);
        rng_t er = rng_stream(seed, K_ELEM, (uint64_t)j);
        uint64_t p = off[j] + shift;
        for (uint32_t i = 0; i < len[j]; ++i)
            out[p + i] = rng_unif(&er) < div[j] ? substitute(&er, src[i]) : src[i];
        shift += len[j];
    }
    free(src);
}

/* ---- repeat-rich (configs C3, C4, C5) ----------------------------------- */
/* GC 41 % iid background (~65 %) interleaved with
 *   ~10 % Alu-like : 50 families x 300 bp consensus, 2-20 % divergence, poly-A tail 10-30 bp
 *   ~17 % L1-like  : 20 families x 6 kb consensus, 5'-truncated (keep the last 300..6000 bp),
 *                    5-20 % divergence
 *   ~3 %  microsatellites: unit 1-6 bp, run 20-200 bp, exact
 *   ~5 %  segmental duplications: families of 10-100 kb, copies at 99-99.9 % identity
 * Element type per event is drawn with probability proportional to its expected
 * count; background gaps are geometric. */
enum { S_BG = 0, S_ALU, S_L1, S_MICRO, S_SD };
typedef struct {
    uint64_t start;
    uint32_t len;
    uint32_t type;
    uint32_t fam;
    uint32_t p0; /* ALU: tail length; L1: truncation offset; MICRO: unit length */
    float div;
} seg_t;

#define ALU_FAMS 50
#define ALU_LEN 300
#define L1_FAMS 20
#define L1_LEN 6000

static uint32_t sd_family_len(uint64_t seed, uint32_t fam) {
    rng_t r = rng_stream(seed, K_SDFAM, ((uint64_t)fam << 1) | 1);
    return (uint32_t)rng_range(&r, 10000, 100000);
}

static int gen_repeat(char *out, uint64_t n, uint64_t seed) {
    const double gc = 0.41;
    const double f_alu = 0.10, f_l1 = 0.17, f_mi = 0.03, f_sd = 0.05;
    const double mu_alu = ALU_LEN + 20.0, mu_l1 = 0.5 * (300 + L1_LEN), mu_mi = 110.0, mu_sd = 55000.0;
    double c_alu = n * f_alu / mu_alu, c_l1 = n * f_l1 / mu_l1, c_mi = n * f_mi / mu_mi, c_sd = n * f_sd / mu_sd;
    double c_tot = c_alu + c_l1 + c_mi + c_sd;
    double gap_mean = n * (1.0 - f_alu - f_l1 - f_mi - f_sd) / c_tot;
    uint32_t sd_fams = (uint32_t)(c_sd / 2.0 + 0.5);
    if (sd_fams < 1) sd_fams = 1;
    double p_alu = c_alu / c_tot, p_l1 = c_l1 / c_tot, p_mi = c_mi / c_tot;

    /* family consensus sequences */
    char *alu = (char *)malloc((size_t)ALU_FAMS * ALU_LEN);
    char *l1 = (char *)malloc((size_t)L1_FAMS * L1_LEN);
    if (!alu || !l1) { free(alu); free(l1); return -1; }
    for (int f = 0; f < ALU_FAMS; ++f) {
        rng_t r = rng_stream(seed, K_ALUFAM, (uint64_t)f);
        for (int i = 0; i < ALU_LEN; ++i) alu[f * ALU_LEN + i] = base_gc(&r, 0.52);
    }
    for (int f = 0; f < L1_FAMS; ++f) {
        rng_t r = rng_stream(seed, K_L1FAM, (uint64_t)f);
        for (int i = 0; i < L1_LEN; ++i) l1[(size_t)f * L1_LEN + i] = base_gc(&r, 0.42);
    }

    /* sequential plan (cheap: ~1.3 segments per kb) */
    size_t cap = 1024, ns = 0;
    seg_t *seg = (seg_t *)malloc(cap * sizeof(seg_t));
    if (!seg) { free(alu); free(l1); return -1; }
    rng_t pr = rng_stream(seed, K_PLAN, 0);
    uint64_t pos = 0;
    while (pos < n) {
        if (ns + 2 > cap) {
            cap *= 2;
            seg_t *t = (seg_t *)realloc(seg, cap * sizeof(seg_t));
            if (!t) { free(seg); free(alu); free(l1); return -1; }
            seg = t;
        }
        uint64_t g = (uint64_t)floor(-gap_mean * log(1.0 - rng_unif(&pr)));
        if (g > 0) {
            seg_t s = {pos, (uint32_t)(g > 0xFFFFFFFFull ? 0xFFFFFFFFull : g), S_BG, 0, 0, 0.f};
            seg[ns++] = s;
            pos += s.len;
            if (pos >= n) break;
        }
        double u = rng_unif(&pr);
        seg_t s = {pos, 0, 0, 0, 0, 0.f};
        if (u < p_alu) {
            s.type = S_ALU; s.fam = (uint32_t)rng_below(&pr, ALU_FAMS);
            s.p0 = (uint32_t)rng_range(&pr, 10, 30);
            s.len = ALU_LEN + s.p0;
            s.div = (float)(0.02 + 0.18 * rng_unif(&pr));
        } else if (u < p_alu + p_l1) {
            s.type = S_L1; s.fam = (uint32_t)rng_below(&pr, L1_FAMS);
            uint32_t keep = (uint32_t)rng_range(&pr, 300, L1_LEN);
            s.p0 = L1_LEN - keep;
            s.len = keep;
            s.div = (float)(0.05 + 0.15 * rng_unif(&pr));
        } else if (u < p_alu + p_l1 + p_mi) {
            s.type = S_MICRO; s.p0 = (uint32_t)rng_range(&pr, 1, 6);
            s.len = (uint32_t)rng_range(&pr, 20, 200);
        } else {
            s.type = S_SD; s.fam = (uint32_t)rng_below(&pr, sd_fams);
            s.len = sd_family_len(seed, s.fam);
            s.div = (float)(0.001 + 0.009 * rng_unif(&pr)); /* identity 99.0 .. 99.9 % */
        }
        seg[ns++] = s;
        pos += s.len;
    }
    if (ns > 0 && seg[ns - 1].start + seg[ns - 1].len > n) seg[ns - 1].len = (uint32_t)(n - seg[ns - 1].start);

    /* parallel fill: each segment has its own stream */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < (int64_t)ns; ++j) {
        const seg_t s = seg[j];
        rng_t r = rng_stream(seed, K_SEG, (uint64_t)j);
        char *o = out + s.start;
        switch (s.type) {
        case S_BG:
            for (uint32_t i = 0; i < s.len; ++i) o[i] = base_gc(&r, gc);
            break;
        case S_ALU: {
            const char *c = alu + (size_t)s.fam * ALU_LEN;
            for (uint32_t i = 0; i < s.len; ++i) {
                char b = i < ALU_LEN ? c[i] : 'A';
                o[i] = rng_unif(&r) < s.div ? substitute(&r, b) : b;
            }
        } break;
        case S_L1: {
            const char *c = l1 + (size_t)s.fam * L1_LEN + s.p0;
            for (uint32_t i = 0; i < s.len; ++i) o[i] = rng_unif(&r) < s.div ? substitute(&r, c[i]) : c[i];
        } break;
        case S_MICRO: {
            char unit[6];
            for (uint32_t i = 0; i < s.p0; ++i) unit[i] = BASES[rng_below(&r, 4)];
            for (uint32_t i = 0; i < s.len; ++i) o[i] = unit[i % s.p0];
        } break;
        default: { /* S_SD: regenerate the family source from its own stream */
            rng_t fr = rng_stream(seed, K_SDFAM, (uint64_t)s.fam << 1);
            for (uint32_t i = 0; i < s.len; ++i) {
                char b = base_gc(&fr, gc);
                o[i] = rng_unif(&r) < s.div ? substitute(&r, b) : b;
            }
        } break;
        }
    }
    free(seg);
    free(alu);
    free(l1);
    return 0;
}

/* ---- public entry points ------------------------------------------------ */

int synth_version(void) { return SYNTH_VERSION; }

/* Writes n upper-case ACGT bytes to out.  kind: 0 uniform iid (C1), 1
 * E. coli-like (C2), 2 repeat-rich (C4/C5), 3 repeat-rich + one exact 100 kb
 * duplication (C3).  Returns 0, or -1 on bad
 * arguments / allocation failure. */
int synth_reference(int kind, uint64_t n, uint64_t seed, char *out, int nthreads) {
    if (!out) return -1;
    set_threads(nthreads);
    switch (kind) {
    case SYNTH_REF_UNIFORM: fill_background(out, n, seed, 0.5); return 0;
    case SYNTH_REF_BACTERIAL: gen_bacterial(out, n, seed); return 0;
    case SYNTH_REF_REPEAT: return gen_repeat(out, n, seed);
    case SYNTH_REF_REPEAT_DUP: {
        /* the repeat-rich recipe plus ONE exact (100 % identity) 100 kb segmental duplication: bases
         * [n/4, n/4 + 100000) copied to [5n/8, 5n/8 + 100000) -- the deepest tie the suffix sort meets
         * (segmental duplications at 99-100 % identity; reading B3) */
        if (gen_repeat(out, n, seed) != 0) return -1;
        const uint64_t L = 100000;
        if (n >= 4 * L) memmove(out + 5 * (n / 8), out + n / 4, L);
        return 0;
    }
    default: return -1;
    }
}

/* Reads q_begin .. q_begin+q_count-1 of a seeded read set over ref[0..n).
 * Read q: length m ~ U[m_min, m_max]; with probability p_random it is iid
 * uniform ACGT (the "miss contig"), otherwise an exact copy of ref[s..s+m) at
 * a uniform start s in [0, n-m] (a random read if n < m); an exact read is
 * given one substitution at a uniform position with probability p_mut_read.
 * Writes packed words (stride words per read, zero beyond the read) and, if
 * lens != NULL, the length of each read.  Returns 0 or -1. */
/* stride == 0 selects the dense layout (fixed length m_min == m_max == m only): read i occupies
 * bases [i*m, (i+1)*m) of one continuous 2-bit stream; q_count must be a multiple of 32 so that
 * every group of 32 reads covers exactly m whole words (groups are written by one thread). */
int synth_reads(const char *ref, uint64_t n, uint64_t q_begin, uint64_t q_count, uint32_t m_min,
                uint32_t m_max, double p_random, double p_mut_read, uint64_t seed, uint64_t *words,
                uint32_t stride, uint32_t *lens, int nthreads) {
    const int dense = stride == 0;
    if (!words || m_min > m_max || (!dense && (uint64_t)stride * 32 < m_max)) return -1;
    if (dense && (m_min != m_max || (q_count & 31) != 0)) return -1;
    if (n > 0 && !ref) return -1;
    set_threads(nthreads);
    if (dense) memset(words, 0, (size_t)(q_count / 32 * m_max) * sizeof(uint64_t));
#pragma omp parallel
    {
        char *buf = (char *)malloc(m_max + 1);
#pragma omp for schedule(static, 32)
        for (int64_t i = 0; i < (int64_t)q_count; ++i) {
            uint64_t q = q_begin + (uint64_t)i;
            rng_t r = rng_stream(seed, K_READ, q);
            uint32_t m = (uint32_t)rng_range(&r, m_min, m_max);
            int is_random = rng_unif(&r) < p_random || n < (uint64_t)m || n == 0;
            if (is_random) {
                for (uint32_t j = 0; j < m; ++j) buf[j] = BASES[rng_below(&r, 4)];
            } else {
                uint64_t s = rng_below(&r, n - m + 1);
                memcpy(buf, ref + s, m);
                for (uint32_t j = 0; j < m; ++j) { /* accept lower case references too */
                    char c = buf[j];
                    buf[j] = (char)(c >= 'a' ? c - 32 : c);
                }
                if (m > 0 && rng_unif(&r) < p_mut_read) {
                    uint32_t j = (uint32_t)rng_below(&r, m);
                    buf[j] = substitute(&r, buf[j]);
                }
            }
            if (dense) {
                const uint64_t b0 = (uint64_t)i * m;  /* base offset of this read in the stream */
                for (uint32_t j = 0; j < m; ++j) {
                    const uint64_t b = b0 + j;
                    words[b >> 5] |= (uint64_t)code_of(buf[j]) << (62 - 2 * (b & 31));
                }
            } else {
                uint64_t *w = words + (uint64_t)i * stride;
                for (uint32_t t = 0; t < stride; ++t) w[t] = 0;
                for (uint32_t j = 0; j < m; ++j)
                    w[j >> 5] |= (uint64_t)code_of(buf[j]) << (62 - 2 * (j & 31));
            }
            if (lens) lens[i] = m;
        }
        free(buf);
    }
    return 0;
}
