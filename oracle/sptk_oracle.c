/*
 * sptk_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64, single-threaded-per-call restatement of the reference
 * `sptucker` hot path (/root/reference/pkg/src/sptucker).  It is the checker
 * for the CUDA library and the CPU baseline timed by bench.py
 * (`cpu_baseline.kind = "port"`).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * path (paper_2204_07104_b200) never does.
 *
 * Pinning: every function below is checked against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py imports the reference and
 * numpy 2.3.5, whose Generator algorithms the reference relies on).
 *
 * Sections and the reference lines they restate:
 *   SeedSequence + PCG64 seeding ... numpy bit_generator.pyx (SeedSequence),
 *       _pcg64.pyx / pcg64.h (XSL-RR 128/64); used by trainer.py:196-198,
 *       trainer.py:214, model.py:97, coo.py:281.
 *   random_interval / Lemire32 ..... numpy distributions.c (random_interval,
 *       buffered_bounded_lemire_uint32, random_bounded_uint64).
 *   permutation .................... Generator.permutation -> shuffle ->
 *       _shuffle_raw (Fisher-Yates, i = n-1..1); trainer.py:196-199.
 *   choice(replace=False) .......... Generator.choice: tail shuffle
 *       (_shuffle_int) when pop > 10000 and k > pop // 50, else Floyd +
 *       _shuffle_int(k, 1); trainer.py:212-221, coo.py:281.
 *   partition ...................... partition.py:47-81 (stable bucketing).
 *   factor_pass .................... _loops.py:17-63.
 *   core_pass ...................... _loops.py:66-104.
 *   predict ........................ model.py:134-146.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* SeedSequence (numpy.random.bit_generator.SeedSequence, pool_size=4) */
/* ------------------------------------------------------------------ */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* entropy: non-negative integers (< 2^64), each expanded to little-endian
 * 32-bit words the way _coerce_to_uint32_array does (0 -> one zero word). */
void orc_seedseq_generate(const uint64_t *entropy, int n_entropy, uint32_t *out, int n_out) {
    uint32_t words[256];
    int nw = 0;
    for (int e = 0; e < n_entropy && nw < 250; ++e) {
        uint64_t x = entropy[e];
        if (x == 0) {
            words[nw++] = 0;
        } else {
            while (x) {
                words[nw++] = (uint32_t)(x & 0xffffffffu);
                x >>= 32;
            }
        }
    }
    uint32_t pool[4];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < nw ? words[i] : 0u, &hc);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = 4; s < nw; ++s)
        for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &hc));
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < n_out; ++i) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        out[i] = v;
    }
}

/* ------------------------------------------------------------------ */
/* PCG64 (XSL-RR 128/64), numpy's buffered 32-bit draws                */
/* ------------------------------------------------------------------ */
typedef struct {
    u128 state, inc;
    int has32;
    uint32_t u32;
} orc_pcg64;

#define PCG_MULT ((((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL)

static inline void pcg_step(orc_pcg64 *r) { r->state = r->state * PCG_MULT + r->inc; }

static inline uint64_t pcg_output(u128 s) {
    uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static inline uint64_t pcg_next64(orc_pcg64 *r) {
    pcg_step(r);
    return pcg_output(r->state);
}

static inline uint32_t pcg_next32(orc_pcg64 *r) {
    if (r->has32) {
        r->has32 = 0;
        return r->u32;
    }
    uint64_t v = pcg_next64(r);
    r->has32 = 1;
    r->u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

/* default_rng(entropy) -> PCG64 state (pcg64_set_seed + srandom_r). */
void orc_pcg64_from_entropy(const uint64_t *entropy, int n_entropy, uint64_t out[4]) {
    uint32_t w[8];
    orc_seedseq_generate(entropy, n_entropy, w, 8);
    uint64_t v[4];
    for (int k = 0; k < 4; ++k) v[k] = (uint64_t)w[2 * k] | ((uint64_t)w[2 * k + 1] << 32);
    u128 initstate = ((u128)v[0] << 64) | v[1];
    u128 initseq = ((u128)v[2] << 64) | v[3];
    orc_pcg64 r;
    r.state = 0;
    r.inc = (initseq << 1) | 1u;
    pcg_step(&r);
    r.state += initstate;
    pcg_step(&r);
    out[0] = (uint64_t)(r.state >> 64);
    out[1] = (uint64_t)r.state;
    out[2] = (uint64_t)(r.inc >> 64);
    out[3] = (uint64_t)r.inc;
}

static void pcg_load(orc_pcg64 *r, const uint64_t s[4]) {
    r->state = ((u128)s[0] << 64) | s[1];
    r->inc = ((u128)s[2] << 64) | s[3];
    r->has32 = 0;
    r->u32 = 0;
}

/* Raw u32 draws, for checking the device generator's stream. */
void orc_pcg64_u32_stream(const uint64_t s[4], int64_t n, uint32_t *out) {
    orc_pcg64 r;
    pcg_load(&r, s);
    for (int64_t i = 0; i < n; ++i) out[i] = pcg_next32(&r);
}

/* distributions.c: random_interval (masked rejection, 32-bit path). */
static inline uint64_t random_interval(orc_pcg64 *r, uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t value;
    if (max <= 0xffffffffULL) {
        while ((value = (pcg_next32(r) & mask)) > max) {
        }
    } else {
        while ((value = (pcg_next64(r) & mask)) > max) {
        }
    }
    return value;
}

/* distributions.c: buffered_bounded_lemire_uint32 (rng < 0xffffffff). */
static inline uint32_t lemire32(orc_pcg64 *r, uint32_t rng) {
    const uint32_t rng_excl = rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(r) * rng_excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < rng_excl) {
        const uint32_t threshold = (0xffffffffu - rng) % rng_excl;
        while (leftover < threshold) {
            m = (uint64_t)pcg_next32(r) * rng_excl;
            leftover = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

/* distributions.c: random_bounded_uint64(off=0, rng, mask=0, masked=0),
 * restricted to rng < 2^32 (all populations on this path are < 2^31). */
static inline uint64_t bounded_u64(orc_pcg64 *r, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xffffffffULL) return pcg_next32(r);
    return lemire32(r, (uint32_t)rng);
}

/* Generator.permutation(n) == shuffle(arange(n)) via _shuffle_raw.
 * Also returns the Fisher-Yates j sequence (j_seq[i] for i=1..n-1; j_seq[0]=0)
 * when j_seq != NULL, for checking the device generator in isolation. */
void orc_permutation(const uint64_t s[4], int64_t n, int64_t *out, int64_t *j_seq) {
    orc_pcg64 r;
    pcg_load(&r, s);
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    if (j_seq && n > 0) j_seq[0] = 0;
    for (int64_t i = n - 1; i >= 1; --i) {
        int64_t j = (int64_t)random_interval(&r, (uint64_t)i);
        if (j_seq) j_seq[i] = j;
        int64_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

/* Generator._shuffle_int(n, first, data). */
static void shuffle_int(orc_pcg64 *r, int64_t n, int64_t first, int64_t *data) {
    for (int64_t i = n - 1; i >= first; --i) {
        int64_t j = (int64_t)bounded_u64(r, (uint64_t)i);
        int64_t t = data[j];
        data[j] = data[i];
        data[i] = t;
    }
}

/* Generator.choice(pop, size=k, replace=False) with shuffle=True.
 * returns 0 (arange path: caller's responsibility), 1 tail, 2 floyd. */
int orc_choice(const uint64_t s[4], int64_t pop, int64_t k, int64_t *out) {
    orc_pcg64 r;
    pcg_load(&r, s);
    if (pop > 10000 && k > pop / 50) {
        int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)pop);
        for (int64_t i = 0; i < pop; ++i) idx[i] = i;
        int64_t first = pop - k > 1 ? pop - k : 1;
        shuffle_int(&r, pop, first, idx);
        memcpy(out, idx + (pop - k), sizeof(int64_t) * (size_t)k);
        free(idx);
        return 1;
    }
    /* Floyd: membership via a bitmap over [0, pop). */
    uint8_t *seen = (uint8_t *)calloc((size_t)(pop / 8 + 1), 1);
    for (int64_t j = pop - k; j < pop; ++j) {
        int64_t val = (int64_t)bounded_u64(&r, (uint64_t)j);
        if (!(seen[val >> 3] & (1u << (val & 7)))) {
            seen[val >> 3] |= (uint8_t)(1u << (val & 7));
            out[j - pop + k] = val;
        } else {
            seen[j >> 3] |= (uint8_t)(1u << (j & 7));
            out[j - pop + k] = j;
        }
    }
    free(seen);
    shuffle_int(&r, k, 1, out);
    return 2;
}

/* ------------------------------------------------------------------ */
/* partition.py:47-81: cuts k*d//m, bucket = searchsorted(right)-1,    */
/* key = sum bucket_n * m^(N-1-n), stable argsort by key.              */
/* out_ids[nnz] = entry ids grouped by key (ascending key, source      */
/* order inside), out_keys[nnz] = key of each out_ids entry.           */
/* ------------------------------------------------------------------ */
int orc_partition(const int64_t *idx, int64_t nnz, int order, const int64_t *dims, int64_t m,
                  int64_t *out_ids, int64_t *out_keys) {
    int64_t nkeys = 1;
    for (int n = 0; n < order; ++n) nkeys *= m;
    int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    for (int64_t e = 0; e < nnz; ++e) {
        int64_t k = 0;
        for (int n = 0; n < order; ++n) {
            int64_t i = idx[e * order + n];
            /* largest b with b*d//m <= i */
            int64_t b = 0;
            int64_t lo = 0, hi = m; /* cuts[hi] = d > i always */
            while (hi - lo > 1) {
                int64_t mid = (lo + hi) / 2;
                if ((mid * dims[n]) / m <= i) lo = mid; else hi = mid;
            }
            b = lo;
            k = k * m + b;
        }
        key[e] = k;
    }
    int64_t *cnt = (int64_t *)calloc((size_t)nkeys + 1, sizeof(int64_t));
    for (int64_t e = 0; e < nnz; ++e) cnt[key[e] + 1]++;
    for (int64_t b = 0; b < nkeys; ++b) cnt[b + 1] += cnt[b];
    for (int64_t e = 0; e < nnz; ++e) {
        int64_t p = cnt[key[e]]++;
        out_ids[p] = e;
        out_keys[p] = key[e];
    }
    free(cnt);
    free(key);
    return 0;
}

/* ------------------------------------------------------------------ */
/* _loops.py:17-63 factor_pass, fp64, identical operation order.       */
/* ------------------------------------------------------------------ */
int orc_factor_pass(const int64_t *idx, const double *vals, const int64_t *visit, int64_t n_visit,
                    double *fac, const int64_t *foff, const double *cor, const int64_t *coff,
                    const int64_t *jr, int n_modes, int64_t rcore, const double *gammas,
                    const double *lambdas) {
    int64_t jmax = 0;
    for (int n = 0; n < n_modes; ++n)
        if (jr[n] > jmax) jmax = jr[n];
    double *c = (double *)malloc(sizeof(double) * (size_t)(n_modes * rcore));
    double *gs = (double *)malloc(sizeof(double) * (size_t)jmax);
    for (int64_t v = 0; v < n_visit; ++v) {
        int64_t s = visit[v];
        double x = vals[s];
        for (int n = 0; n < n_modes; ++n) {
            for (int n0 = 0; n0 < n_modes; ++n0) {
                int64_t jn0 = jr[n0];
                int64_t abase = foff[n0] + idx[s * n_modes + n0] * jn0;
                int64_t bbase = coff[n0];
                for (int64_t r = 0; r < rcore; ++r) {
                    double acc = 0.0;
                    for (int64_t j = 0; j < jn0; ++j) acc += fac[abase + j] * cor[bbase + j * rcore + r];
                    c[n0 * rcore + r] = acc;
                }
            }
            int64_t jn = jr[n];
            for (int64_t j = 0; j < jn; ++j) gs[j] = 0.0;
            int64_t bbase = coff[n];
            for (int64_t r = 0; r < rcore; ++r) {
                double w = 1.0;
                for (int n0 = 0; n0 < n_modes; ++n0)
                    if (n0 != n) w *= c[n0 * rcore + r];
                for (int64_t j = 0; j < jn; ++j) gs[j] += w * cor[bbase + j * rcore + r];
            }
            int64_t abase = foff[n] + idx[s * n_modes + n] * jn;
            double inter = 0.0;
            for (int64_t j = 0; j < jn; ++j) inter += fac[abase + j] * gs[j];
            double gamma = gammas[n], lam = lambdas[n];
            for (int64_t j = 0; j < jn; ++j) {
                double g = -x * gs[j] + lam * fac[abase + j] + inter * gs[j];
                fac[abase + j] -= gamma * g;
            }
        }
    }
    free(gs);
    free(c);
    return 0;
}

/* ------------------------------------------------------------------ */
/* _loops.py:66-104 core_pass, fp64, identical operation order.        */
/* ------------------------------------------------------------------ */
int orc_core_pass(const int64_t *idx, const double *vals, const int64_t *visit, int64_t n_visit,
                  const double *fac, const int64_t *foff, const double *cor, const int64_t *coff,
                  const int64_t *jr, int n_modes, int64_t rcore, double *acc, const int64_t *aoff) {
    double *c = (double *)malloc(sizeof(double) * (size_t)(n_modes * rcore));
    for (int64_t v = 0; v < n_visit; ++v) {
        int64_t s = visit[v];
        double x = vals[s];
        for (int n0 = 0; n0 < n_modes; ++n0) {
            int64_t jn0 = jr[n0];
            int64_t abase = foff[n0] + idx[s * n_modes + n0] * jn0;
            int64_t bbase = coff[n0];
            for (int64_t r = 0; r < rcore; ++r) {
                double dot = 0.0;
                for (int64_t j = 0; j < jn0; ++j) dot += fac[abase + j] * cor[bbase + j * rcore + r];
                c[n0 * rcore + r] = dot;
            }
        }
        double xhat = 0.0;
        for (int64_t r = 0; r < rcore; ++r) {
            double p = 1.0;
            for (int n0 = 0; n0 < n_modes; ++n0) p *= c[n0 * rcore + r];
            xhat += p;
        }
        double resid = xhat - x;
        for (int n = 0; n < n_modes; ++n) {
            int64_t jn = jr[n];
            int64_t abase = foff[n] + idx[s * n_modes + n] * jn;
            int64_t base = aoff[n];
            for (int64_t r = 0; r < rcore; ++r) {
                double w = 1.0;
                for (int n0 = 0; n0 < n_modes; ++n0)
                    if (n0 != n) w *= c[n0 * rcore + r];
                double coef = resid * w;
                for (int64_t j = 0; j < jn; ++j) acc[base + j * rcore + r] += coef * fac[abase + j];
            }
        }
    }
    free(c);
    return 0;
}

/* ------------------------------------------------------------------ */
/* model.py:134-146 predict_entries (row-wise; numpy evaluates         */
/* prod *= A[idx] @ B then sums over r).                               */
/* ------------------------------------------------------------------ */
int orc_predict(const int64_t *idx, int64_t m, const double *fac, const int64_t *foff,
                const double *cor, const int64_t *coff, const int64_t *jr, int n_modes,
                int64_t rcore, double *out) {
    double *prod = (double *)malloc(sizeof(double) * (size_t)rcore);
    for (int64_t e = 0; e < m; ++e) {
        for (int64_t r = 0; r < rcore; ++r) prod[r] = 1.0;
        for (int n = 0; n < n_modes; ++n) {
            int64_t jn = jr[n];
            int64_t abase = foff[n] + idx[e * n_modes + n] * jn;
            for (int64_t r = 0; r < rcore; ++r) {
                double d = 0.0;
                for (int64_t j = 0; j < jn; ++j) d += fac[abase + j] * cor[coff[n] + j * rcore + r];
                prod[r] *= d;
            }
        }
        double sum = 0.0;
        for (int64_t r = 0; r < rcore; ++r) sum += prod[r];
        out[e] = sum;
    }
    free(prod);
    return 0;
}
