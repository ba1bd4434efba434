/* Seeded synthetic inputs, host C implementation (threaded).
 *
 * Holds none of the method's arithmetic: it assembles binary64 bit patterns from
 * a counter-based splitmix64 generator. Same definition as synth/gen.py (numpy)
 * and synth/csrc/gen.cu (device); see synth/gen.py for the definition and
 * SURVEY.md §8(d). Used to stream the 64 GiB config c4 to the oracle without a
 * host buffer of that size.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#define G 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t key_of(uint64_t seed, uint64_t st) { return mix64(seed + G * (st + 1)); }

static inline uint64_t draw_bits(uint64_t key, uint64_t i, int lo, int hi) {
    uint64_t u = mix64(key + G * (2 * i + 1));
    uint64_t v = mix64(key + G * (2 * i + 2));
    uint64_t span = (uint64_t)(hi - lo + 1);
    uint64_t e = ((v >> 32) * span) >> 32;
    uint64_t biased = (uint64_t)((int64_t)e + lo + 1023);
    return (u & 0x8000000000000000ull) | (biased << 52) | (u & ((1ull << 52) - 1));
}

typedef struct {
    uint64_t *out;
    uint64_t start, count;
    uint64_t seed, st;
    int lo, hi;
    /* cancel family */
    int kind;
    uint64_t npairs;
    int plo, phi, tlo, thi;
} job_t;

static void *run_job(void *arg) {
    job_t *j = (job_t *)arg;
    if (j->kind == 0) {
        uint64_t k = key_of(j->seed, j->st);
        for (uint64_t t = 0; t < j->count; ++t) j->out[t] = draw_bits(k, j->start + t, j->lo, j->hi);
    } else if (j->kind == 1) {
        uint64_t ka = key_of(j->seed, 0), kt = key_of(j->seed, 1);
        uint64_t n2 = 2 * j->npairs;
        for (uint64_t t = 0; t < j->count; ++t) {
            uint64_t p = j->start + t;
            if (p < n2) j->out[t] = draw_bits(ka, p >> 1, j->plo, j->phi) ^ ((p & 1) << 63);
            else        j->out[t] = draw_bits(kt, p - n2, j->tlo, j->thi);
        }
    } else { /* kind 2: raw U(seed, st, idx) keys */
        uint64_t k = key_of(j->seed, j->st);
        for (uint64_t t = 0; t < j->count; ++t) j->out[t] = mix64(k + G * (j->start + t + 1));
    }
    return NULL;
}

static void run_threads(job_t proto, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > proto.count / 4096 + 1) nthreads = (int)(proto.count / 4096 + 1);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
    uint64_t per = proto.count / nthreads, rem = proto.count % nthreads, off = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].start = proto.start + off;
        jobs[t].out = proto.out + off;
        jobs[t].count = per + ((uint64_t)t < rem ? 1 : 0);
        off += jobs[t].count;
        pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th); free(jobs);
}

/* out[t] = bits of draw(seed, st, start+t, lo, hi), t < count */
void synth_uniform(uint64_t *out, uint64_t start, uint64_t count, uint64_t seed, uint64_t st,
                   int lo, int hi, int nthreads) {
    job_t j = {0};
    j.out = out; j.start = start; j.count = count; j.seed = seed; j.st = st; j.lo = lo; j.hi = hi;
    j.kind = 0;
    run_threads(j, nthreads);
}

/* c3 before permutation: [a_0,-a_0,a_1,-a_1,...,t_0..], positions [start, start+count) */
void synth_cancel_unpermuted(uint64_t *out, uint64_t start, uint64_t count, uint64_t seed,
                             uint64_t npairs, int plo, int phi, int tlo, int thi, int nthreads) {
    job_t j = {0};
    j.out = out; j.start = start; j.count = count; j.seed = seed;
    j.kind = 1; j.npairs = npairs; j.plo = plo; j.phi = phi; j.tlo = tlo; j.thi = thi;
    run_threads(j, nthreads);
}

/* out[t] = U(seed, st, start+t) */
void synth_keys(uint64_t *out, uint64_t start, uint64_t count, uint64_t seed, uint64_t st, int nthreads) {
    job_t j = {0};
    j.out = out; j.start = start; j.count = count; j.seed = seed; j.st = st; j.kind = 2;
    run_threads(j, nthreads);
}
