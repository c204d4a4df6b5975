/*
 * oracle.c — plain, slow, obviously-correct CPU reference for the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_2405_14642_b200/) never imports, links or
 * executes anything under oracle/, and this file shares no code, header,
 * table or constant with the CUDA path.
 *
 * What it computes (the plain definition):
 *   A = sum_i a_i 2^(32 i), little-endian u32 limbs, fixed width m limbs
 *   ("the result has the same length and element type as
 *   the input integers").
 *   add : out = (A + B) mod 2^(32 m)
 *   mul : out = (A * B) mod 2^(32 m)   (Eq. 1, PAPER.md:338-342, 0 <= i,j,k < M)
 *
 * add follows the sequential ripple of Fig. 1 (left), PAPER.md:125-134:
 * "adds (in a bigger type of double size) the corresponding elements of a
 * and b together with the carry from the previous operation, and then it
 * computes the result element and the carry for the next iteration as the
 * remainder and quotient of the division of the sum to the integer's base".
 *
 * mul is the textbook operand-scanning schoolbook product (Knuth, TAOCP
 * vol. 2, Algorithm 4.3.1M), truncated to m limbs: terms with i + j >= m are
 * never formed (Eq. 1's k < M).  Deliberately NOT the paper's column /
 * product-scanning structure, so a shared mistake is implausible.
 *
 * Parity pins (tests/test_oracle.py, -m "not gpu"): unsigned __int128
 * closed form for m <= 3, exhaustive 16-value limb alphabet for m = 1, 2,
 * random 3-limb pairs, Python-int arbitrary precision for m up to 8192,
 * algebraic invariants, SPEC/PAPER worked examples.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <pthread.h>

/* Fig. 1 left: sequential ripple.  Returns the carry-out of the top limb
 * (dropped by the fixed-width contract; returned for tests only). */
uint32_t oracle_add(uint32_t *out, const uint32_t *a, const uint32_t *b, uint32_t m)
{
    uint64_t c = 0;
    for (uint32_t i = 0; i < m; i++) {
        uint64_t s = (uint64_t)a[i] + (uint64_t)b[i] + c; /* < 2^33 */
        out[i] = (uint32_t)(s % 4294967296ull);           /* remainder */
        c = s / 4294967296ull;                            /* quotient  */
    }
    return (uint32_t)c;
}

/* Truncated schoolbook product: out = a*b mod 2^(32m).
 * t = a_i*b_j + out_{i+j} + c <= (2^32-1)^2 + 2(2^32-1) = 2^64 - 1: no overflow.
 * out may not alias a or b. */
void oracle_mul(uint32_t *out, const uint32_t *a, const uint32_t *b, uint32_t m)
{
    memset(out, 0, (size_t)m * sizeof(uint32_t));
    for (uint32_t i = 0; i < m; i++) {
        uint64_t c = 0;
        for (uint32_t j = 0; i + j < m; j++) {
            uint64_t t = (uint64_t)a[i] * (uint64_t)b[j] + (uint64_t)out[i + j] + c;
            out[i + j] = (uint32_t)t;
            c = t >> 32;
        }
        /* the carry out of column m-1 belongs to 2^(32m) and is dropped */
    }
}

/* Full 2m-limb product (used by residue checks in tests). */
void oracle_mul_full(uint32_t *out2m, const uint32_t *a, const uint32_t *b, uint32_t m)
{
    memset(out2m, 0, (size_t)2 * m * sizeof(uint32_t));
    for (uint32_t i = 0; i < m; i++) {
        uint64_t c = 0;
        for (uint32_t j = 0; j < m; j++) {
            uint64_t t = (uint64_t)a[i] * (uint64_t)b[j] + (uint64_t)out2m[i + j] + c;
            out2m[i + j] = (uint32_t)t;
            c = t >> 32;
        }
        out2m[i + m] = (uint32_t)c;
    }
}

/* ---- the paper's fused workloads, as plain compositions ----
 * 6-Add (Table 1): six dependent additions; the paper does
 * not print the expression, reading R17: r = a + b, then
 * alternately + a, + b (r = 4a + 3b mod 2^(32m)).
 * Poly (Table 2 caption): (a*a + b) * (b*b + b) + a*b,
 * mod 2^(32m), evaluated exactly in that order with the functions above.
 * tmp: 4m scratch words.  out may not alias a or b. */
void oracle_add6(uint32_t *out, const uint32_t *a, const uint32_t *b, uint32_t m)
{
    oracle_add(out, a, b, m);                 /* a + b */
    for (int k = 1; k < 6; k++)               /* + a, + b, + a, + b, + a */
        oracle_add(out, out, (k & 1) ? a : b, m);
}

void oracle_poly(uint32_t *out, const uint32_t *a, const uint32_t *b, uint32_t m, uint32_t *tmp)
{
    uint32_t *aa = tmp, *bb = tmp + m, *t1 = tmp + 2 * (size_t)m, *t2 = tmp + 3 * (size_t)m;
    oracle_mul(aa, a, a, m);                  /* a * a         */
    oracle_add(t1, aa, b, m);                 /* a * a + b     */
    oracle_mul(bb, b, b, m);                  /* b * b         */
    oracle_add(t2, bb, b, m);                 /* b * b + b     */
    oracle_mul(out, t1, t2, m);               /* (..) * (..)   */
    oracle_mul(aa, a, b, m);                  /* a * b         */
    oracle_add(out, out, aa, m);              /* ... + a * b   */
}

/* ---- batch wrappers: instance-major [n_inst][m], one call per instance ---- */

enum { ORACLE_ADD = 0, ORACLE_MUL = 1, ORACLE_ADD6 = 2, ORACLE_POLY = 3 };

typedef struct {
    int op;
    uint32_t *out;
    const uint32_t *a, *b;
    uint64_t lo, hi;
    uint32_t m;
} job_t;

static void *run_job(void *arg)
{
    job_t *j = (job_t *)arg;
    uint32_t *tmp = NULL;
    for (uint64_t i = j->lo; i < j->hi; i++) {
        const uint32_t *ai = j->a + i * j->m, *bi = j->b + i * j->m;
        uint32_t *oi = j->out + i * j->m;
        if (j->op == ORACLE_ADD) {
            oracle_add(oi, ai, bi, j->m);
        } else if (j->op == ORACLE_ADD6) {
            oracle_add6(oi, ai, bi, j->m);
        } else if (j->op == ORACLE_POLY) {
            if (!tmp) tmp = (uint32_t *)malloc((size_t)5 * j->m * sizeof(uint32_t));
            oracle_poly(tmp + 4 * (size_t)j->m, ai, bi, j->m, tmp);
            memcpy(oi, tmp + 4 * (size_t)j->m, (size_t)j->m * sizeof(uint32_t));
        } else {
            /* oracle_mul may not alias: go through a scratch buffer */
            if (!tmp) tmp = (uint32_t *)malloc((size_t)j->m * sizeof(uint32_t));
            oracle_mul(tmp, ai, bi, j->m);
            memcpy(oi, tmp, (size_t)j->m * sizeof(uint32_t));
        }
    }
    free(tmp);
    return NULL;
}

/* Runs the single-threaded oracle on disjoint instance ranges with nthreads
 * POSIX threads (nthreads <= 1: in the calling thread).  Returns 0 on success. */
int oracle_batch(int op, uint32_t *out, const uint32_t *a, const uint32_t *b,
                 uint64_t n_inst, uint32_t m, int nthreads)
{
    if (op < ORACLE_ADD || op > ORACLE_POLY) return -1;
    if (nthreads <= 1 || n_inst < 2) {
        job_t j = {op, out, a, b, 0, n_inst, m};
        run_job(&j);
        return 0;
    }
    if ((uint64_t)nthreads > n_inst) nthreads = (int)n_inst;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
    for (int t = 0; t < nthreads; t++) {
        jobs[t] = (job_t){op, out, a, b, n_inst * t / nthreads, n_inst * (t + 1) / nthreads, m};
        pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}
