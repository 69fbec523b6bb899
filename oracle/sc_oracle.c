/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for SC decoding of polar codes.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (paper_1204_5882_b200)
 * never links or calls it.
 *
 * The reference package ships no decoder: `polar_core` exists only as a
 * specification.  This file restates that
 * specification in plain C, with the conventions fixed by the code that does
 * exist in the reference:
 *
 *   - polar_transform: x = u F^{(x)n}, natural order, no bit reversal,
 *     in-place butterflies, involution
 *   - f(a,b) = sgn a sgn b phi(phi|a| + phi|b|), exact (not min-sum)
 *                                                       SPEC.md:243, :270
 *     evaluated through the algebraically identical boxplus magnitude of the
 *     reference's own construction code          construction.py:300-303
 *   - g(a,b,s) = b + (1-2s) a
 *   - decisions in index order 0..N-1, frozen leaves take the revealed value,
 *     information leaves u = [L < 0] (so L = +-0 decides 0) SPEC.md:243
 *   - explicit (non-recursive) walk with stage-indexed LLR buffers, O(N)
 *                                                       SPEC.md:271
 *   - tree order: f-child (lower indices) first        construction.py:555-557
 *
 * Two arithmetic variants of the same algorithm:
 *   orc_sc_decode_f64 -- double precision, libm expm1/log1p: the formal
 *                        "exact SC" oracle.
 *   orc_sc_decode_f32 -- an fp32 mirror whose f is built only from IEEE
 *                        add/mul/fma/div/rint, written independently of the
 *                        CUDA product but with the same operation sequence,
 *                        so the GPU must reproduce its stage LLRs bit for bit.
 * Both take the revealed frozen values directly (no coset shift), i.e. they
 * are the textbook decoder the SPEC describes.
 *
 * Build: see oracle/Makefile (gcc -O2 -pthread, NO -ffast-math, -ffp-contract=off).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

enum { ORC_F_EXACT = 0, ORC_F_MINSUM = 1 };

/* ------------------------------------------------------------------------- */
/* polar transform on bytes                */

void orc_polar_transform(int n, uint8_t *v)
{
    const size_t N = (size_t)1 << n;
    for (size_t h = 1; h < N; h <<= 1)
        for (size_t i = 0; i < N; i++)
            if ((i & h) == 0) v[i] ^= v[i + h];
}

/* ------------------------------------------------------------------------- */
/* f64 exact boxplus.  |f| = log((1 + e^-a e^-b) / (e^-a + e^-b))
 *                         = log1p((1-e^-a)(1-e^-b) / (e^-a + e^-b)),
 * identical in exact arithmetic to the reference's stable form
 * min + log1p(e^-(a+b)) - log1p(e^-|a-b|)  (construction.py:300-303),
 * but free of its cancellation when both magnitudes are small.            */

double orc_fmag_f64(double a, double b)
{
    double lo = a < b ? a : b, hi = a < b ? b : a;
    if (lo > 300.0) /* e^-lo would underflow; drop the e^-(lo+hi) term (< 1e-260) */
        return lo - log1p(exp(-(hi - lo)));
    double mlo = -expm1(-lo), mhi = -expm1(-hi);
    double den = exp(-lo) + exp(-hi);
    return log1p(mlo * mhi / den);
}

static inline double f_f64(double a, double b, int fmode)
{
    double ma = fabs(a), mb = fabs(b);
    double mag = fmode == ORC_F_MINSUM ? (ma < mb ? ma : mb) : orc_fmag_f64(ma, mb);
    return (signbit(a) != signbit(b)) ? -mag : mag;
}

/* ------------------------------------------------------------------------- */
/* fp32 mirror of the GPU's exact boxplus: the same tables and the same
 * IEEE-only operation sequence (add, mul, fma, floor), so the GPU must
 * reproduce it bit for bit.
 *   lo >= 1:  |f| = (lo - C(hi - lo)) + C(hi + lo),  C(x) = log1p(e^-x)
 *   lo <  1:  |f| = y A(y),  y = T(lo) T(hi),  T(x) = x G(x) = tanh(x/2),
 *             A(y) = 2 atanh(y) / y
 * C, G: piecewise cubics on [0, 24) (1/8 intervals); A on [0, 1/2) (1/64);
 * C(x >= 24) = 0, T(x >= 24) = 1.  Tables: tools/gen_fmag_tables.py.      */

static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

#include "fmag_tables.inc"

static inline float tab_eval(const uint32_t *tab, float xs, int kmax)
{
    float kf = floorf(xs);
    int k = (int)kf;
    if (k > kmax) k = kmax;
    float u = xs - (float)k;
    const uint32_t *c = tab + 4 * k;
    return fmaf(fmaf(fmaf(u2f(c[3]), u, u2f(c[2])), u, u2f(c[1])), u, u2f(c[0]));
}

float orc_fmag_f32(float a, float b)
{
    float lo = fminf(a, b), hi = fmaxf(a, b);
    if (lo >= 1.0f) {
        float dd = hi - lo, ss = hi + lo;
        float cd = dd < 24.0f ? tab_eval(FMAG_TAB_C, dd * 8.0f, 191) : 0.0f;
        float cs = ss < 24.0f ? tab_eval(FMAG_TAB_C, ss * 8.0f, 191) : 0.0f;
        return (lo - cd) + cs;
    }
    float tl = lo * tab_eval(FMAG_TAB_G, lo * 8.0f, 191);
    float th = hi < 24.0f ? hi * tab_eval(FMAG_TAB_G, hi * 8.0f, 191) : 1.0f;
    float y = tl * th;
    return y * tab_eval(FMAG_TAB_A, y * 64.0f, 31);
}

static inline float f_f32(float a, float b, int fmode)
{
    float ma = fabsf(a), mb = fabsf(b);
    float mag = fmode == ORC_F_MINSUM ? fminf(ma, mb) : orc_fmag_f32(ma, mb);
    return u2f(f2u(mag) | ((f2u(a) ^ f2u(b)) & 0x80000000u));
}

/* ------------------------------------------------------------------------- */
/* The SC walk.  Node (d, j) has width W = N >> d and
 * covers leaves [jW, (j+1)W).  Stage buffer d holds the LLRs of the current
 * node at depth d; xs holds x-domain partial sums in place: after node (d,j)
 * is decided, xs[jW:(j+1)W] = T_W(u[jW:(j+1)W]).  When a right child
 * finishes, the left sibling's range ^= the right's, which yields the
 * parent's partial sums (x = (xL ^ xR, xR)).                               */

#define SC_WALK(T, FFN)                                                          \
    const size_t N = (size_t)1 << n;                                             \
    T *buf = (T *)malloc(sizeof(T) * 2 * N);                                     \
    uint8_t *xs = (uint8_t *)calloc(N, 1);                                       \
    if (!buf || !xs) { free(buf); free(xs); return -1; }                         \
    /* stage d lives at buf + (2N - 2W_d); stage 0 = copy of channel LLRs */     \
    memcpy(buf, llr, sizeof(T) * N);                                             \
    if (dump) memcpy(dump, llr, sizeof(T) * N);                                  \
    int d = 0; size_t j = 0; int entering = 1;                                   \
    for (;;) {                                                                   \
        size_t W = N >> d;                                                       \
        if (entering) {                                                          \
            if (W == 1) {                                                        \
                T L = buf[2 * N - 2];                                            \
                uint8_t u = mask[j] ? (frozen_u[j] & 1) : (uint8_t)(L < 0);      \
                if (leaf) leaf[j] = L;                                           \
                u_hat[j] = u; xs[j] = u;                                         \
                entering = 0;                                                    \
                continue;                                                        \
            }                                                                    \
            T *nd = buf + (2 * N - 2 * W), *ch = buf + (2 * N - W);              \
            for (size_t i = 0; i < W / 2; i++) ch[i] = FFN(nd[i], nd[i + W / 2], fmode); \
            d++; j = 2 * j;                                                      \
            if (dump) memcpy(dump + (size_t)d * N + j * (W / 2), ch, sizeof(T) * (W / 2)); \
            continue;                                                            \
        }                                                                        \
        if (d == 0) break;                                                       \
        size_t Wp = W * 2;                                                       \
        if ((j & 1) == 0) { /* left child done: g-step at parent into stage d */ \
            T *nd = buf + (2 * N - 2 * Wp), *ch = buf + (2 * N - Wp);            \
            const uint8_t *s = xs + j * W;                                       \
            for (size_t i = 0; i < W; i++)                                       \
                ch[i] = s[i] ? nd[i + W] - nd[i] : nd[i + W] + nd[i];            \
            j = j + 1; entering = 1;                                             \
            if (dump) memcpy(dump + (size_t)d * N + j * W, ch, sizeof(T) * W);   \
            continue;                                                            \
        }                                                                        \
        /* right child done: combine into the parent's range */                  \
        uint8_t *xl = xs + (j - 1) * W, *xr = xs + j * W;                        \
        for (size_t i = 0; i < W; i++) xl[i] ^= xr[i];                           \
        d--; j >>= 1;                                                            \
    }                                                                            \
    if (x_hat) memcpy(x_hat, xs, N);                                             \
    free(buf); free(xs);                                                         \
    return 0;

/* llr: N channel LLRs; mask: N bytes (1 = frozen); frozen_u: N bytes, the
 * revealed u-values at frozen positions (other entries ignored);
 * u_hat, x_hat (nullable): N bytes out; dump (nullable): (n+1)*N stage LLRs,
 * dump[d*N + j*W + t] = element t of node j at depth d;
 * leaf (nullable): N decision LLRs (= dump[n*N + i]).                        */
int orc_sc_decode_f64(int n, const uint8_t *mask, const double *llr, const uint8_t *frozen_u,
                      int fmode, uint8_t *u_hat, uint8_t *x_hat, double *dump, double *leaf)
{
    SC_WALK(double, f_f64)
}

int orc_sc_decode_f32(int n, const uint8_t *mask, const float *llr, const uint8_t *frozen_u,
                      int fmode, uint8_t *u_hat, uint8_t *x_hat, float *dump, float *leaf)
{
    SC_WALK(float, f_f32)
}

/* Batch drivers: one decoder per worker thread, frames
 * handed out dynamically.  llr is [F][N] fp32 (the GPU's input format); the
 * f64 decoder upcasts each frame exactly.  min_info_abs (nullable, [F]):
 * the smallest |decision LLR| over information positions of each frame, for
 * the "no decision LLR within 1e-4 of zero" parity rule.  0 on success.     */
typedef struct {
    int n, frames, fmode, precision;
    const uint8_t *mask, *frozen_u;
    const float *llr;
    uint8_t *u_hat;
    double *min_info;
    int next, err;
    pthread_mutex_t mu;
} batch_job;

static void *batch_worker(void *arg)
{
    batch_job *b = (batch_job *)arg;
    const size_t N = (size_t)1 << b->n;
    double *ld = b->precision == 64 ? (double *)malloc(sizeof(double) * N) : NULL;
    double *lf = b->min_info ? (double *)malloc(sizeof(double) * N) : NULL;
    float *lf32 = b->min_info ? (float *)malloc(sizeof(float) * N) : NULL;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int f = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (f >= b->frames) break;
        const float *l = b->llr + (size_t)f * N;
        int rc;
        if (b->precision == 64) {
            if (!ld) { rc = -1; }
            else {
                for (size_t i = 0; i < N; i++) ld[i] = (double)l[i];
                rc = orc_sc_decode_f64(b->n, b->mask, ld, b->frozen_u + (size_t)f * N, b->fmode,
                                       b->u_hat + (size_t)f * N, NULL, NULL, lf);
            }
        } else {
            rc = orc_sc_decode_f32(b->n, b->mask, l, b->frozen_u + (size_t)f * N, b->fmode,
                                   b->u_hat + (size_t)f * N, NULL, NULL, lf32);
            if (lf && lf32)
                for (size_t i = 0; i < N; i++) lf[i] = lf32[i];
        }
        if (b->min_info && lf) {
            double m = INFINITY;
            for (size_t i = 0; i < N; i++)
                if (!b->mask[i] && fabs(lf[i]) < m) m = fabs(lf[i]);
            b->min_info[f] = m;
        }
        if (rc) { pthread_mutex_lock(&b->mu); b->err = 1; pthread_mutex_unlock(&b->mu); }
    }
    free(ld);
    free(lf);
    free(lf32);
    return NULL;
}

int orc_sc_decode_batch(int n, const uint8_t *mask, int frames, const float *llr,
                        const uint8_t *frozen_u, int fmode, int precision, int threads,
                        uint8_t *u_hat, double *min_info_abs)
{
    batch_job b = {n, frames, fmode, precision, mask, frozen_u, llr, u_hat, min_info_abs, 0, 0,
                   PTHREAD_MUTEX_INITIALIZER};
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t tid[512];
    int started = 0;
    for (int t = 1; t < threads; t++)
        if (pthread_create(&tid[started], NULL, batch_worker, &b) == 0) started++;
    batch_worker(&b);
    for (int t = 0; t < started; t++) pthread_join(tid[t], NULL);
    return b.err ? -1 : 0;
}

int orc_max_threads(void)
{
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

/* vectorised helpers so tests can pin f itself against the reference form */
void orc_fmag_f32_vec(const float *a, const float *b, float *out, size_t count)
{
    for (size_t i = 0; i < count; i++) out[i] = orc_fmag_f32(a[i], b[i]);
}

void orc_fmag_f64_vec(const double *a, const double *b, double *out, size_t count)
{
    for (size_t i = 0; i < count; i++) out[i] = orc_fmag_f64(a[i], b[i]);
}
