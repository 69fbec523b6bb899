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
/* fp32 mirror of the exact boxplus, IEEE-only operations.
 *   expm(x)  -> e = e^-x, m = 1 - e^-x     (Cody-Waite reduction + Taylor-7 expm1)
 *   log1p(num/den)                          (atanh series after range split)
 *   |f| = log1p(m_lo m_hi / (e_lo + e_hi))            lo <= 40
 *       = lo + log1p(-e / (1 + e)), e = e^-(hi-lo)    lo >  40           */

static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

#define M_LN2_HI 0.693145751953125f
#define M_LN2_LO 1.42860682030941723212e-6f
#define M_INV_LN2 1.44269504088896341f

static inline void expm_f32(float x, float *e, float *m)
{
    if (x > 100.0f) x = 100.0f;
    float kf = rintf(x * M_INV_LN2);
    float r = fmaf(-kf, M_LN2_HI, x);
    r = fmaf(-kf, M_LN2_LO, r);
    float t = -r;
    float h = fmaf(t, 1.0f / 40320.0f, 1.0f / 5040.0f);
    h = fmaf(t, h, 1.0f / 720.0f);
    h = fmaf(t, h, 1.0f / 120.0f);
    h = fmaf(t, h, 1.0f / 24.0f);
    h = fmaf(t, h, 1.0f / 6.0f);
    h = fmaf(t, h, 0.5f);
    float p = fmaf(t * t, h, t); /* expm1(t) */
    int k = (int)kf;
    if (k > 125) { *e = 0.0f; *m = 1.0f; return; }
    float s = u2f((uint32_t)(127 - k) << 23); /* 2^-k */
    *e = fmaf(s, p, s);
    *m = fmaf(-s, p, 1.0f - s);
}

static inline float log1p_ratio_f32(float num, float den)
{
    float s, kf;
    if (num >= -0.29289322f * den && num <= 0.41421356f * den) {
        s = num / (2.0f * den + num);
        kf = 0.0f;
    } else {
        float u = 1.0f + num / den;
        uint32_t b = f2u(u);
        int k = (int)((b >> 23) & 0xffu) - 127;
        float mm = u2f((b & 0x007fffffu) | 0x3f800000u);
        if (mm > 1.41421356f) { mm *= 0.5f; k += 1; }
        s = (mm - 1.0f) / (mm + 1.0f);
        kf = (float)k;
    }
    float z = s * s;
    float h = fmaf(z, 1.0f / 11.0f, 1.0f / 9.0f);
    h = fmaf(z, h, 1.0f / 7.0f);
    h = fmaf(z, h, 1.0f / 5.0f);
    h = fmaf(z, h, 1.0f / 3.0f);
    float s2 = s + s;
    float p = fmaf(s2 * z, h, s2);
    return fmaf(kf, M_LN2_HI, fmaf(kf, M_LN2_LO, p));
}

float orc_fmag_f32(float a, float b)
{
    float lo = fminf(a, b), hi = fmaxf(a, b);
    int big = lo > 40.0f;
    float e1, m1, e2, m2;
    expm_f32(big ? hi - lo : lo, &e1, &m1);
    expm_f32(hi, &e2, &m2);
    float num = big ? -e1 : m1 * m2;
    float den = big ? 1.0f + e1 : e1 + e2;
    float base = big ? lo : 0.0f;
    return base + log1p_ratio_f32(num, den);
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
