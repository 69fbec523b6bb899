/* The literal phi-table fixed-point f of SPEC.md:269, kept only to reproduce
 * the calibration in tools/fixed_point_calibration.py (NOT the product, NOT
 * the oracle):  |f| = min(|a|, |b|, PHI[sat(PHI[|a|] + PHI[|b|])]) with
 * PHI[k] = rint(256 phi(k/256)), 4096 entries uniform on (0, 16].
 * Usage: phi_literal <n> <frames> <mask.bin> <llr.bin f32> <u.bin> <out ok.bin> */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#define Q_MAX 32767
static int16_t PHI[4097];
static int q_sat(int v) { return v > Q_MAX ? Q_MAX : (v < -Q_MAX ? -Q_MAX : v); }
static int f_phi(int a, int b)
{
    int ma = abs(a), mb = abs(b);
    int s = PHI[ma > 4096 ? 4096 : ma] + PHI[mb > 4096 ? 4096 : mb];
    if (s > Q_MAX) s = Q_MAX;
    int m = PHI[s > 4096 ? 4096 : s];
    if (ma < m) m = ma;
    if (mb < m) m = mb;
    return ((a < 0) != (b < 0)) ? -m : m;
}
static void rd(const char *p, void *d, size_t n)
{
    FILE *f = fopen(p, "rb");
    if (!f || fread(d, 1, n, f) != n) { fprintf(stderr, "read %s\n", p); exit(1); }
    fclose(f);
}
int main(int argc, char **argv)
{
    if (argc < 7) return 2;
    int n = atoi(argv[1]), F = atoi(argv[2]);
    size_t N = (size_t)1 << n;
    PHI[0] = Q_MAX;
    for (int k = 1; k <= 4096; k++) { long r = lrint(-log(tanh(k / 512.0)) * 256); PHI[k] = r > Q_MAX ? Q_MAX : r; }
    uint8_t *mask = malloc(N), *u = malloc(N * F), *ok = malloc(F), *xs = malloc(N);
    float *llr = malloc(4 * N * F);
    int *buf = malloc(sizeof(int) * 2 * N);
    uint8_t *uh = malloc(N);
    rd(argv[3], mask, N); rd(argv[4], llr, 4 * N * F); rd(argv[5], u, N * F);
    for (int t = 0; t < F; t++) {
        for (size_t i = 0; i < N; i++) { float r = rintf(llr[t * N + i] * 256.0f); buf[i] = q_sat((int)r); }
        memset(xs, 0, N);
        int d = 0; size_t j = 0; int entering = 1;
        for (;;) {
            size_t W = N >> d;
            if (entering) {
                if (W == 1) { int L = buf[2 * N - 2]; uint8_t v = mask[j] ? u[t * N + j] : (L < 0); uh[j] = v; xs[j] = v; entering = 0; continue; }
                int *nd = buf + (2 * N - 2 * W), *ch = buf + (2 * N - W);
                for (size_t i = 0; i < W / 2; i++) ch[i] = f_phi(nd[i], nd[i + W / 2]);
                d++; j *= 2; continue;
            }
            if (d == 0) break;
            size_t Wp = 2 * W;
            if ((j & 1) == 0) {
                int *nd = buf + (2 * N - 2 * Wp), *ch = buf + (2 * N - Wp);
                for (size_t i = 0; i < W; i++) ch[i] = q_sat(xs[j * W + i] ? nd[i + W] - nd[i] : nd[i + W] + nd[i]);
                j++; entering = 1; continue;
            }
            for (size_t i = 0; i < W; i++) xs[(j - 1) * W + i] ^= xs[j * W + i];
            d--; j >>= 1;
        }
        ok[t] = memcmp(uh, u + t * N, N) == 0;
    }
    FILE *f = fopen(argv[6], "wb");
    fwrite(ok, 1, F, f);
    fclose(f);
    return 0;
}
