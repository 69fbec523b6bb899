// polarsc.cu -- B200-native (sm_100a) successive-cancellation decoder for
// polar codes, behind the C ABI declared in include/polarsc.h.
//
// What is computed is SPEC.md's sc_decode: Arikan's SC
// recursion with the exact boxplus f, g(a,b,s) =
// b + (1-2s)a, decisions in index order, frozen leaves taking the revealed
// values, natural-order F^{(x)n}.  How it is computed is
// B200-first; see DESIGN.md for the full argument.  In short:
//
//  * Coset shift.  Bob knows the revealed frozen u-values v.  With
//    c = polar_transform(v restricted to the frozen set) every node's LLR
//    vector is the textbook one with signs flipped by the node-level codeword
//    of c.  IEEE negation/addition are sign-symmetric and |f| depends only on
//    magnitudes, and the tie rule [L < 0] ignores the sign of zero, so
//    decoding the sign-flipped channel LLRs with all-zero frozen bits makes
//    exactly the same decisions.  The decoder core therefore never needs
//    per-frame frozen values: rate-0 sub-trees have all-zero partial sums.
//  * One CTA per frame walks the whole tree (no host round trips, no
//    per-level launches).  Levels wider than S live in a per-frame HBM/L2
//    scratch; the S-wide sub-tree below is staged in shared memory; sub-trees
//    of width <= 64 are decoded by one warp with LLRs in registers and
//    shuffles (the north star's "bottom five stages by warp shuffles").
//  * Partial sums are bit-packed and kept in place: after node (d,j) is done
//    the bits [jW,(j+1)W) hold T_W(u-hat of that node); a right child's exit
//    XORs into its left sibling, so the frame's final bit array is x-hat
//    (shifted) and u-hat = T(x-hat) comes from the XOR-butterfly kernel.
//  * Decision-exact sub-tree shortcuts (SSC): rate-0 -> bits 0; rate-1 ->
//    hard decisions of the node LLRs, taken only when a conservative bound
//    proves no exact zero can arise inside the sub-tree (so plain SC would
//    make the same decisions); repetition -> the g-chain tree sum in SC's own
//    pairing order.  PQ_OPT_SSC=0 disables all of them.
//  * f uses only IEEE add/mul/fma/div/rint (compiled with --fmad=false), so
//    the fp32 oracle mirror in oracle/sc_oracle.c reproduces every stage LLR
//    bit for bit.

#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <assert.h>

#include <algorithm>
#include <mutex>
#include <climits>
#include <string>
#include <vector>

#include "../../include/polarsc.h"

// ---------------------------------------------------------------------------
// PQ_CHECKED builds (tools/checked_build.sh; compute-sanitizer is not
// available on the GPU pool): device-side bounds asserts on the shared-memory
// and scratch indices, shared memory poisoned (NaN) at kernel start, and
// per-warp random delays at every step of the tree walk and of the TMA ring,
// so that a missing barrier or fence shows up as a parity mismatch or a
// nondeterministic result across runs.
#ifdef PQ_CHECKED
__device__ __forceinline__ uint32_t pq_hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
#define PQ_CHECK(cond)                                                                                 \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("PQ_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,   \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#define PQ_JITTER()                                                                                     \
    do {                                                                                               \
        const uint32_t h_ = pq_hash32((uint32_t)clock() ^ (threadIdx.x >> 5) * 0x9e3779b9u ^ blockIdx.x); \
        if ((h_ & 3u) == 0u) __nanosleep(h_ >> 22);                                                    \
    } while (0)
#else
#define PQ_CHECK(cond) ((void)0)
#define PQ_JITTER() ((void)0)
#endif

// ---------------------------------------------------------------------------
// error plumbing

static thread_local std::string g_last_error;

static int set_err(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int set_err(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return set_err(1 + (int)e_, "%s failed: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------
// device math: the exact boxplus in branch-free, IEEE-only fp32 (add, mul,
// fma, rint and integer bit operations -- no MUFU, no division).  Mirrored
// operation for operation by oracle/sc_oracle.c:orc_fmag_f32; the two must
// agree bit for bit (tests/test_gpu_parity.py checks every stage LLR).

#define LN2_HI 0.693145751953125f
#define LN2_LO 1.42860682030941723212e-6f
#define INV_LN2 1.44269504088896341f

// 1/T_j and log(T_j), T_j = 1 + j/32, rounded to fp32 (same bits in the oracle)
__constant__ uint32_t c_log_tab[64] = {
    0x3f800000u, 0x3f783e10u, 0x3f70f0f1u, 0x3f6a0ea1u, 0x3f638e39u, 0x3f5d67c9u, 0x3f579436u, 0x3f520d21u,
    0x3f4ccccdu, 0x3f47ce0cu, 0x3f430c31u, 0x3f3e82fau, 0x3f3a2e8cu, 0x3f360b61u, 0x3f321643u, 0x3f2e4c41u,
    0x3f2aaaabu, 0x3f272f05u, 0x3f23d70au, 0x3f20a0a1u, 0x3f1d89d9u, 0x3f1a90e8u, 0x3f17b426u, 0x3f14f209u,
    0x3f124925u, 0x3f0fb824u, 0x3f0d3dcbu, 0x3f0ad8f3u, 0x3f088889u, 0x3f064b8au, 0x3f042108u, 0x3f020821u,
    0x00000000u, 0x3cfc14d8u, 0x3d785186u, 0x3db78694u, 0x3df1383bu, 0x3e14aa98u, 0x3e2ff984u, 0x3e4a92d5u,
    0x3e647fbeu, 0x3e7dc8c3u, 0x3e8b3ae5u, 0x3e974716u, 0x3ea30c5eu, 0x3eae8deeu, 0x3eb9cec0u, 0x3ec4d19cu,
    0x3ecf991fu, 0x3eda27bcu, 0x3ee47fbeu, 0x3eeea350u, 0x3ef8947bu, 0x3f012a95u, 0x3f05f397u, 0x3f0aa61fu,
    0x3f0f42fbu, 0x3f13caf1u, 0x3f183ebau, 0x3f1c9f07u, 0x3f20ec7fu, 0x3f2527c3u, 0x3f295169u, 0x3f2d6a02u};
// staged into shared memory at kernel start: lanes index it with divergent j,
// which shared memory serves without bank conflicts (32 distinct words)
__shared__ float pq_tab[64];

__device__ __forceinline__ void load_log_table()
{
    for (int i = threadIdx.x; i < 64; i += blockDim.x) pq_tab[i] = __uint_as_float(c_log_tab[i]);
}

// e = e^-x, m = 1 - e^-x for x >= 0 (x clamped at 86.5: e stays a normal
// float; beyond that e^-x < 2.3e-38 never changes a result).
// Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2; Taylor-7 expm1(-r).
__device__ __forceinline__ void pq_expm(float x, float &e, float &m)
{
    x = fminf(x, 86.5f);
    const float kf = rintf(x * INV_LN2);
    float r = fmaf(-kf, LN2_HI, x);
    r = fmaf(-kf, LN2_LO, r);
    const float t = -r;
    float h = fmaf(t, 1.0f / 40320.0f, 1.0f / 5040.0f);
    h = fmaf(t, h, 1.0f / 720.0f);
    h = fmaf(t, h, 1.0f / 120.0f);
    h = fmaf(t, h, 1.0f / 24.0f);
    h = fmaf(t, h, 1.0f / 6.0f);
    h = fmaf(t, h, 0.5f);
    const float p = fmaf(t * t, h, t);
    const float s = __uint_as_float((uint32_t)(127 - (int)kf) << 23);  // 2^-k
    e = fmaf(s, p, s);
    m = fmaf(-s, p, 1.0f - s);
}

// 1/d for d in [2^-126, 2]: integer seed, three Newton steps (FMA only)
__device__ __forceinline__ float pq_rcp(float d)
{
    float r = __uint_as_float(0x7ef311c7u - __float_as_uint(d));
    float e = fmaf(-d, r, 1.0f);
    r = fmaf(r, e, r);
    e = fmaf(-d, r, 1.0f);
    r = fmaf(r, e, r);
    e = fmaf(-d, r, 1.0f);
    return fmaf(r, e, r);
}

// log1p(q), 0 <= q < 2^100: u = 1 + q with its exact rounding error (Fast2Sum),
// u = 2^k m, m in [T_j, T_j + 1/32), log m = log T_j + log1p((m - T_j)/T_j)
__device__ __forceinline__ float pq_log1p(float q)
{
    const float u = 1.0f + q;
    const float err = (fmaxf(1.0f, q) - u) + fminf(1.0f, q);
    const uint32_t b = __float_as_uint(u);
    const int k = (int)(b >> 23) - 127;
    const uint32_t j = (b >> 18) & 31u;
    const float m = __uint_as_float((b & 0x007fffffu) | 0x3f800000u);
    const float T = __uint_as_float(0x3f800000u | (j << 18));
    const float invT = pq_tab[j], logT = pq_tab[32 + j];
    const float r = (m - T) * invT;
    float p = fmaf(r, -1.0f / 6.0f, 0.2f);
    p = fmaf(r, p, -0.25f);
    p = fmaf(r, p, 1.0f / 3.0f);
    p = fmaf(r, p, -0.5f);
    p = fmaf(r, p, 1.0f);
    p = p * r;
    const float inv_u = __uint_as_float((uint32_t)(127 - k) << 23) * invT;
    const float kf = (float)k;
    return fmaf(kf, LN2_HI, fmaf(kf, LN2_LO, logT + (p + err * inv_u)));
}

// |f| for magnitudes a, b >= 0 (lo = min, hi = max):
//   lo <= 8:  log1p((1 - e^-lo)(1 - e^-hi) / (e^-lo + e^-hi))
//   lo >  8:  lo - log1p(e^-(hi - lo))      (drops log1p(e^-(lo+hi)) < 1.2e-7, i.e.
//                                            < 2e-8 relative to a result >= 7.3)
// = log((1 + e^-a e^-b)/(e^-a + e^-b)) = phi(phi(a) + phi(b)),
// the reference's stable boxplus (construction.py:132-135) in a form free of
// its cancellation at small magnitudes.  Max relative error ~3.4e-7.
__device__ __forceinline__ float pq_fmag(float a, float b)
{
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    const bool big = lo > 8.0f;
    float e1, m1, e2, m2;
    pq_expm(big ? hi - lo : lo, e1, m1);
    pq_expm(hi, e2, m2);
    const float q = (m1 * m2) * pq_rcp(e1 + e2);
    const float l = pq_log1p(big ? e1 : q);
    return big ? lo - l : l;
}

// The same exact boxplus with the SFU's transcendental approximations
// (ex2/lg2/rcp.approx, ~2 ulp): ~60 instructions and ~130 cycles latency
// instead of ~92 and 232, max relative error ~1e-6.  Not reproducible by a
// CPU mirror (SFU results are not IEEE-specified), so its parity is checked
// against the f64 oracle with the north star's tolerance.
//   m = 1 - e^-x: Taylor-7 for x < 1/2 (cancellation), else 1 - ex2(...)
//   log1p(Q): series to Q^10 for Q < 1/4, else lg2(1+Q) ln2 + err/(1+Q)
//             with the exact rounding error err of 1+Q (Fast2Sum)
__device__ __forceinline__ float fast_m(float x, float e)
{
    float h = fmaf(x, 1.0f / 5040.0f, -1.0f / 720.0f);
    h = fmaf(x, h, 1.0f / 120.0f);
    h = fmaf(x, h, -1.0f / 24.0f);
    h = fmaf(x, h, 1.0f / 6.0f);
    h = fmaf(x, h, -0.5f);
    h = fmaf(x, h, 1.0f);
    return x < 0.5f ? x * h : 1.0f - e;
}

__device__ __forceinline__ float fast_log1p(float q)
{
    // series: q - q^2/2 + ... - q^10/10
    float h = fmaf(q, -0.1f, 1.0f / 9.0f);
    h = fmaf(q, h, -0.125f);
    h = fmaf(q, h, 1.0f / 7.0f);
    h = fmaf(q, h, -1.0f / 6.0f);
    h = fmaf(q, h, 0.2f);
    h = fmaf(q, h, -0.25f);
    h = fmaf(q, h, 1.0f / 3.0f);
    h = fmaf(q, h, -0.5f);
    h = fmaf(q, h, 1.0f);
    const float ser = q * h;
    const float u = 1.0f + q;
    const float err = (fmaxf(1.0f, q) - u) + fminf(1.0f, q);
    // 1/u within a factor 2 is plenty for the tiny correction err/u
    const float inv_u = __uint_as_float(0x7f000000u - (__float_as_uint(u) & 0x7f800000u));
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u));
    const float big = fmaf(lg, 0.69314718055994531f, err * inv_u);
    return q < 0.25f ? ser : big;
}

__device__ __forceinline__ float fast_ex2(float x)
{
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float fast_rcp(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float pq_fmag_fast(float a, float b)
{
    const float lo = fminf(a, b), hi = fmaxf(a, b);
    const bool big = lo > 8.0f;
    const float x1 = fminf(big ? hi - lo : lo, 86.5f), x2 = fminf(hi, 86.5f);
    const float e1 = fast_ex2(x1 * -1.44269504088896341f), e2 = fast_ex2(x2 * -1.44269504088896341f);
    const float m1 = fast_m(x1, e1), m2 = fast_m(x2, e2);
    const float q = (m1 * m2) * fast_rcp(e1 + e2);
    const float l = fast_log1p(big ? e1 : q);
    return big ? lo - l : l;
}


// g(a, b, s) = b + (1 - 2s) a
__device__ __forceinline__ float pq_g(float a, float b, uint32_t s) { return s ? b - a : b + a; }

// ---- fixed point: Q8.8 raw values carried in fp32
// registers (integers |r| <= 32767 are exact), saturating adds, and the exact
// boxplus by table lookup (oracle/sc_oracle.c explains the choice of table):
//   |f| = max(0, min(|a|, |b|) + CORR[min(|a| + |b|, 4096)] - CORR[min(||a| - |b||, 4096)])
// CORR[k] = rint(256 ln(1 + e^(-k/256))) held as fp32 in shared memory (no
// int/float conversions; the two lookups are independent).
#define Q_MAX 32767.0f
__constant__ float CORR_TAB_C[4097];
// C[k] = 0 for every k >= 1598 (256 ln(1 + e^(-k/256)) < 1/2), so the shared
// copy keeps 2048 entries and f clamps its index at 2047 -- the same values as
// the 4097-entry table clamped at 4096 (fixed_tables checks it), 8 KB less
// shared memory per CTA
#define CORR_SMEM 2048
__shared__ float pq_corrtab[CORR_SMEM];

template <int FM>
__device__ __forceinline__ float qadd(float x, float y)
{
    const float r = x + y;
    return FM == PQ_F_FIXED ? fminf(fmaxf(r, -Q_MAX), Q_MAX) : r;
}

// g with the mode's addition (saturating in fixed point)
template <int FM>
__device__ __forceinline__ float pq_gt(float a, float b, uint32_t s) { return qadd<FM>(b, s ? -a : a); }

// exact small integer held in a float -> int, with full-rate ALU ops
__device__ __forceinline__ int small_f2i(float x) { return __float_as_int(x + 12582912.0f) - 0x4B400000; }

// table entry for an index held as a small exact integer in a float, x in
// [0, 2047]: x + 1.5 * 2^21 has an ulp of 1/4, so its bit pattern is
// 0x4A400000 + 4 x -- the byte offset into the fp32 table plus a constant.
// One integer add of (table base - 0x4A400000) gives the shared-memory
// address: no index conversion, no scaling (PQ_F_LEA; two instructions per
// f fewer than the index form in the upper and block bands).
#ifndef PQ_F_LEA
#define PQ_F_LEA 0  // measured: c3 / c4 -0.3 %, c2 +-0 (profiles/r02/ab_upper_band.txt)
#endif
__device__ __forceinline__ float corr_at(float x)
{
#if PQ_F_LEA
    const uint32_t k = (uint32_t)__cvta_generic_to_shared(pq_corrtab) - 0x4A400000u;
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(__float_as_uint(x + 3145728.0f) + k));
    return v;
#else
    return pq_corrtab[small_f2i(x)];
#endif
}

// magnitudes ma, mb (raw codes)
__device__ __forceinline__ float pq_fmag_fixed(float ma, float mb)
{
    const float cs = corr_at(fminf(ma + mb, (float)(CORR_SMEM - 1)));
    const float cd = corr_at(fminf(fabsf(ma - mb), (float)(CORR_SMEM - 1)));
    return fmaxf(fminf(ma, mb) + cs - cd, 0.0f);
}

template <int FM>
__device__ __forceinline__ float pq_f(float a, float b)
{
    const float ma = fabsf(a), mb = fabsf(b);
    const float mag = FM == PQ_F_MINSUM ? fminf(ma, mb)
                      : FM == PQ_F_FAST ? pq_fmag_fast(ma, mb)
                      : FM == PQ_F_FIXED ? pq_fmag_fixed(ma, mb)
                                         : pq_fmag(ma, mb);
    return __uint_as_float(__float_as_uint(mag) | ((__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u));
}

// Rate-1 shortcut guard.  b(t) = 0.427 t^2 (t < 1), max(0.427, t - ln 2)
// (t >= 1) lower-bounds |boxplus(t, t)| in exact arithmetic; chained k times
// from m = min|L| of a rate-1 node of width 2^k it lower-bounds every LLR
// inside the node's sub-tree (|g| >= max of its operands there -- the signs
// agree by construction -- and boxplus is monotone).  A chain result >= 1e-30
// proves no fp32 underflow to an exact zero can occur, the only way plain SC
// could decide differently from the node's hard decisions.  RATE1_TAU[k] is
// the smallest fp32 m (rounded up, plus one ulp) whose chain reaches 1e-30;
// tests/test_oracle.py re-derives the table and checks b(t) <= |f(t, t)|.
__constant__ float RATE1_TAU[26] = {
    1.000000097210625e-30f, 1.5303335787713972e-15f, 5.986585449591075e-08f, 0.00037443434121087193f,
    0.02961242012679577f, 0.26334378123283386f, 0.7853217124938965f, 1.4785218238830566f,
    2.171721935272217f, 2.864922046661377f, 3.558121919631958f, 4.251322269439697f,
    4.944522380828857f, 5.637722492218018f, 6.3309221267700195f, 7.02412223815918f,
    7.71732234954834f, 8.410523414611816f, 9.103723526000977f, 9.79692268371582f,
    10.49012279510498f, 11.18332290649414f, 11.8765230178833f, 12.569723129272461f,
    13.262923240661621f, 13.956123352050781f};

// Fixed-point (Q8.8) counterpart, in raw units: L(t) = min over a, b >= t of
// |f_fix(a, b)| (a suffix minimum, so non-decreasing); RATE1_TAU_FIX[k] is the
// smallest raw m whose k-fold chain m -> L(m) stays >= 1 LSB.  Computed on the
// host from the table at first use (fixed_tables).
__constant__ float RATE1_TAU_FIX[26];

template <int FM>
__device__ __forceinline__ float tau(int k) { return FM == PQ_F_FIXED ? RATE1_TAU_FIX[k] : RATE1_TAU[k]; }

// the fixed-point decoder's single-warp band (widths <= 2048)
#ifndef PQ_WIDE_WARP_LOG2
#define PQ_WIDE_WARP_LOG2 11  // widest node the serial warp takes (wider: block steps)
#endif
#include "serial_q88.cuh"
#ifndef PQ_SE2
#define PQ_SE2 1
#endif

template <int FM>
__device__ __forceinline__ bool rate1_guard(float m, int k) { return m >= tau<FM>(k); }

// ---------------------------------------------------------------------------
// node types (host computes them from the frozen mask; heap order)

enum : uint8_t { NT_MIXED = 0, NT_RATE0 = 1, NT_RATE1 = 2, NT_REP = 3 };

struct DecParams {
    int n, log2S, plain, frames;
    uint32_t N, S, wpf;          // block length, shared sub-tree width, words per frame
    const float *llr;            // [F][N] fp32 channel LLRs (or null when ybits / llr16)
    const short *llr16;          // [F][N] Q8.8 raw channel codes (fixed mode), or null
    const uint32_t *ybits;       // [F][wpf] BSC received bits (or null)
    float mag;                   // BSC LLR magnitude
    const uint32_t *cw;          // [F][wpf] coset words c = T(v & mask), or null
    const uint8_t *types;        // [2N] heap-order node types
    float *scr;                  // [F][N] stage buffers for widths > S
    uint32_t *X;                 // [F][wpf] out: shifted x-hat partial sums
    float *dump;                 // [F][n+1][N] stage dump (plain mode), or null
    int fixed;                   // 1: quantise channel LLRs to Q8.8 raw codes on load
    unsigned long long *prof;    // [F][PQ_PROF_SLOTS] clock64 cycles per step class, or null
    uint32_t wmax;               // widest node the single-warp band takes (32..256)
    uint32_t K;                  // CTAs per frame (a thread-block cluster; 1, 2, 4 or 8)
    const uint32_t *fmask;       // [wpf] frozen mask words (bit i = leaf i frozen), shared by frames
};

// step classes for the optional per-frame cycle profile (PQ_OPT_PROFILE)
enum { PR_UP_F = 0, PR_UP_G, PR_UP_OTHER, PR_SM_F, PR_SM_G, PR_SM_OTHER, PR_WARP, PR_TYPES, PR_RATE1,
       PR_TOTAL, PR_NODES_WARP, PR_NODES_BLOCK };

struct FrameCtx {
    const float *llr;
    const short *l16;
    const uint32_t *y, *cw;
    float *scr;
    uint32_t *X;
    float *dump;
};

__device__ __forceinline__ float chan_load(const DecParams &p, const FrameCtx &fc, uint32_t i)
{
    uint32_t c = fc.cw ? (fc.cw[i >> 5] >> (i & 31)) & 1u : 0u;
    if (fc.y) {
        const uint32_t y = (fc.y[i >> 5] >> (i & 31)) & 1u;
        return (y ^ c) ? -p.mag : p.mag;  // p.mag is pre-quantised in fixed mode
    }
    float v;
    if (fc.l16) {
        v = (float)fc.l16[i];  // already a Q8.8 code (|raw| <= 32767 by contract)
    } else {
        v = fc.llr[i];
        if (p.fixed) v = fminf(fmaxf(rintf(v * 256.0f), -Q_MAX), Q_MAX);
    }
    return c ? -v : v;
}

// four consecutive channel LLRs (i % 4 == 0), sign-flipped by the coset word
__device__ __forceinline__ float4 chan_load4(const DecParams &p, const FrameCtx &fc, uint32_t i)
{
    const uint32_t c4 = fc.cw ? (__ldg(fc.cw + (i >> 5)) >> (i & 31)) & 15u : 0u;
    float4 v;
    if (fc.y) {
        const uint32_t y4 = ((__ldg(fc.y + (i >> 5)) >> (i & 31)) & 15u) ^ c4;
        v.x = (y4 & 1u) ? -p.mag : p.mag;
        v.y = (y4 & 2u) ? -p.mag : p.mag;
        v.z = (y4 & 4u) ? -p.mag : p.mag;
        v.w = (y4 & 8u) ? -p.mag : p.mag;
        return v;
    }
    if (fc.l16) {
        const short4 q = __ldg(reinterpret_cast<const short4 *>(fc.l16 + i));
        v = make_float4((float)q.x, (float)q.y, (float)q.z, (float)q.w);
    } else {
        v = __ldg(reinterpret_cast<const float4 *>(fc.llr + i));
    }
    if (p.fixed && !fc.l16) {
        v.x = fminf(fmaxf(rintf(v.x * 256.0f), -Q_MAX), Q_MAX);
        v.y = fminf(fmaxf(rintf(v.y * 256.0f), -Q_MAX), Q_MAX);
        v.z = fminf(fmaxf(rintf(v.z * 256.0f), -Q_MAX), Q_MAX);
        v.w = fminf(fmaxf(rintf(v.w * 256.0f), -Q_MAX), Q_MAX);
    }
    v.x = __uint_as_float(__float_as_uint(v.x) ^ ((c4 & 1u) << 31));
    v.y = __uint_as_float(__float_as_uint(v.y) ^ ((c4 & 2u) << 30));
    v.z = __uint_as_float(__float_as_uint(v.z) ^ ((c4 & 4u) << 29));
    v.w = __uint_as_float(__float_as_uint(v.w) ^ ((c4 & 8u) << 28));
    return v;
}

// smem layout: [2S floats stage LLRs][SW words partial sums][2S bytes types][SW words frozen mask]
struct Smem {
    float *st;
    uint32_t *xs;
    uint8_t *ty;
    uint32_t *fm;  // frozen-mask words of the current S-sub-tree (fixed-point serial engine)
};

// stage pointer for a node of width W at depth d >= 1
__device__ __forceinline__ float *stage_ptr(const DecParams &p, const FrameCtx &fc, const Smem &sm,
                                            uint32_t W)
{
    PQ_CHECK(W >= 1 && W <= p.N && (W & (W - 1)) == 0 && (W <= p.S || fc.scr != nullptr));
    return W <= p.S ? sm.st + (2 * p.S - 2 * W) : fc.scr + (p.N - 2 * W);
}

// ---------------------------------------------------------------------------
// warp-level decoding of sub-trees of width W <= 256, all LLRs in registers.
//
// W = 32V (V = 2, 4, 8): lane l holds elements l + 32t, t < V.  The f- and
// g-steps down to W = 32 are in-lane (element i pairs with i + W/2 in the
// same lane), so these levels need no shuffles at all.
//
// W <= 32: an iterative engine (no calls, no local memory).  Register A holds
// the root node (lane l = element l); register B holds the current node of
// every depth e >= 1 side by side, depth e at lanes [o(e), o(e) + 32>>e) with
// o(e) = 32 - 2^(6-e) (0, 16, 24, 28, 30).  The f-step stores the shuffled
// operand pair (a, b) in registers Ca/Cb at the child's lanes, so the later
// g-step of the same node reuses them without shuffling.  Left-child partial
// sums of every depth are packed into one uniform word XL at bit offset o(e).
// Node types (2 bits each) and the leaf frozen bits are fetched once per
// engine entry into three uniform bit masks.

__device__ __forceinline__ int eng_off(int e) { return e == 0 ? 0 : 32 - (64 >> e); }
__device__ __forceinline__ uint32_t lowmask(int w) { return w >= 32 ? 0xffffffffu : ((1u << w) - 1u); }
__device__ __forceinline__ int ilog2(uint32_t w) { return 31 - __clz(w); }

struct WarpCtx {
    const uint8_t *ty;   // S-sub-tree-local heap types (shared memory)
    float *dump;         // frame dump base (plain mode) or null
    uint32_t N;
    int plain;
    int dS;              // absolute depth of the S-sub-tree root
    uint32_t jS;         // its index
    unsigned long long *prof;  // shared {cycles in <=32-wide decoders, calls} or null
};

#ifdef PQ_UBENCH_TIMING
__device__ unsigned long long g_ub_time[16], g_ub_count[16];
#define UB_BEGIN() const long long ub_t0_ = clock64()
#define UB_END(slot)                                                   \
    do {                                                               \
        if ((threadIdx.x & 31) == 0) {                                 \
            atomicAdd(&g_ub_time[slot], (unsigned long long)(clock64() - ub_t0_)); \
            atomicAdd(&g_ub_count[slot], 1ull);                        \
        }                                                              \
    } while (0)
#else
#define UB_BEGIN()
#define UB_END(slot)
#endif

// Node types of one width-32 sub-tree as uniform bit masks, indexed by the
// sub-tree-local heap index h (root h = 1, children 2h, 2h+1): internal
// nodes h < 32 carry 2 type bits (tb0, tb1); leaves h = 32..63 carry the
// frozen flag in `leaf` (bit h - 32).  Sub-trees narrower than 32 (blocks
// shorter than 32 only) sit at the leftmost node of that width.
struct TypeBits {
    uint32_t tb0, tb1, leaf;
};
__device__ __forceinline__ uint32_t tget(const TypeBits &T, int h)
{
    return ((T.tb0 >> h) & 1u) | (((T.tb1 >> h) & 1u) << 1);
}

// absolute position of a node, for the plain-mode stage dump
struct NodePos {
    float *dump;
    uint32_t N;
    int d;
    uint32_t j;
};
__device__ __forceinline__ NodePos child_pos(const NodePos &p, int side)
{
    NodePos c = p;
    c.d = p.d + 1;
    c.j = 2 * p.j + side;
    return c;
}
// write node values held in registers (lane 0 writes; every lane holds them)
template <int W>
__device__ __forceinline__ void dump_regs(const NodePos &p, const float (&x)[W])
{
    if (p.dump && (threadIdx.x & 31) == 0) {
        float *o = p.dump + (size_t)p.d * p.N + (size_t)p.j * W;
#pragma unroll
        for (int i = 0; i < W; i++) o[i] = x[i];
    }
}
// write node values held one per lane (lanes 0..W-1)
__device__ __forceinline__ void dump_lanes(const NodePos &p, float v, int W)
{
    const int lane = threadIdx.x & 31;
    if (p.dump && lane < W) p.dump[(size_t)p.d * p.N + (size_t)p.j * W + lane] = v;
}

// ---- closed forms: the node's values are in registers of every lane; the
// whole sub-tree is decided without shuffles or loops (uniform branches only)

template <int FM, bool plain>
__device__ __forceinline__ uint32_t dec2(float a, float b, const TypeBits &T, int h, const NodePos &np)
{
    const uint32_t t = plain ? NT_MIXED : tget(T, h);
    if (t == NT_RATE0) return 0u;
    if (t == NT_REP) return qadd<FM>(b, a) < 0.0f ? 3u : 0u;
    if (t == NT_RATE1 && fminf(fabsf(a), fabsf(b)) >= tau<FM>(1))
        return (a < 0.0f ? 1u : 0u) | (b < 0.0f ? 2u : 0u);
    const bool fa = (T.leaf >> (2 * h - 32)) & 1u, fb = (T.leaf >> (2 * h - 31)) & 1u;
    const float l = pq_f<FM>(a, b);
    const uint32_t u0 = fa ? 0u : (l < 0.0f ? 1u : 0u);
    const float r = pq_gt<FM>(a, b, u0);
    const uint32_t u1 = fb ? 0u : (r < 0.0f ? 1u : 0u);
    if (plain && np.dump && (threadIdx.x & 31) == 0) {
        np.dump[(size_t)(np.d + 1) * np.N + 2 * np.j] = l;
        np.dump[(size_t)(np.d + 1) * np.N + 2 * np.j + 1] = r;
    }
    return (u0 ^ u1) | (u1 << 1);
}

// W = 4 node whose four values every lane holds: the whole sub-tree in
// registers, no shuffles (uniform branches on the node types only).
template <int FM, bool plain>
__device__ __forceinline__ uint32_t dec4(float x0, float x1, float x2, float x3, const TypeBits &T, int h,
                                         const NodePos &np)
{
    const uint32_t t = plain ? NT_MIXED : tget(T, h);
    if (t == NT_RATE0) return 0u;
    if (t == NT_REP) return qadd<FM>(qadd<FM>(x3, x1), qadd<FM>(x2, x0)) < 0.0f ? 15u : 0u;
    if (t == NT_RATE1 &&
        fminf(fminf(fabsf(x0), fabsf(x1)), fminf(fabsf(x2), fabsf(x3))) >= tau<FM>(2))
        return (x0 < 0.0f ? 1u : 0u) | (x1 < 0.0f ? 2u : 0u) | (x2 < 0.0f ? 4u : 0u) | (x3 < 0.0f ? 8u : 0u);
    uint32_t xl = 0, xr = 0;
    const bool lane0 = (threadIdx.x & 31) == 0;
    if (plain || tget(T, 2 * h) != NT_RATE0) {
        const float c0 = pq_f<FM>(x0, x2), c1 = pq_f<FM>(x1, x3);
        if (plain && np.dump && lane0) {
            np.dump[(size_t)(np.d + 1) * np.N + 4 * np.j] = c0;
            np.dump[(size_t)(np.d + 1) * np.N + 4 * np.j + 1] = c1;
        }
        xl = dec2<FM, plain>(c0, c1, T, 2 * h, child_pos(np, 0));
    }
    if (plain || tget(T, 2 * h + 1) != NT_RATE0) {
        const float c0 = pq_gt<FM>(x0, x2, xl & 1u), c1 = pq_gt<FM>(x1, x3, (xl >> 1) & 1u);
        if (plain && np.dump && lane0) {
            np.dump[(size_t)(np.d + 1) * np.N + 4 * np.j + 2] = c0;
            np.dump[(size_t)(np.d + 1) * np.N + 4 * np.j + 3] = c1;
        }
        xr = dec2<FM, plain>(c0, c1, T, 2 * h + 1, child_pos(np, 1));
    }
    return ((xl ^ xr) & 3u) | (xr << 2);
}

// ---- lane-parallel levels: lane i holds element i of a W = 8 / 16 / 32 node

// rate-1 / repetition handling of a node held one element per lane (lanes < W)
template <int FM>
__device__ __forceinline__ bool lanes_special(float v, int W, uint32_t t, uint32_t &bits)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    if (t == NT_RATE0) {
        bits = 0;
        return true;
    }
    if (t == NT_RATE1) {
        // both votes issue back to back: guard (all |L| >= tau) and the signs
        const bool ok = __all_sync(FULL, lane >= W || fabsf(v) >= tau<FM>(ilog2((uint32_t)W)));
        const uint32_t neg = __ballot_sync(FULL, lane < W && v < 0.0f);
        if (ok) {
            bits = neg & lowmask(W);
            return true;
        }
    }
    if (t == NT_REP) {
        // SC's g-chain sum in its pairing order, x[i] <- x[i + hh] + x[i] for
        // hh = W/2 .. 1: a shuffle-down tree (lane i < hh reads lane i + hh < W)
        float x = v;
        for (int hh = W >> 1; hh >= 1; hh >>= 1) x = qadd<FM>(__shfl_down_sync(FULL, x, hh), x);
        bits = __shfl_sync(FULL, x, 0) < 0.0f ? lowmask(W) : 0u;
        return true;
    }
    return false;
}

// ---- frozen-pattern-specialised width-8 nodes.  The polar partial order
// leaves very few frozen patterns for mixed width-8 nodes (6-10 in the
// BASELINE codes, covering ~100% of them), so each common pattern gets a
// straight-line SC routine: no type dispatch, no loops, only shuffles and
// the f chain.  Rate-1 children are hard decisions behind the same guard as
// elsewhere; if any guard fails the caller redoes the node generically.
// Values are lane-distributed (lane i = element i); results are uniform.

// width-4 sub-node, frozen nibble P (bit i = leaf i frozen), lanes 0..3
template <int FM, uint32_t P>
__device__ __forceinline__ uint32_t w4_pat(float v, bool &ok)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    if constexpr (P == 0xF) {  // rate-0
        return 0u;
    } else if constexpr (P == 0x0) {  // rate-1
        ok &= __all_sync(FULL, lane >= 4 || fabsf(v) >= tau<FM>(2));
        return __ballot_sync(FULL, lane < 4 && v < 0.0f) & 15u;
    } else if constexpr (P == 0x7) {  // repetition: (L3 + L1) + (L2 + L0), SC's pairing
        float sum = qadd<FM>(v, __shfl_down_sync(FULL, v, 2));
        sum = qadd<FM>(__shfl_down_sync(FULL, sum, 1), sum);
        return __shfl_sync(FULL, sum, 0) < 0.0f ? 15u : 0u;
    } else if constexpr (P == 0x1) {  // SPC: REP(2) left, rate-1 right
        const float b = __shfl_down_sync(FULL, v, 2);
        const float l = pq_f<FM>(v, b);
        const float l0 = __shfl_sync(FULL, l, 0), l1 = __shfl_sync(FULL, l, 1);
        const uint32_t u = qadd<FM>(l1, l0) < 0.0f ? 1u : 0u;
        const float r = pq_gt<FM>(v, b, u);
        ok &= __all_sync(FULL, lane >= 2 || fabsf(r) >= tau<FM>(1));
        const uint32_t xr = __ballot_sync(FULL, lane < 2 && r < 0.0f) & 3u;
        return ((u ? 3u : 0u) ^ xr) | (xr << 2);
    } else if constexpr (P == 0x3) {  // rate-0 left, rate-1 right
        const float r = qadd<FM>(__shfl_down_sync(FULL, v, 2), v);
        ok &= __all_sync(FULL, lane >= 2 || fabsf(r) >= tau<FM>(1));
        const uint32_t xr = __ballot_sync(FULL, lane < 2 && r < 0.0f) & 3u;
        return xr | (xr << 2);
    } else {  // P == 0x5: REP(2) left, REP(2) right
        const float b = __shfl_down_sync(FULL, v, 2);
        const float l = pq_f<FM>(v, b);
        const uint32_t u1 = qadd<FM>(__shfl_sync(FULL, l, 1), __shfl_sync(FULL, l, 0)) < 0.0f ? 1u : 0u;
        const float r = pq_gt<FM>(v, b, u1);
        const uint32_t u3 = qadd<FM>(__shfl_sync(FULL, r, 1), __shfl_sync(FULL, r, 0)) < 0.0f ? 1u : 0u;
        return ((u1 ? 3u : 0u) ^ (u3 ? 3u : 0u)) | ((u3 ? 3u : 0u) << 2);
    }
}

template <int FM, uint32_t LP, uint32_t RP>
__device__ __forceinline__ uint32_t w8_pat(float v, bool &ok)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float b = __shfl_down_sync(FULL, v, 4);
    uint32_t xl = 0;
    if constexpr (LP != 0xF) xl = w4_pat<FM, LP>(pq_f<FM>(v, b), ok);
    const float r = pq_gt<FM>(v, b, (xl >> (lane & 3)) & 1u);
    const uint32_t xr = w4_pat<FM, RP>(r, ok);
    return (xl ^ xr) | (xr << 4);
}

// returns true and the bits if the width-8 node's frozen pattern has a routine
template <int FM>
__device__ __forceinline__ bool w8_fast(float v, uint32_t pat, uint32_t &bits)
{
    bool ok = true;
    switch (pat) {
    case 0x01: bits = w8_pat<FM, 0x1, 0x0>(v, ok); break;  // F I I I I I I I
    case 0x17: bits = w8_pat<FM, 0x7, 0x1>(v, ok); break;  // F F F I F I I I
    case 0x1F: bits = w8_pat<FM, 0xF, 0x1>(v, ok); break;  // F F F F F I I I
    case 0x07: bits = w8_pat<FM, 0x7, 0x0>(v, ok); break;  // F F F I I I I I
    case 0x03: bits = w8_pat<FM, 0x3, 0x0>(v, ok); break;  // F F I I I I I I
    case 0x3F: bits = w8_pat<FM, 0xF, 0x3>(v, ok); break;  // F F F F F F I I
    case 0x05: bits = w8_pat<FM, 0x5, 0x0>(v, ok); break;  // F I F I I I I I
    case 0x15: bits = w8_pat<FM, 0x5, 0x1>(v, ok); break;  // F I F I F I I I
    default: return false;
    }
    return ok;
}

// W = 8 node, lane i holds element i (lanes 0..7).  One copy (noinline):
// lane-parallel f/g step, then the width-4 children in registers.
template <int FM, bool plain>
__device__ __noinline__ uint32_t dec8(float v, const TypeBits T, int h, const NodePos np)
{
    UB_BEGIN();
    const unsigned FULL = 0xffffffffu;
    uint32_t bits;
#ifndef PQ_W8_PATTERNS
#define PQ_W8_PATTERNS 1
#endif
    if (PQ_W8_PATTERNS && !plain && tget(T, h) == NT_MIXED && w8_fast<FM>(v, (T.leaf >> (8 * (h - 4))) & 0xffu, bits)) {
        UB_END(4);
        return bits;
    }
    if (!plain && lanes_special<FM>(v, 8, tget(T, h), bits)) {
        UB_END(5);
        return bits;
    }
    const float b = __shfl_down_sync(FULL, v, 4);
    uint32_t xl = 0, xr = 0;
    if (plain || tget(T, 2 * h) != NT_RATE0) {
        const float c = pq_f<FM>(v, b);
        if (plain) dump_lanes(child_pos(np, 0), c, 4);
        xl = dec4<FM, plain>(__shfl_sync(FULL, c, 0), __shfl_sync(FULL, c, 1), __shfl_sync(FULL, c, 2),
                      __shfl_sync(FULL, c, 3), T, 2 * h, child_pos(np, 0));
    }
    if (plain || tget(T, 2 * h + 1) != NT_RATE0) {
        const float c = pq_gt<FM>(v, b, (xl >> ((threadIdx.x & 31) & 3)) & 1u);
        if (plain) dump_lanes(child_pos(np, 1), c, 4);
        xr = dec4<FM, plain>(__shfl_sync(FULL, c, 0), __shfl_sync(FULL, c, 1), __shfl_sync(FULL, c, 2),
                      __shfl_sync(FULL, c, 3), T, 2 * h + 1, child_pos(np, 1));
    }
    UB_END(0);
    return (xl ^ xr) | (xr << 4);
}

template <int FM, bool plain>
__device__ __forceinline__ uint32_t dec16(float v, const TypeBits &T, int h, const NodePos &np)
{
    UB_BEGIN();
    const int lane = threadIdx.x & 31;
    uint32_t bits;
    if (!plain && lanes_special<FM>(v, 16, tget(T, h), bits)) {
        UB_END(6);
        return bits;
    }
    const float b = __shfl_down_sync(0xffffffffu, v, 8);
    uint32_t xl = 0, xr = 0;
    if (plain || tget(T, 2 * h) != NT_RATE0) {
        const float c = pq_f<FM>(v, b);
        if (plain) dump_lanes(child_pos(np, 0), c, 8);
        xl = dec8<FM, plain>(c, T, 2 * h, child_pos(np, 0));
    }
    if (plain || tget(T, 2 * h + 1) != NT_RATE0) {
        const float c = pq_gt<FM>(v, b, (xl >> (lane & 7)) & 1u);
        if (plain) dump_lanes(child_pos(np, 1), c, 8);
        xr = dec8<FM, plain>(c, T, 2 * h + 1, child_pos(np, 1));
    }
    UB_END(3);
    return (xl ^ xr) | (xr << 8);
}

template <int FM, bool plain>
__device__ __forceinline__ uint32_t dec32_body(float v, const TypeBits T, const NodePos np);
template <int FM, bool plain>
__device__ __noinline__ uint32_t dec32(float v, const TypeBits T, const NodePos np)
{
    UB_BEGIN();
    const uint32_t r = dec32_body<FM, plain>(v, T, np);
    UB_END(1);
    return r;
}
template <int FM, bool plain>
__device__ __forceinline__ uint32_t dec32_body(float v, const TypeBits T, const NodePos np)
{
    const int lane = threadIdx.x & 31;
    uint32_t bits;
    if (!plain && lanes_special<FM>(v, 32, tget(T, 1), bits)) return bits;
    const float b = __shfl_down_sync(0xffffffffu, v, 16);
    uint32_t xl = 0, xr = 0;
    if (plain || tget(T, 2) != NT_RATE0) {
        const float c = pq_f<FM>(v, b);
        if (plain) dump_lanes(child_pos(np, 0), c, 16);
        xl = dec16<FM, plain>(c, T, 2, child_pos(np, 0));
    }
    if (plain || tget(T, 3) != NT_RATE0) {
        const float c = pq_gt<FM>(v, b, (xl >> (lane & 15)) & 1u);
        if (plain) dump_lanes(child_pos(np, 1), c, 16);
        xr = dec16<FM, plain>(c, T, 3, child_pos(np, 1));
    }
    return (xl ^ xr) | (xr << 16);
}

// Load the TypeBits of the node at S-local heap index `root`, width W0 <= 32.
__device__ __forceinline__ TypeBits load_typebits(const uint8_t *ty, uint32_t root, int W0, bool plain)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int h0 = 32 / W0, k0 = ilog2((uint32_t)h0);
    uint32_t tint = NT_MIXED;
    if (lane >= h0) {
        const int k = ilog2((uint32_t)lane) - k0;  // relative depth below the root
        if (k >= 0 && (lane >> k) == h0) tint = ty[(root << k) + (uint32_t)(lane - (h0 << k))];
    }
    if (plain) tint = NT_MIXED;
    const uint8_t tl = lane < W0 ? ty[(root << ilog2((uint32_t)W0)) + (uint32_t)lane] : NT_RATE1;
    TypeBits T;
    T.tb0 = __ballot_sync(FULL, tint & 1u);
    T.tb1 = __ballot_sync(FULL, tint & 2u);
    T.leaf = __ballot_sync(FULL, tl == NT_RATE0);
    return T;
}

template <int FM, bool plain>
__device__ __forceinline__ uint32_t engine32_dispatch(float A, int W0, const TypeBits &T, const NodePos &np)
{
    if (W0 == 32) return dec32<FM, plain>(A, T, np);
    if (W0 == 16) return dec16<FM, plain>(A, T, 2, np);
    if (W0 == 8) return dec8<FM, plain>(A, T, 4, np);
    float x[4];
#pragma unroll
    for (int i = 0; i < 4; i++) x[i] = __shfl_sync(0xffffffffu, A, i);
    if (W0 == 4) return dec4<FM, plain>(x[0], x[1], x[2], x[3], T, 8, np);
    if (W0 == 2) return dec2<FM, plain>(x[0], x[1], T, 16, np);
    // W0 == 1: a single leaf
    return ((T.leaf & 1u) || !(x[0] < 0.0f)) ? 0u : 1u;
}

// Decode the node at S-local heap index `root` of width W0 <= 32 whose
// values are held one per lane in A (lane l = element l).  Returns its bits.
template <int FM>
__device__ __forceinline__ uint32_t engine32_body(float A, uint32_t root, int W0, const WarpCtx c)
{
    const TypeBits T = load_typebits(c.ty, root, W0, c.plain != 0);
    const int el = ilog2(root);
    NodePos np;
    np.dump = c.dump;
    np.N = c.N;
    np.d = c.dS + el;
    np.j = (c.jS << el) + (root - (1u << el));
    if (c.plain) return engine32_dispatch<FM, true>(A, W0, T, np);
    return engine32_dispatch<FM, false>(A, W0, T, np);
}

template <int FM>
__device__ __forceinline__ uint32_t engine32(float A, uint32_t root, int W0, const WarpCtx c)
{
    const long long pr_t0 = c.prof ? clock64() : 0;
    const uint32_t r = engine32_body<FM>(A, root, W0, c);
    if (c.prof && (threadIdx.x & 31) == 0) {
        c.prof[0] += clock64() - pr_t0;
        c.prof[1] += 1;
    }
    return r;
}

// ---------------------------------------------------------------------------
// bit-range helpers on packed partial sums

// write W (<= 64) bits at bit position pos of word array x (single thread)
__device__ __forceinline__ void put_bits(uint32_t *x, uint32_t pos, uint32_t W, uint64_t bits)
{
    if (W >= 32) {
        x[pos >> 5] = (uint32_t)bits;
        if (W == 64) x[(pos >> 5) + 1] = (uint32_t)(bits >> 32);
    } else {
        const uint32_t sh = pos & 31, m = ((1u << W) - 1u) << sh;
        uint32_t *w = x + (pos >> 5);
        *w = (*w & ~m) | (((uint32_t)bits << sh) & m);
    }
}

__device__ __forceinline__ uint32_t get_bit(const uint32_t *x, uint32_t pos) { return (x[pos >> 5] >> (pos & 31)) & 1u; }

// block-wide: zero W bits at pos (W >= 32: word aligned)
__device__ __forceinline__ void zero_bits_block(uint32_t *x, uint32_t pos, uint32_t W)
{
    if (W < 32) {
        if (threadIdx.x == 0) put_bits(x, pos, W, 0);
        return;
    }
    for (uint32_t w = threadIdx.x; w < W / 32; w += blockDim.x) x[(pos >> 5) + w] = 0;
}

// block-wide: bits[lpos .. lpos+W) ^= bits[lpos+W .. lpos+2W)
__device__ __forceinline__ void combine_block(uint32_t *x, uint32_t lpos, uint32_t W)
{
    if (W < 32) {
        if (threadIdx.x == 0) {
            uint32_t *w = x + (lpos >> 5);
            const uint32_t sh = lpos & 31, m = (1u << W) - 1u;
            const uint32_t r = (*w >> (sh + W)) & m;
            *w ^= r << sh;
        }
        return;
    }
    const uint32_t nw = W / 32, b = lpos >> 5;
    for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x) x[b + w] ^= x[b + nw + w];
}

// cluster-sliced word ranges of the global partial sums (W >= S >= 2048 bits,
// so every CTA of a cluster of <= 8 gets >= 8 words): words [b, b + nw) = 0,
// and words [b, b + nw) ^= words [b + nw, b + 2 nw)
// (16-byte accesses, four independent load pairs in flight per thread: one
// thread's words are dependent L2 round trips otherwise -- the combine steps
// were 10 % of the upper band's samples with the scalar loop)
// Out of line (PQ_COMBINE_OOL): inlined, the batched loads raise the kernel's
// register pressure and ptxas spills in the serial band (every config -10 %).
#ifndef PQ_COMBINE_V4
#define PQ_COMBINE_V4 1
#endif
#ifndef PQ_COMBINE_OOL
#define PQ_COMBINE_OOL 0
#endif
#ifndef PQ_COMBINE_U
#define PQ_COMBINE_U 1  // uint4 load pairs in flight per thread (2 or more: the serial band's compile degrades)
#endif
#if PQ_COMBINE_OOL
#define PQ_COMBINE_ATTR __noinline__
#else
#define PQ_COMBINE_ATTR __forceinline__
#endif
__device__ __forceinline__ void zero_words_slice(uint32_t *x, uint32_t b, uint32_t nw, uint32_t rank, uint32_t K)
{
    const uint32_t q = nw / K, w0 = rank * q;
    if (PQ_COMBINE_V4 && q % 4 == 0 && (reinterpret_cast<uintptr_t>(x + b + w0) & 15u) == 0) {  // else: the word loop
        uint4 *xa = reinterpret_cast<uint4 *>(x + b + w0);
        for (uint32_t i = threadIdx.x; i < q / 4; i += blockDim.x) xa[i] = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    for (uint32_t w = w0 + threadIdx.x; w < w0 + q; w += blockDim.x) x[b + w] = 0;
}
__device__ PQ_COMBINE_ATTR void combine_words_slice(uint32_t *x, uint32_t b, uint32_t nw, uint32_t rank, uint32_t K)
{
    const uint32_t q = nw / K, w0 = rank * q;
    if (PQ_COMBINE_V4 && q % 4 == 0 && (reinterpret_cast<uintptr_t>(x + b + w0) & 15u) == 0) {
        uint4 *xa = reinterpret_cast<uint4 *>(x + b + w0);
        const uint4 *xb = reinterpret_cast<const uint4 *>(x + b + nw + w0);
        const uint32_t q4 = q / 4, nthr = blockDim.x;
#pragma unroll 1
        for (uint32_t i0 = threadIdx.x; i0 < q4; i0 += PQ_COMBINE_U * nthr) {
            uint4 l[PQ_COMBINE_U], r[PQ_COMBINE_U];
#pragma unroll
            for (int k = 0; k < PQ_COMBINE_U; k++) {
                const uint32_t i = i0 + k * nthr;
                if (i < q4) {
                    l[k] = xa[i];
                    r[k] = xb[i];
                }
            }
#pragma unroll
            for (int k = 0; k < PQ_COMBINE_U; k++) {
                const uint32_t i = i0 + k * nthr;
                if (i < q4) xa[i] = make_uint4(l[k].x ^ r[k].x, l[k].y ^ r[k].y, l[k].z ^ r[k].z, l[k].w ^ r[k].w);
            }
        }
        return;
    }
    for (uint32_t w = w0 + threadIdx.x; w < w0 + q; w += blockDim.x) x[b + w] ^= x[b + nw + w];
}

__device__ __forceinline__ float block_min(float v, float *red)
{
    uint32_t m = __float_as_uint(v);
    m = __reduce_min_sync(0xffffffffu, m);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) ((uint32_t *)red)[warp] = m;
    __syncthreads();
    uint32_t r = lane < nw ? ((uint32_t *)red)[lane] : 0x7f800000u;
    r = __reduce_min_sync(0xffffffffu, r);
    return __uint_as_float(r);
}

// ---------------------------------------------------------------------------
// the per-frame tree walk

// One warp decodes the sub-tree rooted at (d0, j0), width 32 <= W0 <= 256,
// inside the shared-memory sub-tree: node values in the shared stage buffers
// (width W at st_end - 2W), partial sums in xs (bit position (jW) mod S).
// The walk is unrolled at compile time over the widths (walk_node<W> calls
// walk_node<W/2> for both children): no loop-carried (d, j) state, every
// per-lane element count is a constant, and the plain-SC/dump path is a
// separate instantiation, so the SSC path carries no dump checks.  Nodes of
// width 32 go to the register decoder dec32; wider ones take warp-synchronous
// f/g steps (<= 4 elements per lane, independent f's in flight).
struct WalkCtx {
    float *st_end;
    uint32_t *xs;
    const uint8_t *ty;
    float *dump;
    uint32_t N;
    int dS;
    uint32_t jS;
};

// absolute (depth, index) of the node at S-local heap index lh (dump only)
__device__ __forceinline__ NodePos walk_pos(const WalkCtx &c, uint32_t lh)
{
    const int e = ilog2(lh);
    NodePos np;
    np.dump = c.dump;
    np.N = c.N;
    np.d = c.dS + e;
    np.j = (c.jS << e) + (lh - (1u << e));
    return np;
}

template <int FM, bool PLAIN>
__device__ __forceinline__ void walk_leaf32(const WalkCtx &c, uint32_t lh, uint32_t pos)
{
    const int lane = threadIdx.x & 31;
    const float v = (c.st_end - 64)[lane];
    const TypeBits T = load_typebits(c.ty, lh, 32, PLAIN);
    NodePos np;
    if (PLAIN) {
        np = walk_pos(c, lh);
    } else {
        np.dump = nullptr;
        np.N = c.N;
        np.d = 0;
        np.j = 0;
    }
    const uint32_t bits = dec32<FM, PLAIN>(v, T, np);
    if (lane == 0) c.xs[pos >> 5] = bits;
    __syncwarp();
}

template <int FM, bool PLAIN, int W>
__device__ __forceinline__ void walk_node(const WalkCtx &c, uint32_t lh, uint32_t pos);

#ifndef PQ_WALK_NOINLINE
#define PQ_WALK_NOINLINE 0
#endif
// a child of the warp walk: one out-of-line copy per width (code size: the
// inlined recursion duplicates every level 2^k times)
template <int FM, bool PLAIN, int W>
__device__ __noinline__ void walk_child_ool(const WalkCtx c, uint32_t lh, uint32_t pos)
{
    walk_node<FM, PLAIN, W>(c, lh, pos);
}
template <int FM, bool PLAIN, int W>
__device__ __forceinline__ void walk_child(const WalkCtx &c, uint32_t lh, uint32_t pos)
{
    if constexpr (W == 32) walk_leaf32<FM, PLAIN>(c, lh, pos);
    else if constexpr (PQ_WALK_NOINLINE && !PLAIN) walk_child_ool<FM, PLAIN, W>(c, lh, pos);
    else walk_node<FM, PLAIN, W>(c, lh, pos);
}

template <int FM, bool PLAIN, int W>
__device__ __forceinline__ void walk_node(const WalkCtx &c, uint32_t lh, uint32_t pos)
{
    constexpr uint32_t V = W / 32, H = W / 2, Vh = V / 2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const float *nd = c.st_end - 2 * W;
    uint32_t *xw = c.xs + (pos >> 5);  // this node's partial-sum words (V of them)
    if (!PLAIN) {
        const uint8_t t = c.ty[lh];
        if (t == NT_RATE0) {
            if (lane < (int)V) xw[lane] = 0;
            __syncwarp();
            return;
        }
        if (t == NT_RATE1) {
            uint32_t m = 0x7f800000u;
#pragma unroll
            for (uint32_t q = 0; q < V; q++) m = min(m, __float_as_uint(nd[32 * q + lane]) & 0x7fffffffu);
            m = __reduce_min_sync(FULL, m);
            if (rate1_guard<FM>(__uint_as_float(m), ilog2(W))) {
#pragma unroll
                for (uint32_t q = 0; q < V; q++) {
                    const uint32_t bits = __ballot_sync(FULL, nd[32 * q + lane] < 0.0f);
                    if (lane == 0) xw[q] = bits;
                }
                __syncwarp();
                return;
            }
        }
        if (t == NT_REP) {
            // SC's g-chain with zero partial sums, in SC's pairing order
            float sm8[V];
#pragma unroll
            for (uint32_t q = 0; q < V; q++) sm8[q] = nd[32 * q + lane];
#pragma unroll
            for (uint32_t hv = V / 2; hv >= 1; hv >>= 1)
#pragma unroll
                for (uint32_t q = 0; q < hv; q++) sm8[q] = qadd<FM>(sm8[q + hv], sm8[q]);
            float s0 = sm8[0];
#pragma unroll
            for (int hh = 16; hh >= 1; hh >>= 1) s0 = qadd<FM>(__shfl_down_sync(FULL, s0, hh), s0);
            const uint32_t bits = __shfl_sync(FULL, s0, 0) < 0.0f ? FULL : 0u;
            if (lane < (int)V) xw[lane] = bits;
            __syncwarp();
            return;
        }
    }
    float *ch = c.st_end - W;  // stage buffer of both children
    // ---- left child: f-step unless it is rate-0
    if (!PLAIN && c.ty[2 * lh] == NT_RATE0) {
        if (lane < (int)Vh) xw[lane] = 0;
        __syncwarp();
    } else {
        float a[Vh], b[Vh];
#pragma unroll
        for (uint32_t q = 0; q < Vh; q++) {
            a[q] = nd[32 * q + lane];
            b[q] = nd[32 * q + lane + H];
        }
#pragma unroll
        for (uint32_t q = 0; q < Vh; q++) {
            const float v = pq_f<FM>(a[q], b[q]);
            ch[32 * q + lane] = v;
            if (PLAIN && c.dump) {
                const NodePos np = walk_pos(c, 2 * lh);
                c.dump[(size_t)np.d * c.N + (size_t)np.j * H + 32 * q + lane] = v;
            }
        }
        __syncwarp();
        walk_child<FM, PLAIN, H>(c, 2 * lh, pos);
    }
    // ---- right child: g-step with the left child's partial sums
    if (!PLAIN && c.ty[2 * lh + 1] == NT_RATE0) {
        if (lane < (int)Vh) xw[Vh + lane] = 0;
        __syncwarp();
    } else {
        float a[Vh], b[Vh];
        uint32_t sw[Vh];
#pragma unroll
        for (uint32_t q = 0; q < Vh; q++) {
            a[q] = nd[32 * q + lane];
            b[q] = nd[32 * q + lane + H];
            sw[q] = xw[q];
        }
#pragma unroll
        for (uint32_t q = 0; q < Vh; q++) {
            const float v = pq_gt<FM>(a[q], b[q], (sw[q] >> lane) & 1u);
            ch[32 * q + lane] = v;
            if (PLAIN && c.dump) {
                const NodePos np = walk_pos(c, 2 * lh + 1);
                c.dump[(size_t)np.d * c.N + (size_t)np.j * H + 32 * q + lane] = v;
            }
        }
        __syncwarp();
        walk_child<FM, PLAIN, H>(c, 2 * lh + 1, pos + H);
    }
    // ---- partial sums of this node: (xl ^ xr, xr)
    if (lane < (int)Vh) xw[lane] ^= xw[Vh + lane];
    __syncwarp();
}

template <int FM, bool PLAIN>
__device__ __forceinline__ void walk_root(const WalkCtx &c, uint32_t W, uint32_t lh, uint32_t pos)
{
    if (W == 512) walk_node<FM, PLAIN, 512>(c, lh, pos);
    else if (W == 256) walk_node<FM, PLAIN, 256>(c, lh, pos);
    else if (W == 128) walk_node<FM, PLAIN, 128>(c, lh, pos);
    else if (W == 64) walk_node<FM, PLAIN, 64>(c, lh, pos);
    else walk_leaf32<FM, PLAIN>(c, lh, pos);
}

template <int FM>
__device__ __noinline__ void warp_walk(float *st_end, uint32_t *xs, const uint8_t *ty, float *dump, uint32_t N,
                                       uint32_t S, int dS, uint32_t jS, int plain_i, int d0, uint32_t j0)
{
    WalkCtx c;
    c.st_end = st_end;
    c.xs = xs;
    c.ty = ty;
    c.dump = dump;
    c.N = N;
    c.dS = dS;
    c.jS = jS;
    const uint32_t W = N >> d0;
    const int e = d0 - dS;
    const uint32_t lh = (1u << e) + (j0 & ((1u << e) - 1u));
    const uint32_t pos = (j0 * W) & (S - 1);
    UB_BEGIN();
    if (plain_i) walk_root<FM, true>(c, W, lh, pos);
    else walk_root<FM, false>(c, W, lh, pos);
    UB_END(2);
}

// ---- register-resident warp walk (SSC path; plain mode and the stage dump
// keep warp_walk).  Lane l holds elements l + 32q of every node of width
// W >= 32 in registers; f/g steps are in-lane (no shared-memory round trip,
// no __syncwarp); partial sums travel as warp-uniform words returned by the
// children.  Node types of the walk's upper levels (widths W0 .. 32 below the
// root, relative heap positions 1..31) are two uniform bit masks built once
// per walk; REL (the relative heap position) is a template parameter, so
// every type test is a shift by a constant.
struct W2Ctx {
    const uint8_t *ty;  // S-local heap-order types (shared memory)
    uint32_t root;      // S-local heap index of the walk root
    uint32_t wb0, wb1;  // type bits of relative heap positions 1..31
    int k32;            // relative depth of the width-32 level below the root
};
template <int REL>
__device__ __forceinline__ uint32_t w2_type(const W2Ctx &c)
{
    return ((c.wb0 >> REL) & 1u) | (((c.wb1 >> REL) & 1u) << 1);
}

template <int FM, int W, int REL>
__device__ __forceinline__ void w2_node(const float (&x)[W / 32], const W2Ctx &c, uint32_t (&xo)[W / 32]);

// width-32 child at relative position REL: TypeBits from shared memory, then
// the register engine (lane l = element l)
template <int FM, int REL>
__device__ __forceinline__ uint32_t w2_leaf(float v, const W2Ctx &c)
{
    const uint32_t lh = (c.root << c.k32) + (uint32_t)REL - (1u << c.k32);
    const TypeBits T = load_typebits(c.ty, lh, 32, false);
    NodePos np;
    np.dump = nullptr;
    np.N = 0;
    np.d = 0;
    np.j = 0;
    return dec32<FM, false>(v, T, np);
}

template <int FM, int H, int REL>
__device__ __forceinline__ void w2_child(const float (&x)[H / 32], const W2Ctx &c, uint32_t (&xo)[H / 32])
{
    if constexpr (H == 32) xo[0] = w2_leaf<FM, REL>(x[0], c);
    else w2_node<FM, H, REL>(x, c, xo);
}

template <int FM, int W, int REL>
__device__ __forceinline__ void w2_node(const float (&x)[W / 32], const W2Ctx &c, uint32_t (&xo)[W / 32])
{
    constexpr int V = W / 32, Vh = V / 2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t t = w2_type<REL>(c);
    if (t == NT_RATE0) {
#pragma unroll
        for (int q = 0; q < V; q++) xo[q] = 0u;
        return;
    }
    if (t == NT_RATE1) {
        uint32_t m = 0x7f800000u;
#pragma unroll
        for (int q = 0; q < V; q++) m = min(m, __float_as_uint(x[q]) & 0x7fffffffu);
        m = __reduce_min_sync(FULL, m);
        if (rate1_guard<FM>(__uint_as_float(m), ilog2((uint32_t)W))) {
#pragma unroll
            for (int q = 0; q < V; q++) xo[q] = __ballot_sync(FULL, x[q] < 0.0f);
            return;
        }
    }
    if (t == NT_REP) {
        // SC's g-chain with zero partial sums, in SC's pairing order
        float sm8[V];
#pragma unroll
        for (int q = 0; q < V; q++) sm8[q] = x[q];
#pragma unroll
        for (int hv = V / 2; hv >= 1; hv >>= 1)
#pragma unroll
            for (int q = 0; q < hv; q++) sm8[q] = qadd<FM>(sm8[q + hv], sm8[q]);
        float s0 = sm8[0];
#pragma unroll
        for (int hh = 16; hh >= 1; hh >>= 1) s0 = qadd<FM>(__shfl_down_sync(FULL, s0, hh), s0);
        const uint32_t bits = __shfl_sync(FULL, s0, 0) < 0.0f ? FULL : 0u;
#pragma unroll
        for (int q = 0; q < V; q++) xo[q] = bits;
        return;
    }
    float ch[Vh];
    uint32_t xl[Vh], xr[Vh];
    if (w2_type<2 * REL>(c) == NT_RATE0) {
#pragma unroll
        for (int q = 0; q < Vh; q++) xl[q] = 0u;
    } else {
#pragma unroll
        for (int q = 0; q < Vh; q++) ch[q] = pq_f<FM>(x[q], x[q + Vh]);
        w2_child<FM, W / 2, 2 * REL>(ch, c, xl);
    }
    if (w2_type<2 * REL + 1>(c) == NT_RATE0) {
#pragma unroll
        for (int q = 0; q < Vh; q++) xr[q] = 0u;
    } else {
#pragma unroll
        for (int q = 0; q < Vh; q++) ch[q] = pq_gt<FM>(x[q], x[q + Vh], (xl[q] >> lane) & 1u);
        w2_child<FM, W / 2, 2 * REL + 1>(ch, c, xr);
    }
#pragma unroll
    for (int q = 0; q < Vh; q++) {
        xo[q] = xl[q] ^ xr[q];
        xo[Vh + q] = xr[q];
    }
}

template <int FM, int W>
__device__ __forceinline__ void w2_root(const float *nd, uint32_t *xw, const W2Ctx &c)
{
    constexpr int V = W / 32;
    const int lane = threadIdx.x & 31;
    float x[V];
    uint32_t xo[V];
#pragma unroll
    for (int q = 0; q < V; q++) x[q] = nd[32 * q + lane];
    w2_node<FM, W, 1>(x, c, xo);
#pragma unroll
    for (int q = 0; q < V; q++)
        if (lane == q) xw[q] = xo[q];
    __syncwarp();
}

// the SSC warp walk from the stage buffer of the root (width W, 64..512)
template <int FM>
__device__ __noinline__ void warp_walk2(float *st_end, uint32_t *xs, const uint8_t *ty, uint32_t S, int dS, int d0,
                                        uint32_t j0)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t W = S >> (d0 - dS);
    const int e = d0 - dS;
    W2Ctx c;
    c.ty = ty;
    c.root = (1u << e) + (j0 & ((1u << e) - 1u));
    c.k32 = ilog2(W) - 5;
    // types of relative heap positions 1..31 down to the width-32 level
    uint32_t tint = NT_MIXED;
    if (lane >= 1) {
        const int k = ilog2((uint32_t)lane);
        if (k <= c.k32) tint = ty[(c.root << k) + (uint32_t)lane - (1u << k)];
    }
    c.wb0 = __ballot_sync(FULL, tint & 1u);
    c.wb1 = __ballot_sync(FULL, tint & 2u);
    const float *nd = st_end - 2 * W;
    uint32_t *xw = xs + (((j0 * W) & (S - 1)) >> 5);
    UB_BEGIN();
    if (W == 512) w2_root<FM, 512>(nd, xw, c);
    else if (W == 256) w2_root<FM, 256>(nd, xw, c);
    else if (W == 128) w2_root<FM, 128>(nd, xw, c);
    else w2_root<FM, 64>(nd, xw, c);
    UB_END(2);
}

// ---- the widest warp-band levels (W = 1024, 2048: SSC path): one warp takes
// the node's f/g steps itself, from the shared-memory stage buffers (W/64 f's
// per lane per step, independent), and hands the 512-wide children to
// warp_walk2 -- no block barriers and no trip through the block-level main
// loop for these nodes
template <int FM, int W>
__device__ __forceinline__ void warp_wide(float *st_end, uint32_t *xs, const uint8_t *ty, uint32_t S, int dS, int d0,
                                          uint32_t j0)
{
    constexpr int V = W / 32, Vh = V / 2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int e = d0 - dS;
    const uint32_t lh = (1u << e) + (j0 & ((1u << e) - 1u));
    const float *nd = st_end - 2 * W;
    float *ch = st_end - W;
    uint32_t *xw = xs + (((j0 * W) & (S - 1)) >> 5);
    const uint8_t t = ty[lh], tl = ty[2 * lh], tr = ty[2 * lh + 1];
    if (t == NT_RATE0) {
        for (int q = lane; q < V; q += 32) xw[q] = 0u;
        __syncwarp();
        return;
    }
    if (t == NT_RATE1) {
        uint32_t m = 0x7f800000u;
#pragma unroll 8
        for (int q = 0; q < V; q++) m = min(m, __float_as_uint(nd[32 * q + lane]) & 0x7fffffffu);
        m = __reduce_min_sync(FULL, m);
        if (rate1_guard<FM>(__uint_as_float(m), ilog2((uint32_t)W))) {
            for (int q = 0; q < V; q++) {
                const uint32_t b = __ballot_sync(FULL, nd[32 * q + lane] < 0.0f);
                if (lane == 0) xw[q] = b;
            }
            __syncwarp();
            return;
        }
    }
    if (t == NT_REP) {
        // SC's g-chain with zero partial sums, in SC's pairing order
        float acc[V];
#pragma unroll
        for (int q = 0; q < V; q++) acc[q] = nd[32 * q + lane];
#pragma unroll
        for (int hv = V / 2; hv >= 1; hv >>= 1)
#pragma unroll
            for (int q = 0; q < hv; q++) acc[q] = qadd<FM>(acc[q + hv], acc[q]);
        float s0 = acc[0];
#pragma unroll
        for (int hh = 16; hh >= 1; hh >>= 1) s0 = qadd<FM>(__shfl_down_sync(FULL, s0, hh), s0);
        const uint32_t bits = __shfl_sync(FULL, s0, 0) < 0.0f ? FULL : 0u;
        for (int q = lane; q < V; q += 32) xw[q] = bits;
        __syncwarp();
        return;
    }
    // left child
    if (tl == NT_RATE0) {
        for (int q = lane; q < Vh; q += 32) xw[q] = 0u;
        __syncwarp();
    } else {
#pragma unroll 8
        for (int q = 0; q < Vh; q++) ch[32 * q + lane] = pq_f<FM>(nd[32 * q + lane], nd[32 * q + lane + W / 2]);
        __syncwarp();
        if constexpr (W / 2 > 512) warp_wide<FM, W / 2>(st_end, xs, ty, S, dS, d0 + 1, 2 * j0);
        else warp_walk2<FM>(st_end, xs, ty, S, dS, d0 + 1, 2 * j0);
    }
    // right child: g-step with the left child's partial sums
    if (tr == NT_RATE0) {
        for (int q = lane; q < Vh; q += 32) xw[Vh + q] = 0u;
        __syncwarp();
    } else {
#pragma unroll 8
        for (int q = 0; q < Vh; q++)
            ch[32 * q + lane] = pq_gt<FM>(nd[32 * q + lane], nd[32 * q + lane + W / 2], (xw[q] >> lane) & 1u);
        __syncwarp();
        if constexpr (W / 2 > 512) warp_wide<FM, W / 2>(st_end, xs, ty, S, dS, d0 + 1, 2 * j0 + 1);
        else warp_walk2<FM>(st_end, xs, ty, S, dS, d0 + 1, 2 * j0 + 1);
    }
    for (int q = lane; q < Vh; q += 32) xw[q] ^= xw[Vh + q];
    __syncwarp();
}

template <int FM>
__device__ __noinline__ void warp_wide_root(float *st_end, uint32_t *xs, const uint8_t *ty, uint32_t S, int dS,
                                            int d0, uint32_t j0)
{
    const uint32_t W = S >> (d0 - dS);
#if PQ_WIDE_WARP_LOG2 >= 13
    if (W == 8192) warp_wide<FM, 8192>(st_end, xs, ty, S, dS, d0, j0);
    else
#endif
#if PQ_WIDE_WARP_LOG2 >= 12
    if (W == 4096) warp_wide<FM, 4096>(st_end, xs, ty, S, dS, d0, j0);
    else
#endif
#if PQ_WIDE_WARP_LOG2 >= 11
    if (W == 2048) warp_wide<FM, 2048>(st_end, xs, ty, S, dS, d0, j0);
    else
#endif
    warp_wide<FM, 1024>(st_end, xs, ty, S, dS, d0, j0);
}

template <int FM>
__device__ __forceinline__ void warp_small(const float *src, bool chan, const DecParams &p, const FrameCtx &fc,
                                           uint32_t lh, const WarpCtx &wc, uint32_t *xs, uint32_t pos, int W)
{
    // W < 32 only happens for blocks shorter than 32 (the root itself)
    const int lane = threadIdx.x & 31;
    float v = 0.0f;
    if (lane < W) v = chan ? chan_load(p, fc, lane) : src[lane];
    const uint32_t bits = engine32<FM>(v, lh, W, wc);
    if (lane == 0) put_bits(xs, pos, W, bits);
}

// ---- upper band through a TMA ring.  A frame's upper band is one CTA (or
// cluster) streaming its stage vectors through HBM/L2; with register loads
// the bytes in flight per CTA -- and so the per-frame bandwidth -- are capped
// by registers (measured: latency-bound, ~17 GB/s per frame).  Instead one
// thread issues 1-D bulk copies (cp.async.bulk, the TMA engine) of C-element
// chunks of both operands (plus the bit words the step needs) into a ring of
// D stages in the shared-memory stage area (idle during upper steps), with
// an mbarrier per stage; the CTA consumes chunk c while chunks c+1..c+D-1
// are in flight.  Only steps whose output stays in global memory use it (the
// ring occupies the whole stage area); the f/g-steps into a width-S child
// keep the register path.

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// the same copy with an L2 evict-first policy: operands read for the last time
__device__ __forceinline__ void bulk_g2s_ef(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("{\n\t.reg .b64 pol;\n\t"
                 "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
                 "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async;" ::: "memory");
}

// one upper step's operands: A/B element vectors (fp32 stage or channel
// LLRs), or the channel's received bits; optional coset words; optional
// left-child partial sums (g-steps).  Offsets are element indices.
struct UpSrc {
    const float *a, *b;          // stage or fp32 channel halves (null: BSC bits)
    const short *a16, *b16;      // Q8.8 channel halves (fixed mode, int16 input), or null
    const uint32_t *ya, *yb;     // BSC received-bit halves (or null)
    const uint32_t *ca, *cb;     // coset words of the halves (or null)
    const uint32_t *xl;          // g-step: left-child partial sums (bit e of the range), or null
    bool chan;                   // operands are channel LLRs (quantise in fixed mode, coset flips)
};

struct Ring {
    uint64_t *bar;   // D mbarriers
    uint32_t *cnt;   // D counters: warps that have left the stage (PQ_RING_WARPREL)
    float *base;     // ring start in shared memory
    uint32_t C;      // elements per chunk (multiple of 256)
    uint32_t D;      // stages
    uint32_t sbytes; // bytes per stage
};

// stage layout: [A: C floats][B: C floats][ya][yb][ca][cb][xl] (C/32 words each)
#ifndef PQ_ST_EVICT_LAST
#define PQ_ST_EVICT_LAST 0
#endif
#ifndef PQ_F_EF_BYTES
#define PQ_F_EF_BYTES 0
#endif
#ifndef PQ_G_EVICT_FIRST
#define PQ_G_EVICT_FIRST 1
#endif
// ef: the stage operands are read for the last time (a g-step reads its
// parent node once, after the left sub-tree), so they are loaded evict-first
// and leave L2 to the children the next steps re-read
__device__ __forceinline__ uint32_t ring_bytes(const UpSrc &u, uint32_t C)
{
    const uint32_t wb = C / 8;  // bytes of C bits
    uint32_t bytes = 0;
    if (u.a) bytes += 8 * C;
    if (u.a16) bytes += 4 * C;
    if (u.ya) bytes += 2 * wb;
    if (u.ca) bytes += 2 * wb;
    if (u.xl) bytes += wb;
    return bytes;
}

// the bulk copies of one C-element chunk (operand offset e0) into the stage at st
__device__ __forceinline__ void ring_copies(const UpSrc &u, unsigned char *st, uint32_t C, uint32_t e0, uint64_t *bar,
                                            bool ef)
{
    const uint32_t wb = C / 8;
    if (u.a && ef) {
        bulk_g2s_ef(st, u.a + e0, 4 * C, bar);
        bulk_g2s_ef(st + 4 * C, u.b + e0, 4 * C, bar);
    } else if (u.a) {
        bulk_g2s(st, u.a + e0, 4 * C, bar);
        bulk_g2s(st + 4 * C, u.b + e0, 4 * C, bar);
    }
    if (u.a16) {
        bulk_g2s(st, u.a16 + e0, 2 * C, bar);
        bulk_g2s(st + 4 * C, u.b16 + e0, 2 * C, bar);
    }
    if (u.ya) {
        bulk_g2s(st + 8 * C, u.ya + e0 / 32, wb, bar);
        bulk_g2s(st + 8 * C + wb, u.yb + e0 / 32, wb, bar);
    }
    if (u.ca) {
        bulk_g2s(st + 8 * C + 2 * wb, u.ca + e0 / 32, wb, bar);
        bulk_g2s(st + 8 * C + 3 * wb, u.cb + e0 / 32, wb, bar);
    }
    if (u.xl) bulk_g2s(st + 8 * C + 4 * wb, u.xl + e0 / 32, wb, bar);
}

__device__ __forceinline__ void ring_issue(const Ring &r, const UpSrc &u, uint32_t e0, uint32_t s, bool ef = false)
{
    unsigned char *st = reinterpret_cast<unsigned char *>(r.base) + (size_t)s * r.sbytes;
    mbar_expect_tx(&r.bar[s], ring_bytes(u, r.C));
    ring_copies(u, st, r.C, e0, &r.bar[s], ef);
}

// what the ring steps need of DecParams (passed by value: the steps can be
// compiled out of line, PQ_RING_OOL)
struct ChanQ {
    float mag;
    int fixed;
};
#ifndef PQ_RING_OOL
#define PQ_RING_OOL 3
#endif

// four consecutive operands (k % 4 == 0) of one half from a landed stage
template <int FM>
__device__ __forceinline__ float4 ring_val4(const ChanQ &p, const UpSrc &u, const unsigned char *st,
                                            uint32_t C, int half, uint32_t k)
{
    const uint32_t wb = C / 8;
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(st + 8 * C + (2 + half) * wb);
    const uint32_t c4 = u.ca ? (cw[k >> 5] >> (k & 31)) & 15u : 0u;
    float4 v;
    if (u.ya) {
        const uint32_t *yw = reinterpret_cast<const uint32_t *>(st + 8 * C + half * wb);
        const uint32_t y4 = ((yw[k >> 5] >> (k & 31)) & 15u) ^ c4;
        v.x = (y4 & 1u) ? -p.mag : p.mag;
        v.y = (y4 & 2u) ? -p.mag : p.mag;
        v.z = (y4 & 4u) ? -p.mag : p.mag;
        v.w = (y4 & 8u) ? -p.mag : p.mag;
        return v;
    }
    if (u.a16) {
        const short4 q = *reinterpret_cast<const short4 *>(st + (size_t)half * 4 * C + 2 * k);
        v = make_float4((float)q.x, (float)q.y, (float)q.z, (float)q.w);
    } else {
        v = *reinterpret_cast<const float4 *>(st + (size_t)half * 4 * C + 4 * k);
    }
    if (u.chan) {
        if (p.fixed && !u.a16) {  // channel LLRs -> Q8.8 codes on load, as chan_load4
            v.x = fminf(fmaxf(rintf(v.x * 256.0f), -Q_MAX), Q_MAX);
            v.y = fminf(fmaxf(rintf(v.y * 256.0f), -Q_MAX), Q_MAX);
            v.z = fminf(fmaxf(rintf(v.z * 256.0f), -Q_MAX), Q_MAX);
            v.w = fminf(fmaxf(rintf(v.w * 256.0f), -Q_MAX), Q_MAX);
        }
        v.x = __uint_as_float(__float_as_uint(v.x) ^ ((c4 & 1u) << 31));
        v.y = __uint_as_float(__float_as_uint(v.y) ^ ((c4 & 2u) << 30));
        v.z = __uint_as_float(__float_as_uint(v.z) ^ ((c4 & 4u) << 29));
        v.w = __uint_as_float(__float_as_uint(v.w) ^ ((c4 & 8u) << 28));
    }
    return v;
}

// A warp is done with stage s.  PQ_RING_WARPREL = 0: a CTA barrier per chunk,
// thread 0 refills the stage.  1: no barrier -- every warp counts itself out
// of the stage (its reads ordered before the count) and the last one out
// refills it, so warps run ahead of each other by up to D - 1 chunks instead
// of all waiting for the slowest one at every chunk.
// PQ_RING_WARPREL / PQ_FUSE2: 0 = off, 1 = every kernel, 2 = the clustered kernels only
#ifndef PQ_RING_WARPREL
#define PQ_RING_WARPREL 0
#endif
#ifndef PQ_RING_UNROLL2
#define PQ_RING_UNROLL2 0
#endif
#define PQ_MODE_ON(mode, CL) ((mode) == 1 || ((mode) == 2 && (CL)))
template <bool WR, class Issue>
__device__ __forceinline__ void ring_release(const Ring &r, uint32_t s, bool more, Issue issue)
{
    if constexpr (WR) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
            __threadfence_block();
            const uint32_t old = atomicAdd(&r.cnt[s], 1u);
            if (old + 1 == (blockDim.x >> 5)) {
                r.cnt[s] = 0;
                __threadfence_block();
                if (more) issue();
            }
        }
    } else {
        __syncthreads();  // stage s fully consumed
        if (threadIdx.x == 0 && more) issue();
    }
}

// One upper step over output elements [lo, hi) of this CTA through the ring:
// f-step (IS_G = false) or g-step with the left child's partial sums.
// dst: the output stage vector (global, or shared memory for a width-S
// child).  All threads call it; thread 0 issues the copies.  ph holds the
// CTA-uniform parity bit of every stage's mbarrier.
// SCR = true: both operands are fp32 stage vectors (no channel input, coset
// or received-bit words) -- the common case, compiled without those branches
template <int FM, bool IS_G, bool SCR, bool WR>
__device__ __forceinline__ uint32_t ring_step_impl(const ChanQ p, const Ring r, const UpSrc u, float *dst, uint32_t lo,
                                                  uint32_t hi, uint32_t ph, bool ef_f)
{
    const uint32_t C = r.C, D = r.D, tid = threadIdx.x, nthr = blockDim.x;
    const bool ef = IS_G ? (bool)PQ_G_EVICT_FIRST : ef_f;
#if PQ_ST_EVICT_LAST
    // children are re-read by the next step: keep them in L2
    uint64_t st_pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(st_pol));
#endif
    const uint32_t nch = (hi - lo) / C;
    if (tid == 0)
        for (uint32_t c = 0; c < nch && c < D; c++) ring_issue(r, u, lo + c * C, c, ef);
    uint32_t s = 0;
    for (uint32_t c = 0; c < nch; c++) {
        PQ_JITTER();
        mbar_wait(&r.bar[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        const unsigned char *st = reinterpret_cast<const unsigned char *>(r.base) + (size_t)s * r.sbytes;
        const uint32_t e0 = lo + c * C;
        auto ld = [&](int half, uint32_t k) -> float4 {
            return SCR ? *reinterpret_cast<const float4 *>(st + (size_t)half * 4 * C + 4 * k)
                       : ring_val4<FM>(p, u, st, C, half, k);
        };
        auto sgn = [&](uint32_t k) -> uint32_t {
            const uint32_t *xw = reinterpret_cast<const uint32_t *>(st + 8 * C + 4 * (C / 8));
            return IS_G ? (xw[k >> 5] >> (k & 31)) & 15u : 0u;
        };
        auto comp = [&](const float4 &a, const float4 &b, uint32_t sb) -> float4 {
            float4 v;
            if (IS_G) {
                v.x = pq_gt<FM>(a.x, b.x, sb & 1u);
                v.y = pq_gt<FM>(a.y, b.y, sb & 2u);
                v.z = pq_gt<FM>(a.z, b.z, sb & 4u);
                v.w = pq_gt<FM>(a.w, b.w, sb & 8u);
            } else {
                v.x = pq_f<FM>(a.x, b.x);
                v.y = pq_f<FM>(a.y, b.y);
                v.z = pq_f<FM>(a.z, b.z);
                v.w = pq_f<FM>(a.w, b.w);
            }
            return v;
        };
        auto put = [&](uint32_t k, const float4 &v) {
#if PQ_ST_EVICT_LAST
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst + e0 + k), "f"(v.x),
                         "f"(v.y), "f"(v.z), "f"(v.w), "l"(st_pol)
                         : "memory");
#else
            *reinterpret_cast<float4 *>(dst + e0 + k) = v;
#endif
        };
        const uint32_t kstep = 4 * nthr;
        uint32_t k = 4 * tid;
#if PQ_RING_UNROLL2
        // two quads per thread in flight (all loads ahead of the stores: dst is a
        // generic pointer, so the compiler cannot move a load across a store)
#pragma unroll 1
        for (; k + kstep < C; k += 2 * kstep) {
            const float4 a0 = ld(0, k), b0 = ld(1, k), a1 = ld(0, k + kstep), b1 = ld(1, k + kstep);
            const uint32_t s0 = sgn(k), s1 = sgn(k + kstep);
            const float4 v0 = comp(a0, b0, s0), v1 = comp(a1, b1, s1);
            put(k, v0);
            put(k + kstep, v1);
        }
#endif
#pragma unroll 1
        for (; k < C; k += kstep) put(k, comp(ld(0, k), ld(1, k), sgn(k)));
        ring_release<WR>(r, s, c + D < nch, [&]() { ring_issue(r, u, lo + (c + D) * C, s, ef); });
        s = s + 1 == D ? 0 : s + 1;
    }
    return ph;
}

// Two upper steps in one pass (PQ_FUSE2): the step into a child of width 2*Hh
// (f-step, or g-step with the left sibling's partial sums) fused with the
// f-step into that child's left child.  Every child of the upper band is
// consumed by an f-step right after it is written; here the thread that
// computes child elements i and i + Hh (from four operand quads instead of
// two) also computes the grandchild element f(c[i], c[i + Hh]) from its
// registers, so the child is written once (the later g-step reads it) but
// never re-read by an f-step: a third of the level's stage bytes, one ring
// pass and its barriers less.  A stage holds two half-size sub-stages in the
// ordinary layout (chunk offsets e0 and e0 + Hh); [lo, hi) is this CTA's
// slice of the grandchild's index range.
#ifndef PQ_FUSE2
#define PQ_FUSE2 0
#endif
template <int FM, bool IS_G, bool SCR, bool WR>
__device__ __forceinline__ uint32_t ring_step2_impl(const ChanQ p, const Ring r, const UpSrc u, float *dst1, float *dst2,
                                                   uint32_t Hh, uint32_t lo, uint32_t hi, uint32_t ph)
{
    const uint32_t C2 = r.C / 2, D = r.D, tid = threadIdx.x, nthr = blockDim.x;
    const uint32_t sb2 = r.sbytes / 2;  // 8 C2 + 5 (C2 / 8)
    const bool ef = IS_G ? (bool)PQ_G_EVICT_FIRST : false;
    const uint32_t nch = (hi - lo) / C2;
    const uint32_t tx = 2 * ring_bytes(u, C2);
    auto issue = [&](uint32_t c, uint32_t s) {
        unsigned char *st = reinterpret_cast<unsigned char *>(r.base) + (size_t)s * r.sbytes;
        mbar_expect_tx(&r.bar[s], tx);
        ring_copies(u, st, C2, lo + c * C2, &r.bar[s], ef);
        ring_copies(u, st + sb2, C2, Hh + lo + c * C2, &r.bar[s], ef);
    };
    if (tid == 0)
        for (uint32_t c = 0; c < nch && c < D; c++) issue(c, c);
    uint32_t s = 0;
    for (uint32_t c = 0; c < nch; c++) {
        PQ_JITTER();
        mbar_wait(&r.bar[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        const unsigned char *st0 = reinterpret_cast<const unsigned char *>(r.base) + (size_t)s * r.sbytes;
        const unsigned char *st1 = st0 + sb2;
        const uint32_t e0 = lo + c * C2;
#pragma unroll 1
        for (uint32_t k = 4 * tid; k < C2; k += 4 * nthr) {
            const float4 a0 = SCR ? *reinterpret_cast<const float4 *>(st0 + 4 * k) : ring_val4<FM>(p, u, st0, C2, 0, k);
            const float4 b0 =
                SCR ? *reinterpret_cast<const float4 *>(st0 + 4 * (size_t)C2 + 4 * k) : ring_val4<FM>(p, u, st0, C2, 1, k);
            const float4 a1 = SCR ? *reinterpret_cast<const float4 *>(st1 + 4 * k) : ring_val4<FM>(p, u, st1, C2, 0, k);
            const float4 b1 =
                SCR ? *reinterpret_cast<const float4 *>(st1 + 4 * (size_t)C2 + 4 * k) : ring_val4<FM>(p, u, st1, C2, 1, k);
            float4 c0, c1, v;
            if (IS_G) {
                const uint32_t *xw0 = reinterpret_cast<const uint32_t *>(st0 + 8 * C2 + 4 * (C2 / 8));
                const uint32_t *xw1 = reinterpret_cast<const uint32_t *>(st1 + 8 * C2 + 4 * (C2 / 8));
                const uint32_t s0 = (xw0[k >> 5] >> (k & 31)) & 15u, s1 = (xw1[k >> 5] >> (k & 31)) & 15u;
                c0.x = pq_gt<FM>(a0.x, b0.x, s0 & 1u);
                c0.y = pq_gt<FM>(a0.y, b0.y, s0 & 2u);
                c0.z = pq_gt<FM>(a0.z, b0.z, s0 & 4u);
                c0.w = pq_gt<FM>(a0.w, b0.w, s0 & 8u);
                c1.x = pq_gt<FM>(a1.x, b1.x, s1 & 1u);
                c1.y = pq_gt<FM>(a1.y, b1.y, s1 & 2u);
                c1.z = pq_gt<FM>(a1.z, b1.z, s1 & 4u);
                c1.w = pq_gt<FM>(a1.w, b1.w, s1 & 8u);
            } else {
                c0.x = pq_f<FM>(a0.x, b0.x);
                c0.y = pq_f<FM>(a0.y, b0.y);
                c0.z = pq_f<FM>(a0.z, b0.z);
                c0.w = pq_f<FM>(a0.w, b0.w);
                c1.x = pq_f<FM>(a1.x, b1.x);
                c1.y = pq_f<FM>(a1.y, b1.y);
                c1.z = pq_f<FM>(a1.z, b1.z);
                c1.w = pq_f<FM>(a1.w, b1.w);
            }
            *reinterpret_cast<float4 *>(dst1 + e0 + k) = c0;
            *reinterpret_cast<float4 *>(dst1 + Hh + e0 + k) = c1;
            v.x = pq_f<FM>(c0.x, c1.x);
            v.y = pq_f<FM>(c0.y, c1.y);
            v.z = pq_f<FM>(c0.z, c1.z);
            v.w = pq_f<FM>(c0.w, c1.w);
            *reinterpret_cast<float4 *>(dst2 + e0 + k) = v;
        }
        ring_release<WR>(r, s, c + D < nch, [&]() { issue(c + D, s); });
        s = s + 1 == D ? 0 : s + 1;
    }
    return ph;
}

// The ring steps out of line (OOL) or inlined into the walk.  Out of line the
// kernel body is ~2000 instructions shorter and the serial engine inlined into
// it compiles a little better: c3 / c4 +1.5 %; the clustered kernels lose
// 1.2 % (c5), so PQ_RING_OOL = 3 takes it for the unclustered kernels only
// (0: never, 1: always).
template <int FM, bool IS_G, bool SCR, bool WR>
__device__ __noinline__ uint32_t ring_step_ool(const ChanQ p, const Ring r, const UpSrc u, float *dst, uint32_t lo,
                                               uint32_t hi, uint32_t ph, bool ef_f)
{
    return ring_step_impl<FM, IS_G, SCR, WR>(p, r, u, dst, lo, hi, ph, ef_f);
}
template <int FM, bool IS_G, bool SCR, bool WR, bool OOL>
__device__ __forceinline__ uint32_t ring_step(const ChanQ p, const Ring r, const UpSrc u, float *dst, uint32_t lo,
                                              uint32_t hi, uint32_t ph, bool ef_f = false)
{
    if constexpr (OOL) return ring_step_ool<FM, IS_G, SCR, WR>(p, r, u, dst, lo, hi, ph, ef_f);
    else return ring_step_impl<FM, IS_G, SCR, WR>(p, r, u, dst, lo, hi, ph, ef_f);
}
template <int FM, bool IS_G, bool SCR, bool WR>
__device__ __noinline__ uint32_t ring_step2_ool(const ChanQ p, const Ring r, const UpSrc u, float *dst1, float *dst2,
                                                uint32_t Hh, uint32_t lo, uint32_t hi, uint32_t ph)
{
    return ring_step2_impl<FM, IS_G, SCR, WR>(p, r, u, dst1, dst2, Hh, lo, hi, ph);
}
template <int FM, bool IS_G, bool SCR, bool WR, bool OOL>
__device__ __forceinline__ uint32_t ring_step2(const ChanQ p, const Ring r, const UpSrc u, float *dst1, float *dst2,
                                               uint32_t Hh, uint32_t lo, uint32_t hi, uint32_t ph)
{
    if constexpr (OOL) return ring_step2_ool<FM, IS_G, SCR, WR>(p, r, u, dst1, dst2, Hh, lo, hi, ph);
    else return ring_step2_impl<FM, IS_G, SCR, WR>(p, r, u, dst1, dst2, Hh, lo, hi, ph);
}

// ---- thread-block clusters: K CTAs share one frame's upper band
// (configs with fewer frames than SMs).  Every step on a node wider than S is
// split over the cluster's CTAs by contiguous slices and bracketed by a
// cluster barrier (release/acquire at cluster scope orders the global-memory
// stage buffers and partial sums between the CTAs); nodes of width <= S --
// the shared-memory and single-warp bands -- run on the leader CTA (rank 0)
// alone while the others wait at the next cluster barrier.
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// minimum over the cluster of one float per CTA (after a block_min)
__device__ __forceinline__ float cluster_min(float m, float *slot, uint32_t K)
{
    if (threadIdx.x == 0) *slot = m;
    cluster_sync_all();
    float r = m;
    for (uint32_t q = 0; q < K; q++) {
        uint32_t a = (uint32_t)__cvta_generic_to_shared(slot), ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(q));
        float v;
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
        r = fminf(r, v);
    }
    return r;
}

// DIAG = false: the production instantiation -- no plain-SC mode, stage dump
// or cycle profile in the code at all (a smaller, branch-free main loop: the
// serial band's code competes with it for the SM's instruction caches)
// NT = 512: one CTA per SM (clusters with frames x K <= SMs, e.g. c5): twice
// the warps for the upper band, whose per-CTA chunk work bounds it
// KC > 0: the cluster size as a compile-time constant (the fixed-point
// 512-thread kernels).  With K a run-time value the clustered body keeps a
// few more registers live and ptxas compiles se::w32 in its uniform-datapath
// form (660 instructions, 29 R2UR); with K constant it takes the vector form
// of the unclustered kernel (556): c5 12.25 -> 12.71 Gbit/s.
template <int FM, bool CL, bool DIAG, int NT, int KC = 0>
__global__ void __launch_bounds__(NT, NT == 512 ? 1 : 2) sc_decode_kernel(DecParams p)
{
    if (!DIAG) {
        p.plain = 0;
        p.dump = nullptr;
        p.prof = nullptr;
    }
    constexpr bool WR = PQ_MODE_ON(PQ_RING_WARPREL, CL), FUSE2 = PQ_MODE_ON(PQ_FUSE2, CL);
    constexpr bool ROOL = PQ_RING_OOL == 1 || (PQ_RING_OOL == 3 && !CL);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ float red[32];
    const uint32_t S = p.S, N = p.N;
#ifdef PQ_CHECKED
    {
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        for (uint32_t i = threadIdx.x; i < dyn / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem_raw)[i] = 0x7fc00001u;
        __syncthreads();
    }
#endif
    Smem sm;
    sm.st = (float *)smem_raw;
    sm.xs = (uint32_t *)(sm.st + 2 * S);
    const uint32_t SW = S >= 32 ? S / 32 : 1;
    sm.ty = (uint8_t *)(sm.xs + SW);
    sm.fm = (uint32_t *)(sm.ty + 2 * S);
    const bool se2 = FM == PQ_F_FIXED && PQ_SE2 && !p.plain && p.dump == nullptr;

    load_log_table();
    if (FM == PQ_F_FIXED) {
        for (int i = threadIdx.x; i < CORR_SMEM; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
        if (PQ_SE2) se::load_tables();
    }
    __syncthreads();
    const uint32_t K = !CL ? 1u : KC > 0 ? (uint32_t)KC : p.K;  // CL = false: compiled without slicing
    const uint32_t rank = blockIdx.x & (K - 1);  // CTA rank in the frame's cluster
    const bool lead = rank == 0;
    const uint32_t frame = blockIdx.x / K;
    __shared__ float cl_slot;
    FrameCtx fc;
    fc.llr = p.llr ? p.llr + (size_t)frame * N : nullptr;
    fc.l16 = p.llr16 ? p.llr16 + (size_t)frame * N : nullptr;
    fc.y = p.ybits ? p.ybits + (size_t)frame * p.wpf : nullptr;
    fc.cw = p.cw ? p.cw + (size_t)frame * p.wpf : nullptr;
    fc.scr = p.scr ? p.scr + (size_t)frame * N : nullptr;
    fc.X = p.X + (size_t)frame * p.wpf;
    fc.dump = p.dump ? p.dump + (size_t)frame * (p.n + 1) * N : nullptr;

    const int tid = threadIdx.x, nthr = blockDim.x;
    const int dS = p.n - p.log2S;  // depth of the shared-memory sub-tree roots
    // The narrow sub-trees are decoded by one warp.  Co-resident CTAs pick
    // different warps so that their serial work lands on different SM
    // sub-partitions (scheduler = hardware warp slot mod 4).
    __shared__ int lw_sh;
    if (tid == 0) {
        uint32_t ws;
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(ws));
        const uint32_t nw = (uint32_t)(nthr >> 5);
        lw_sh = (int)(((ws / nw) & 3u) % nw);
    }
    __syncthreads();
    const int lw = lw_sh;
    // nodes this wide or narrower: one warp (the SSC path also takes the
    // widest levels, 1024 / 2048, with warp_wide)
    const uint32_t wmax_eff = (!p.plain && p.dump == nullptr && p.wmax == 512u) ? (1u << PQ_WIDE_WARP_LOG2) : p.wmax;
    const uint32_t WMAX = S < wmax_eff ? S : wmax_eff;

    // TMA ring for the upper band (S >= 2048 so that chunks are >= 256 elements;
    // the stage dump keeps the register path)
    __shared__ __align__(8) uint64_t ring_bar[8];
    __shared__ uint32_t ring_cnt[8];
    const bool use_ring = S >= 2048 && p.dump == nullptr;
    uint32_t ring_ph = 0;
    if (use_ring) {
        if (tid == 0) {
            for (int q = 0; q < 8; q++) {
                mbar_init(&ring_bar[q], 1);
                ring_cnt[q] = 0;
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // PQ_RING_DEPTH stages of S/4-element chunks over the stage area (A/B-measured on
    // c3: chunk size matters -- S/8 was 8 % slower -- depth 2 vs 3 does not:
    // with every frame streaming, the upper band then runs near HBM peak)
    Ring ring;
    ring.bar = ring_bar;
    ring.cnt = ring_cnt;
    ring.C = S / 4;
    ring.sbytes = 8 * ring.C + 5 * (ring.C / 8);
    ring.D = WR ? 3 : 2;
    ring.base = sm.st;
    ChanQ cq;
    cq.mag = p.mag;
    cq.fixed = p.fixed;

    __shared__ unsigned long long eng_prof[4];
    if (tid < 4) eng_prof[tid] = 0;
    WarpCtx wc;
    wc.prof = p.prof ? eng_prof : nullptr;
    wc.ty = sm.ty;
    wc.dump = fc.dump;
    wc.N = N;
    wc.plain = p.plain;
    wc.dS = dS;
    wc.jS = 0;

    if (fc.dump)
        for (uint32_t i = tid; i < N; i += nthr) fc.dump[i] = chan_load(p, fc, i);

    // type of node (d, j): nodes strictly inside the loaded sub-tree come from
    // shared memory, everything else from the global heap-order table
    auto ntype = [&](int d, uint32_t j) -> uint8_t {
        const uint32_t W = N >> d;
        uint8_t t;
        if (W < S) {
            const int e = d - dS;
            t = sm.ty[(1u << e) + (j & ((1u << e) - 1u))];
        } else {
            t = __ldg(p.types + ((size_t)1 << d) + j);
        }
        return t;
    };
    auto xptr = [&](uint32_t W) -> uint32_t * { return W <= S ? sm.xs : fc.X; };
    auto xpos = [&](uint32_t W, uint32_t pos) -> uint32_t { return W <= S ? (pos & (S - 1)) : pos; };

    // barrier before a step on data wider than S: the whole cluster when K > 1
    auto wsync = [&](bool wide) {
        if (K > 1 && wide) cluster_sync_all();
        else __syncthreads();
    };
    // this CTA's slice [lo, hi) of a range of L elements (L / K a multiple of 32)
    auto slice_lo = [&](uint32_t L) -> uint32_t { return rank * (L / K); };
    // may the step into the width-Wc child (dc, jc) of type tc be fused with the
    // f-step into its left child?  Both outputs stay in the global stage buffers,
    // the child is neither skipped (rate-0) nor guarded first (rate-1), its
    // left child is not rate-0, and a half chunk still feeds every thread.
    auto fuse2_ok = [&](uint32_t Wc, uint8_t tc, int dc, uint32_t jc) -> bool {
        return !p.plain && Wc / 2 > S && ring.C / 2 >= 4u * (uint32_t)nthr && tc != NT_RATE0 && tc != NT_RATE1 &&
               ntype(dc + 1, 2 * jc) != NT_RATE0;
    };

    int d = 0;
    uint32_t j = 0;
    bool entering = true;
    // profile: thread 0 charges the cycles since the previous mark to the class
    // of the step that just ran (every step starts behind a barrier)
    unsigned long long pr_acc[PQ_PROF_SLOTS];
    unsigned long long pr_last = 0, pr_start = 0;
    int pr_cls = PR_SM_OTHER;
    const bool prof = p.prof != nullptr && lead && tid == 32 * lw;  // the lower-band warp's lane 0
    if (prof) {
        for (int q = 0; q < PQ_PROF_SLOTS; q++) pr_acc[q] = 0;
        pr_start = pr_last = clock64();
    }
#define PROF_MARK(cls)                                         \
    do {                                                       \
        if (prof) {                                            \
            const unsigned long long now_ = clock64();         \
            pr_acc[pr_cls] += now_ - pr_last;                  \
            pr_last = now_;                                    \
            pr_cls = (cls);                                    \
        }                                                      \
    } while (0)
    for (;;) {
        PQ_JITTER();
        const uint32_t W = N >> d;
        if (entering) {
            if (!lead && W <= S) {  // the leader decodes it; wait at the next cluster barrier
                entering = false;
                continue;
            }
            uint8_t t = ntype(d, j);
            if (p.plain && W > 1) t = NT_MIXED;
            if (t == NT_RATE0) {
                PROF_MARK(W > S ? PR_UP_OTHER : PR_SM_OTHER);
                wsync(W > S);
                if (W > S) zero_words_slice(fc.X, (j * W) >> 5, W >> 5, rank, K);
                else zero_bits_block(xptr(W), xpos(W, j * W), W);
                entering = false;
                continue;
            }
            if (W == S) {
                wc.jS = j;
                PROF_MARK(PR_TYPES);
                // entering a shared-memory sub-tree: stage its node types
                __syncthreads();
                // the fixed-point serial engine reads node types down to the
                // width-32 level only (below it the frozen-mask words): S / 16
                // bytes instead of 2 S
                const uint32_t qlim = se2 && S >= 32 ? S / 16 : 2 * S;
                if (S >= 128) {
                    // levels e >= 4 are 16-byte aligned runs in both layouts: copy
                    // them as uint4 (4 loads per thread at S = 8192 instead of 64)
                    if (tid < 15 && 1 + tid < qlim) {
                        const uint32_t q = 1 + tid;
                        const int e = 31 - __clz(q);
                        sm.ty[q] = __ldg(p.types + ((size_t)1 << (dS + e)) + ((size_t)j << e) + (q - (1u << e)));
                    }
                    for (uint32_t c = tid; 16 + 16 * c < qlim; c += nthr) {
                        const uint32_t q = 16 + 16 * c;
                        const int e = 31 - __clz(q);
                        const uint4 *src = reinterpret_cast<const uint4 *>(
                            p.types + ((size_t)1 << (dS + e)) + ((size_t)j << e) + (q - (1u << e)));
                        *reinterpret_cast<uint4 *>(sm.ty + q) = __ldg(src);
                    }
                } else {
                    for (uint32_t q = 1 + tid; q < qlim; q += nthr) {
                        const int e = 31 - __clz(q);
                        sm.ty[q] = __ldg(p.types + ((size_t)1 << (dS + e)) + ((size_t)j << e) + (q - (1u << e)));
                    }
                }
                if (se2 && S >= 32)
                    for (uint32_t w = tid; w < S / 32; w += nthr) sm.fm[w] = __ldg(p.fmask + (size_t)j * (S / 32) + w);
                __syncthreads();  // the types are read right below (before the next step's barrier)
            }
            if (W <= WMAX) {
                PROF_MARK(PR_WARP);
                if (prof) pr_acc[PR_NODES_WARP]++;
                __syncthreads();
                if ((tid >> 5) == lw) {
                    const bool chan = d == 0;
                    const int e = d - dS;
                    const uint32_t lh = (1u << e) + (j & ((1u << e) - 1u));
                    const uint32_t pos = (j * W) & (S - 1);
                    if (W >= 32) {
                        if (chan) {  // whole block <= 256: stage the channel LLRs once
                            float *dst = stage_ptr(p, fc, sm, W);
                            for (uint32_t i = tid & 31; i < W; i += 32) dst[i] = chan_load(p, fc, i);
                            __syncwarp();
                        }
#ifndef PQ_WALK2
#define PQ_WALK2 1
#endif
                        if (se2)
                            se::root<(CL || SE_SP_ALL) && (SE_W32_NPAT > 0)>(sm.st + 2 * S, sm.xs, sm.ty, sm.fm, S, dS, d, j);
                        else if (!p.plain && fc.dump == nullptr && W > 512)
                            warp_wide_root<FM>(sm.st + 2 * S, sm.xs, sm.ty, S, dS, d, j);
                        else if (PQ_WALK2 && !p.plain && fc.dump == nullptr && W >= 64)
                            warp_walk2<FM>(sm.st + 2 * S, sm.xs, sm.ty, S, dS, d, j);
                        else
                            warp_walk<FM>(sm.st + 2 * S, sm.xs, sm.ty, fc.dump, N, S, dS, wc.jS, p.plain, d, j);
                    } else {
                        const float *src = chan ? nullptr : stage_ptr(p, fc, sm, W);
                        warp_small<FM>(src, chan, p, fc, lh, wc, sm.xs, pos, (int)W);
                    }
                }
                entering = false;
                continue;
            }
            const float *src = d == 0 ? nullptr : stage_ptr(p, fc, sm, W);
            if (t == NT_RATE1 && !p.plain) {
                PROF_MARK(PR_RATE1);
                wsync(W > S);
                const bool split = K > 1 && W > S;
                const uint32_t lo = split ? slice_lo(W) : 0, hi = split ? lo + W / K : W;
                // one pass: min |L| and, speculatively, the hard decisions (the
                // node's own partial-sum words; a failed guard decodes the node
                // normally, which rewrites them).  Each warp takes 256 elements
                // (8 words) per iteration, all 8 loads in flight.
                float m = __int_as_float(0x7f800000);
                uint32_t *xb = xptr(W);
                const uint32_t base = xpos(W, j * W) >> 5;
                {
                    const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
#pragma unroll 1
                    for (uint32_t i0 = lo + 256u * wid; i0 < hi; i0 += 256u * nw) {
                        float v[8];
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const uint32_t i = i0 + 32u * q + lane;
                            v[q] = i < hi ? (d == 0 ? chan_load(p, fc, i) : src[i]) : __int_as_float(0x7f800000);
                        }
                        uint32_t word = 0;
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            m = fminf(m, fabsf(v[q]));
                            const uint32_t b = __ballot_sync(0xffffffffu, v[q] < 0.0f);
                            if (lane == q) word = b;
                        }
                        if (lane < 8 && i0 + 32u * lane < hi) xb[base + ((i0 + 32u * lane) >> 5)] = word;
                    }
                }
                m = block_min(m, red);
                if (split) m = cluster_min(m, &cl_slot, K);
                int k = 0;
                for (uint32_t w = W; w > 1; w >>= 1) k++;
                if (rate1_guard<FM>(m, k)) {
                    entering = false;
                    continue;
                }
            }
            // mixed node: f-step into the left child unless it is rate-0
            const uint32_t H = W / 2;
            const uint8_t tl = p.plain ? NT_MIXED : ntype(d + 1, 2 * j);
            PROF_MARK(W > S ? PR_UP_F : PR_SM_F);
            if (prof) pr_acc[PR_NODES_BLOCK]++;
            // every writer orders its generic-proxy stores before the barrier that
            // precedes the ring's bulk (async-proxy) reads of them
            if (use_ring && H > S) fence_proxy_async();
            wsync(W > S);
            if (tl == NT_RATE0) {
                if (H > S) zero_words_slice(fc.X, (2 * j * H) >> 5, H >> 5, rank, K);
                else if (lead) zero_bits_block(xptr(H), xpos(H, 2 * j * H), H);
                d++;
                j = 2 * j;
                entering = false;
                continue;
            }
            float *dst = stage_ptr(p, fc, sm, H);
            float *dmp = fc.dump ? fc.dump + (size_t)(d + 1) * N + (size_t)(2 * j) * H : nullptr;
            // f-step, 4 consecutive elements per thread (H >= 256 here, so every
            // chunk is a whole float4)
            const bool ch0 = d == 0;
            // a child wider than S is split over the cluster; one of width S
            // lands in the leader's shared memory and is the leader's alone
            const bool fsplit = K > 1 && H > S;
            const uint32_t flo = fsplit ? slice_lo(H) : 0, fhi = fsplit ? flo + H / K : H;
            if (!lead && !fsplit) {
                // nothing for this CTA
            } else if (use_ring && H > S) {
                UpSrc u;
                memset(&u, 0, sizeof u);
                if (ch0) {
                    u.chan = true;
                    if (fc.l16) {
                        u.a16 = fc.l16;
                        u.b16 = fc.l16 + H;
                    } else if (fc.llr) {
                        u.a = fc.llr;
                        u.b = fc.llr + H;
                    } else {
                        u.ya = fc.y;
                        u.yb = fc.y + H / 32;
                    }
                    if (fc.cw) {
                        u.ca = fc.cw;
                        u.cb = fc.cw + H / 32;
                    }
                } else {
                    u.a = src;
                    u.b = src + H;
                }
                // the parent's g-step re-read comes after its whole left
                // sub-tree: when the level's parents outgrow L2 it cannot
                // hit, so the f-step reads them evict-first as well
                const bool f_ef = PQ_F_EF_BYTES > 0 && (uint64_t)8 * H * (gridDim.x / K) > (uint64_t)PQ_F_EF_BYTES;
                // the child is consumed by an f-step right away: both steps in one pass
                if constexpr (FUSE2) {
                    if (fuse2_ok(H, tl, d + 1, 2 * j)) {
                        const uint32_t Hh = H / 2;
                        const uint32_t lo2 = fsplit ? slice_lo(Hh) : 0, hi2 = fsplit ? lo2 + Hh / K : Hh;
                        float *dst2 = stage_ptr(p, fc, sm, Hh);
                        if (ch0) ring_ph = ring_step2<FM, false, false, WR, ROOL>(cq, ring, u, dst, dst2, Hh, lo2, hi2, ring_ph);
                        else ring_ph = ring_step2<FM, false, true, WR, ROOL>(cq, ring, u, dst, dst2, Hh, lo2, hi2, ring_ph);
                        d += 2;
                        j = 4 * j;
                        continue;
                    }
                }
                if (ch0) ring_ph = ring_step<FM, false, false, WR, ROOL>(cq, ring, u, dst, flo, fhi, ring_ph, f_ef);
                else ring_ph = ring_step<FM, false, true, WR, ROOL>(cq, ring, u, dst, flo, fhi, ring_ph, f_ef);
            } else if (!ch0 && W > S && (fhi - flo) % (8 * nthr) == 0) {
                // from HBM/L2: two chunks per thread in flight
#pragma unroll 1
                for (uint32_t i = flo + 4 * tid; i < fhi; i += 8 * nthr) {
                    const uint32_t i2 = i + 4 * nthr;
                    const float4 a = *reinterpret_cast<const float4 *>(src + i);
                    const float4 b = *reinterpret_cast<const float4 *>(src + i + H);
                    const float4 a2 = *reinterpret_cast<const float4 *>(src + i2);
                    const float4 b2 = *reinterpret_cast<const float4 *>(src + i2 + H);
                    float4 v, v2;
                    v.x = pq_f<FM>(a.x, b.x);
                    v.y = pq_f<FM>(a.y, b.y);
                    v.z = pq_f<FM>(a.z, b.z);
                    v.w = pq_f<FM>(a.w, b.w);
                    *reinterpret_cast<float4 *>(dst + i) = v;
                    v2.x = pq_f<FM>(a2.x, b2.x);
                    v2.y = pq_f<FM>(a2.y, b2.y);
                    v2.z = pq_f<FM>(a2.z, b2.z);
                    v2.w = pq_f<FM>(a2.w, b2.w);
                    *reinterpret_cast<float4 *>(dst + i2) = v2;
                    if (dmp) {
                        *reinterpret_cast<float4 *>(dmp + i) = v;
                        *reinterpret_cast<float4 *>(dmp + i2) = v2;
                    }
                }
            } else if (!ch0) {  // stage operands: no channel branches in the loop
#pragma unroll 1
                for (uint32_t i = flo + 4 * tid; i < fhi; i += 4 * nthr) {
                    const float4 a = *reinterpret_cast<const float4 *>(src + i);
                    const float4 b = *reinterpret_cast<const float4 *>(src + i + H);
                    float4 v;
                    v.x = pq_f<FM>(a.x, b.x);
                    v.y = pq_f<FM>(a.y, b.y);
                    v.z = pq_f<FM>(a.z, b.z);
                    v.w = pq_f<FM>(a.w, b.w);
                    *reinterpret_cast<float4 *>(dst + i) = v;
                    if (dmp) *reinterpret_cast<float4 *>(dmp + i) = v;
                }
            } else {
#pragma unroll 1
                for (uint32_t i = flo + 4 * tid; i < fhi; i += 4 * nthr) {
                    const float4 a = chan_load4(p, fc, i);
                    const float4 b = chan_load4(p, fc, i + H);
                    float4 v;
                    v.x = pq_f<FM>(a.x, b.x);
                    v.y = pq_f<FM>(a.y, b.y);
                    v.z = pq_f<FM>(a.z, b.z);
                    v.w = pq_f<FM>(a.w, b.w);
                    *reinterpret_cast<float4 *>(dst + i) = v;
                    if (dmp) *reinterpret_cast<float4 *>(dmp + i) = v;
                }
            }
            d++;
            j = 2 * j;
            continue;
        }
        // ---- node (d, j) is decided; its partial sums are in place
        if (W == S && S < N) {
            PROF_MARK(PR_UP_OTHER);
            __syncthreads();
            if (lead)
                for (uint32_t w = tid; w < S / 32; w += nthr) fc.X[(j * S) / 32 + w] = sm.xs[w];
        }
        if (d == 0) {
            if (S >= N) {
                __syncthreads();
                if (N >= 32) {
                    for (uint32_t w = tid; w < N / 32; w += nthr) fc.X[w] = sm.xs[w];
                } else if (tid == 0) {
                    fc.X[0] = sm.xs[0] & ((1u << N) - 1u);
                }
            }
            PROF_MARK(PR_SM_OTHER);
            if (prof) {
                pr_acc[PR_TOTAL] = clock64() - pr_start;
                pr_acc[12] = eng_prof[0];
                pr_acc[13] = eng_prof[1];
                pr_acc[14] = eng_prof[2];
                for (int q = 0; q < PQ_PROF_SLOTS; q++) p.prof[(size_t)frame * PQ_PROF_SLOTS + q] = pr_acc[q];
            }
            if (K > 1) cluster_sync_all();  // no CTA exits while a peer may read its shared memory
            break;
        }
        if ((j & 1) == 0) {
            // left child done -> g-step at the parent into the right child
            const uint32_t jr = j + 1;
            const uint8_t tr = p.plain ? NT_MIXED : ntype(d, jr);
            PROF_MARK(2 * W > S ? PR_UP_G : PR_SM_G);
            if (use_ring && W > S) fence_proxy_async();
            wsync(2 * W > S);
            if (tr == NT_RATE0) {
                if (W > S) zero_words_slice(fc.X, (jr * W) >> 5, W >> 5, rank, K);
                else if (lead) zero_bits_block(xptr(W), xpos(W, jr * W), W);
                j = jr;
                continue;  // still exiting: the right child is decided
            }
            const uint32_t W2 = 2 * W;
            const float *src = d - 1 == 0 ? nullptr : stage_ptr(p, fc, sm, W2);
            const uint32_t *xl = xptr(W);
            const uint32_t lpos = xpos(W, j * W);
            float *dst = stage_ptr(p, fc, sm, W);
            float *dmp = fc.dump ? fc.dump + (size_t)d * N + (size_t)jr * W : nullptr;
            const bool ch0 = d - 1 == 0;
            const bool gsplit = K > 1 && W > S;
            const uint32_t glo = gsplit ? slice_lo(W) : 0, ghi = gsplit ? glo + W / K : (lead ? W : 0);
            const bool gring = use_ring && W > S;
            if (gring && ghi > glo) {
                UpSrc u;
                memset(&u, 0, sizeof u);
                if (ch0) {
                    u.chan = true;
                    if (fc.l16) {
                        u.a16 = fc.l16;
                        u.b16 = fc.l16 + W;
                    } else if (fc.llr) {
                        u.a = fc.llr;
                        u.b = fc.llr + W;
                    } else {
                        u.ya = fc.y;
                        u.yb = fc.y + W / 32;
                    }
                    if (fc.cw) {
                        u.ca = fc.cw;
                        u.cb = fc.cw + W / 32;
                    }
                } else {
                    u.a = src;
                    u.b = src + W;
                }
                u.xl = fc.X + (j * W) / 32;  // the left child's bits (a width-S child's were copied out)
                if constexpr (FUSE2) {
                    if (fuse2_ok(W, tr, d, jr)) {
                        const uint32_t Hh = W / 2;
                        const uint32_t lo2 = gsplit ? slice_lo(Hh) : 0, hi2 = gsplit ? lo2 + Hh / K : Hh;
                        float *dst2 = stage_ptr(p, fc, sm, Hh);
                        if (ch0) ring_ph = ring_step2<FM, true, false, WR, ROOL>(cq, ring, u, dst, dst2, Hh, lo2, hi2, ring_ph);
                        else ring_ph = ring_step2<FM, true, true, WR, ROOL>(cq, ring, u, dst, dst2, Hh, lo2, hi2, ring_ph);
                        d += 1;
                        j = 2 * jr;
                        entering = true;
                        continue;
                    }
                }
                if (ch0) ring_ph = ring_step<FM, true, false, WR, ROOL>(cq, ring, u, dst, glo, ghi, ring_ph);
                else ring_ph = ring_step<FM, true, true, WR, ROOL>(cq, ring, u, dst, glo, ghi, ring_ph);
            }
            // g-step: W >= 256 here; 4 elements per thread, 4 chunks in flight
            // (the operand loads are unswitched on the channel case)
#pragma unroll 1
            for (uint32_t base = glo; base < (gring ? glo : ghi); base += 16 * nthr) {
                float4 a[4], b[4];
                uint32_t sb[4];
                if (!ch0) {
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t i = base + 4 * (tid + k * nthr);
                        if (i < ghi) {
                            a[k] = *reinterpret_cast<const float4 *>(src + i);
                            b[k] = *reinterpret_cast<const float4 *>(src + i + W);
                            sb[k] = (xl[(lpos + i) >> 5] >> ((lpos + i) & 31)) & 15u;
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const uint32_t i = base + 4 * (tid + k * nthr);
                        if (i < ghi) {
                            a[k] = chan_load4(p, fc, i);
                            b[k] = chan_load4(p, fc, i + W);
                            sb[k] = (xl[(lpos + i) >> 5] >> ((lpos + i) & 31)) & 15u;
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t i = base + 4 * (tid + k * nthr);
                    if (i < ghi) {
                        float4 v;
                        v.x = pq_gt<FM>(a[k].x, b[k].x, sb[k] & 1u);
                        v.y = pq_gt<FM>(a[k].y, b[k].y, sb[k] & 2u);
                        v.z = pq_gt<FM>(a[k].z, b[k].z, sb[k] & 4u);
                        v.w = pq_gt<FM>(a[k].w, b[k].w, sb[k] & 8u);
                        *reinterpret_cast<float4 *>(dst + i) = v;
                        if (dmp) *reinterpret_cast<float4 *>(dmp + i) = v;
                    }
                }
            }
            j = jr;
            entering = true;
            continue;
        }
        // right child done -> parent's partial sums = (xl ^ xr, xr)
        PROF_MARK(2 * W > S ? PR_UP_OTHER : PR_SM_OTHER);
        wsync(2 * W > S);
        if (2 * W > S) combine_words_slice(fc.X, ((j - 1) * W) >> 5, W >> 5, rank, K);
        else combine_block(xptr(2 * W), xpos(2 * W, (j - 1) * W), W);
        d--;
        j >>= 1;
    }
}

// ---------------------------------------------------------------------------
// polar transform on packed frames (XOR butterflies)
// x = u F^{(x)n}: for h = 1, 2, ..., N/2 and i with (i & h) == 0: v[i] ^= v[i+h]
// Pass 1: within a tile of TW <= 1024 words (intra-word stages by mask/shift,
// cross-word stages in shared memory).  Pass 2: the remaining stages across
// tiles, as a column transform with row stride TW.

__device__ __forceinline__ uint32_t intra_word_transform(uint32_t v, uint32_t nbits)
{
    if (nbits > 1) v ^= (v >> 1) & 0x55555555u;
    if (nbits > 2) v ^= (v >> 2) & 0x33333333u;
    if (nbits > 4) v ^= (v >> 4) & 0x0f0f0f0fu;
    if (nbits > 8) v ^= (v >> 8) & 0x00ff00ffu;
    if (nbits > 16) v ^= (v >> 16) & 0x0000ffffu;
    return v;
}

struct XfParams {
    const uint32_t *in;
    uint32_t *out;
    const uint32_t *and_mask;  // [wpf] applied on load (shared by frames), or null
    const uint32_t *xor_post;  // [F][wpf] XORed into the output of the final pass, or null
    uint32_t wpf, TW, nbits_word;
    int final_pass;
};

__global__ void __launch_bounds__(256) xf_pass1(XfParams p)
{
    extern __shared__ uint32_t tile[];
    const uint32_t tiles_per_frame = p.wpf / p.TW;
    const uint32_t frame = blockIdx.x / tiles_per_frame, t = blockIdx.x % tiles_per_frame;
    const size_t base = (size_t)frame * p.wpf + (size_t)t * p.TW;
    for (uint32_t w = threadIdx.x; w < p.TW; w += blockDim.x) {
        uint32_t v = p.in[base + w];
        if (p.and_mask) v &= p.and_mask[t * p.TW + w];
        tile[w] = intra_word_transform(v, p.nbits_word);
    }
    for (uint32_t h = 1; h < p.TW; h <<= 1) {
        __syncthreads();
        for (uint32_t w = threadIdx.x; w < p.TW; w += blockDim.x)
            if ((w & h) == 0) tile[w] ^= tile[w + h];
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < p.TW; w += blockDim.x) {
        uint32_t v = tile[w];
        if (p.nbits_word < 32) v &= (1u << p.nbits_word) - 1u;
        if (p.final_pass && p.xor_post) v ^= p.xor_post[base + w];
        p.out[base + w] = v;
    }
}

// rows R = wpf / TW; each CTA owns 32 adjacent columns of one frame
__global__ void __launch_bounds__(256) xf_pass2(XfParams p)
{
    extern __shared__ uint32_t colbuf[];  // [R][32]
    const uint32_t R = p.wpf / p.TW, cgroups = p.TW / 32;
    const uint32_t frame = blockIdx.x / cgroups, cg = blockIdx.x % cgroups;
    const size_t fbase = (size_t)frame * p.wpf + (size_t)cg * 32;
    const uint32_t lane = threadIdx.x & 31, rw = threadIdx.x >> 5, nrw = blockDim.x >> 5;
    for (uint32_t r = rw; r < R; r += nrw) colbuf[r * 32 + lane] = p.out[fbase + (size_t)r * p.TW + lane];
    for (uint32_t h = 1; h < R; h <<= 1) {
        __syncthreads();
        for (uint32_t r = rw; r < R; r += nrw)
            if ((r & h) == 0) colbuf[r * 32 + lane] ^= colbuf[(r + h) * 32 + lane];
    }
    __syncthreads();
    for (uint32_t r = rw; r < R; r += nrw) {
        uint32_t v = colbuf[r * 32 + lane];
        if (p.xor_post) v ^= p.xor_post[fbase + (size_t)r * p.TW + lane];
        p.out[fbase + (size_t)r * p.TW + lane] = v;
    }
}

template <int FM>
__global__ void fmag_kernel(const float *a, const float *b, float *out, int n)
{
    load_log_table();
    if (FM == PQ_F_FIXED)
        for (int i = threadIdx.x; i < CORR_SMEM; i += blockDim.x) pq_corrtab[i] = CORR_TAB_C[i];
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = pq_f<FM>(a[i], b[i]);
}

__global__ void xor_words(const uint32_t *a, const uint32_t *b, uint32_t *out, size_t nwords)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nwords; i += (size_t)gridDim.x * blockDim.x)
        out[i] = a[i] ^ b[i];
}

__global__ void xor_masked(uint32_t *u, const uint32_t *v, const uint32_t *mask, uint32_t wpf, size_t nwords)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nwords; i += (size_t)gridDim.x * blockDim.x)
        u[i] ^= v[i] & mask[i % wpf];
}

static int launch_transform(const uint32_t *in, uint32_t *out, int n, int frames, const uint32_t *and_mask,
                            const uint32_t *xor_post, cudaStream_t st, int *launches)
{
    const uint32_t N = 1u << n;
    const uint32_t wpf = N >= 32 ? N / 32 : 1;
    XfParams p;
    p.in = in;
    p.out = out;
    p.and_mask = and_mask;
    p.xor_post = xor_post;
    p.wpf = wpf;
    p.TW = wpf < 1024 ? wpf : 1024;
    p.nbits_word = N >= 32 ? 32 : N;
    const bool two = wpf > p.TW;
    p.final_pass = two ? 0 : 1;
    const uint32_t tiles = wpf / p.TW;
    xf_pass1<<<(unsigned)(frames * tiles), 256, p.TW * 4, st>>>(p);
    CUDA_TRY(cudaGetLastError());
    (*launches)++;
    if (two) {
        const uint32_t R = wpf / p.TW;
        const size_t smem = (size_t)R * 32 * 4;
        if (smem > 227 * 1024) return set_err(-1, "polar transform: n=%d too large", n);
        CUDA_TRY(cudaFuncSetAttribute(xf_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        p.in = out;
        p.final_pass = 1;
        xf_pass2<<<(unsigned)(frames * (p.TW / 32)), 256, smem, st>>>(p);
        CUDA_TRY(cudaGetLastError());
        (*launches)++;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// host side

#define PQ_TIMING_SLOTS 64

struct pq_decoder {
    int n, max_frames, fmode, device, ssc, log2S_opt;
    uint32_t N, wpf;
    int have_mask;
    int sm_count;
    uint8_t *d_types;
    uint32_t *d_mask;
    uint32_t *d_cw;
    uint32_t *d_x;
    float *d_scr;
    size_t scr_elems;
    size_t ws_bytes;
    int last_launches;
    int profile;
    int warp_log2;
    int cluster_opt;  // PQ_OPT_CLUSTER: 0 = auto, else CTAs per frame
    int threads_opt;  // PQ_OPT_THREADS: 0 = auto, else 128 or 256 threads per CTA
    int last_K;       // CTAs per frame of the last decode launch
    int last_log2S, last_threads;
    unsigned long long *d_prof;
    int timing;                       // PQ_OPT_TIMING
    cudaEvent_t ev[2 * PQ_TIMING_SLOTS];  // kernel start/end events (created on first use)
    int n_timed;                      // decodes timed since the option was set
};

// CTAs per frame: split the upper band of a frame over a thread-block cluster
// when frames alone leave SMs idle (e.g. c5: 32 frames on 148 SMs -> 4 CTAs
// per frame).  Only with an upper band and S >= 2048 (every cluster slice of a
// wide node is then >= 512 elements / 16 words).
static int choose_K(const pq_decoder *h, int frames, int log2S, bool dump)
{
    if (dump || ((uint32_t)1 << log2S) >= h->N || log2S < 11) return 1;
    if (h->cluster_opt > 0) return h->cluster_opt;
    int K = 1;
    while (K < 8 && (size_t)frames * K * 2 <= (size_t)h->sm_count) K *= 2;
    return K;
}

template <int FM>
static int launch_dec(const DecParams &p, int frames, int nthreads, size_t smem, cudaStream_t st)
{
#ifdef PQ_NO_DECODE_KERNELS
    // microbenchmarks that include this file for its device functions only
    return set_err(-1, "built without the decode kernels");
#else
    const bool diag = p.plain || p.dump || p.prof;
    if (p.K == 1) {
        auto kern = diag ? sc_decode_kernel<FM, false, true, 256> : sc_decode_kernel<FM, false, false, 256>;
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<frames, nthreads, smem, st>>>(p);
        CUDA_TRY(cudaGetLastError());
        return 0;
    }
    auto ckern = diag ? sc_decode_kernel<FM, true, true, 256>
                      : nthreads == 512 ? sc_decode_kernel<FM, true, false, 512> : sc_decode_kernel<FM, true, false, 256>;
#ifndef PQ_NO_KC
    if (FM == PQ_F_FIXED && !diag && nthreads == 512) {  // cluster size compiled in (see sc_decode_kernel)
        if (p.K == 2) ckern = sc_decode_kernel<FM, true, false, 512, (FM == PQ_F_FIXED ? 2 : 0)>;
        else if (p.K == 4) ckern = sc_decode_kernel<FM, true, false, 512, (FM == PQ_F_FIXED ? 4 : 0)>;
        else if (p.K == 8) ckern = sc_decode_kernel<FM, true, false, 512, (FM == PQ_F_FIXED ? 8 : 0)>;
    }
#endif
    CUDA_TRY(cudaFuncSetAttribute(ckern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3((unsigned)frames * p.K, 1, 1);
    cfg.blockDim = dim3(nthreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, ckern, p));
    return 0;
#endif
}

// threads per CTA: 256 when frames leave <= 2 per SM (latency: a frame's
// block steps get 8 warps), else 128 (throughput: the 128-register kernel then
// fits 4 CTAs -- 4 serial warps, one per SM sub-partition -- per SM)
static int choose_threads(const pq_decoder *h, int frames)
{
    if (h->threads_opt) return h->threads_opt;
    // (64 -- 8 two-warp CTAs per SM, one wave for c2's 1024 frames -- measured
    // 4 % slower than 128 on c2: the upper band loses more than the wave gains)
    return frames > 2 * h->sm_count ? 128 : 256;
}

static int choose_log2S(const pq_decoder *h, int frames, int nthreads)
{
    const int lo = h->n < 6 ? h->n : 6;  // warp sub-trees (W <= 64) must sit inside S
    if (h->log2S_opt > 0) {
        int k = h->log2S_opt < h->n ? h->log2S_opt : h->n;
        return k < lo ? lo : k;
    }
    // resident CTAs per SM (the kernel's 128 registers per thread cap them)
    const int cap = nthreads == 64 ? 8 : nthreads == 128 ? 4 : 2;
    int per_sm = (frames + h->sm_count - 1) / h->sm_count;
    if (per_sm > cap) per_sm = cap;
    if (per_sm < 1) per_sm = 1;
    int best = 6;
    for (int k = 6; k <= 14; k++) {
        const size_t S = (size_t)1 << k;
        // dynamic (stage LLRs, partial sums, types, frozen-mask words) + static
        // (tables, barriers; the fixed-point serial engine's 4 KB byte table)
        const size_t bytes = 8 * S + (S / 32) * 8 + 2 * S + 10 * 1024 + (h->fmode == PQ_F_FIXED ? 4096 : 0);
        if ((size_t)per_sm * bytes <= 226 * 1024) best = k;
    }
    if (best > h->n) best = h->n;
    return best;
}

static size_t dec_smem_bytes(uint32_t S)
{
    const uint32_t SW = S >= 32 ? S / 32 : 1;
    return (size_t)8 * S + (size_t)SW * 4 + (size_t)2 * S + (size_t)SW * 4;
}

// Q8.8 phi table and the fixed-point rate-1 thresholds, computed
// on the host (double-precision libm, rounded to nearest) and uploaded once
// per device.  oracle/sc_oracle.c builds the same table the same way.
static void fixed_tables(float *corr, float *tau)
{
    int C[4097];
    for (int k = 0; k <= 4096; k++) {
        C[k] = (int)lrint(log1p(exp(-(double)k / 256.0)) * 256.0);
        corr[k] = (float)C[k];
    }
    for (int k = CORR_SMEM - 1; k <= 4096; k++) assert(C[k] == 0);  // the shared copy's clamp is exact
    // L(a) = min over b >= a of |f(a, b)| = max(0, a + min_d (C[2a + d] - C[d]))
    // (d = b - a; both indices clamp at 4096, so d <= 4096 covers every b)
    std::vector<int> L(32768);
    for (int a = 0; a < 32768; a++) {
        int best = INT_MAX;
        if (2 * a >= 4096) {
            best = C[4096] - C[0];
        } else {
            for (int d = 0; d <= 4096; d++) best = std::min(best, C[std::min(2 * a + d, 4096)] - C[d]);
        }
        L[a] = std::max(0, a + best);
    }
    for (int a = 32766; a >= 0; a--) L[a] = std::min(L[a], L[a + 1]);  // suffix min: non-decreasing
    auto chain = [&](int t, int k) {
        for (int i = 0; i < k; i++) t = L[t];
        return t;
    };
    for (int k = 0; k < 26; k++) {
        if (chain(32767, k) < 1) {
            tau[k] = 1e30f;  // never take the shortcut
            continue;
        }
        int lo = 0, hi = 32767;  // chain(hi) >= 1; find the smallest such t
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (chain(mid, k) >= 1) hi = mid;
            else lo = mid;
        }
        tau[k] = (float)hi;
    }
}

static int ensure_fixed_tables()
{
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    static std::mutex mu;
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lock(mu);  // one upload per device, whatever the host threads
    if (dev < 64 && done[dev]) return 0;
    static float corr[4097];
    float tau[26];
    fixed_tables(corr, tau);
    CUDA_TRY(cudaMemcpyToSymbol(CORR_TAB_C, corr, sizeof corr));
    CUDA_TRY(cudaMemcpyToSymbol(RATE1_TAU_FIX, tau, sizeof tau));
    int taui[26];
    for (int k = 0; k < 26; k++) taui[k] = tau[k] > 1e9f ? INT_MAX : (int)tau[k];
    CUDA_TRY(cudaMemcpyToSymbol(se::TAUI, taui, sizeof taui));
    // pageable uploads may return before the DMA lands; a decode on a
    // non-blocking stream is not ordered after them, so wait here once
    CUDA_TRY(cudaDeviceSynchronize());
    if (dev < 64) done[dev] = true;
    return 0;
}

// Select `dev` for the calling host thread and restore the caller's device on
// scope exit (every C-ABI entry that touches a handle's device uses one).
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
#define DEVICE_GUARD(dev)                                                                          \
    DeviceGuard dg_(dev);                                                                          \
    if (dg_.err != cudaSuccess)                                                                    \
        return set_err(1 + (int)dg_.err, "cudaSetDevice(%d): %s", (int)(dev), cudaGetErrorString(dg_.err))

// error text for the other translation units of the library (verify.cu)
int pq_set_error_text(int code, const char *msg) { return set_err(code, "%s", msg); }

extern "C" {

const char *pq_last_error(void) { return g_last_error.c_str(); }
int pq_abi_version(void) { return PQ_ABI_VERSION; }

int pq_decoder_create(pq_decoder **out, int n, int max_frames, int f_mode, int device)
{
    if (!out) return set_err(-1, "out is NULL");
    *out = nullptr;
    if (n < 1 || n > 25) return set_err(-1, "n must be in [1, 25], got %d", n);
    if (max_frames < 1) return set_err(-1, "max_frames must be >= 1, got %d", max_frames);
    if (f_mode != PQ_F_EXACT && f_mode != PQ_F_MINSUM && f_mode != PQ_F_FAST && f_mode != PQ_F_FIXED)
        return set_err(-1, "unknown f mode %d", f_mode);
    DEVICE_GUARD(device);
    pq_decoder *h = new pq_decoder();
    h->n = n;
    h->max_frames = max_frames;
    h->fmode = f_mode;
    h->device = device;
    h->ssc = 1;
    h->log2S_opt = 0;
    h->warp_log2 = 9;
    h->N = 1u << n;
    h->wpf = h->N >= 32 ? h->N / 32 : 1;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        delete h;
        return set_err(1 + (int)e, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
    }
    h->sm_count = prop.multiProcessorCount;
    const size_t wbytes = (size_t)max_frames * h->wpf * 4;
    h->scr_elems = (size_t)max_frames * h->N;
    size_t total = 0;
#define ALLOC(ptr, bytes)                                                                  \
    do {                                                                                   \
        e = cudaMalloc((void **)&(ptr), (bytes));                                          \
        if (e != cudaSuccess) {                                                            \
            pq_decoder_destroy(h);                                                         \
            return set_err(1 + (int)e, "cudaMalloc(%zu): %s", (size_t)(bytes), cudaGetErrorString(e)); \
        }                                                                                  \
        total += (bytes);                                                                  \
    } while (0)
    ALLOC(h->d_types, (size_t)2 * h->N);
    ALLOC(h->d_mask, (size_t)h->wpf * 4);
    ALLOC(h->d_cw, wbytes);
    ALLOC(h->d_x, wbytes);
    ALLOC(h->d_scr, h->scr_elems * 4);
#undef ALLOC
    h->ws_bytes = total;
    *out = h;
    return 0;
}

int pq_decoder_destroy(pq_decoder *h)
{
    if (!h) return 0;
    cudaFree(h->d_types);
    cudaFree(h->d_mask);
    cudaFree(h->d_cw);
    cudaFree(h->d_x);
    cudaFree(h->d_scr);
    cudaFree(h->d_prof);
    for (int i = 0; i < 2 * PQ_TIMING_SLOTS; i++)
        if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    delete h;
    return 0;
}

size_t pq_decoder_workspace_bytes(const pq_decoder *h) { return h ? h->ws_bytes : 0; }
int pq_decoder_last_launches(const pq_decoder *h) { return h ? h->last_launches : 0; }
int pq_decoder_last_ctas_per_frame(const pq_decoder *h) { return h ? h->last_K : 0; }

int pq_decoder_kernel_times(pq_decoder *h, float *ms_out, int count)
{
    if (!h || !ms_out) return set_err(-1, "NULL argument");
    const int avail = h->n_timed < PQ_TIMING_SLOTS ? h->n_timed : PQ_TIMING_SLOTS;
    if (count < 0 || count > avail)
        return set_err(-1, "count=%d outside [0, %d] (decodes timed since PQ_OPT_TIMING was set)", count, avail);
    DEVICE_GUARD(h->device);
    for (int i = 0; i < count; i++) {
        const int slot = (h->n_timed - count + i) % PQ_TIMING_SLOTS;
        CUDA_TRY(cudaEventSynchronize(h->ev[2 * slot + 1]));
        CUDA_TRY(cudaEventElapsedTime(&ms_out[i], h->ev[2 * slot], h->ev[2 * slot + 1]));
    }
    return 0;
}

int pq_decoder_last_config(const pq_decoder *h, int *log2S, int *threads_per_cta, int *ctas_per_frame)
{
    if (!h) return set_err(-1, "handle is NULL");
    if (log2S) *log2S = h->last_log2S;
    if (threads_per_cta) *threads_per_cta = h->last_threads;
    if (ctas_per_frame) *ctas_per_frame = h->last_K;
    return 0;
}

#ifdef PQ_UBENCH_TIMING
// instrumented builds only (tools/ub_profile.py): per-slot cycles and calls
int pq_debug_ub(unsigned long long *out, int reset)
{
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out, g_ub_time, sizeof(unsigned long long) * 16));
    CUDA_TRY(cudaMemcpyFromSymbol(out + 16, g_ub_count, sizeof(unsigned long long) * 16));
    if (reset) {
        unsigned long long z[16] = {0};
        CUDA_TRY(cudaMemcpyToSymbol(g_ub_time, z, sizeof z));
        CUDA_TRY(cudaMemcpyToSymbol(g_ub_count, z, sizeof z));
    }
    return 0;
}
#endif

int pq_decoder_set_option(pq_decoder *h, int key, int value)
{
    if (!h) return set_err(-1, "handle is NULL");
    switch (key) {
    case PQ_OPT_SSC: h->ssc = value ? 1 : 0; return 0;
    case PQ_OPT_SUBTREE_LOG2:
        if (value != 0 && (value < 1 || value > 14)) return set_err(-1, "subtree log2 must be 0 or 1..14");
        h->log2S_opt = value;
        return 0;
    case PQ_OPT_FMODE:
        if (value != PQ_F_EXACT && value != PQ_F_MINSUM && value != PQ_F_FAST && value != PQ_F_FIXED)
            return set_err(-1, "unknown f mode %d", value);
        h->fmode = value;
        return 0;
    case PQ_OPT_WARP_LOG2:
        if (value < 5 || value > 9) return set_err(-1, "warp band log2 width must be in 5..9");
        h->warp_log2 = value;
        return 0;
    case PQ_OPT_THREADS:
        if (value != 0 && value != 64 && value != 128 && value != 256)
            return set_err(-1, "threads must be 0 (auto), 64, 128 or 256");
        h->threads_opt = value;
        return 0;
    case PQ_OPT_CLUSTER:
        if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
            return set_err(-1, "cluster size must be 0 (auto), 1, 2, 4 or 8");
        h->cluster_opt = value;
        return 0;
    case PQ_OPT_TIMING:
        if (value && !h->ev[0]) {
            DEVICE_GUARD(h->device);
            for (int i = 0; i < 2 * PQ_TIMING_SLOTS; i++) CUDA_TRY(cudaEventCreate(&h->ev[i]));
        }
        h->timing = value ? 1 : 0;
        h->n_timed = 0;
        return 0;
    case PQ_OPT_PROFILE:
        if (value && !h->d_prof) {
            cudaError_t e = cudaMalloc((void **)&h->d_prof, (size_t)h->max_frames * PQ_PROF_SLOTS * 8);
            if (e != cudaSuccess) return set_err(1 + (int)e, "cudaMalloc(profile): %s", cudaGetErrorString(e));
            cudaMemset(h->d_prof, 0, (size_t)h->max_frames * PQ_PROF_SLOTS * 8);
        }
        h->profile = value ? 1 : 0;
        return 0;
    default: return set_err(-1, "unknown option %d", key);
    }
}

int pq_decoder_read_profile(const pq_decoder *h, unsigned long long *out, int frames)
{
    if (!h || !out) return set_err(-1, "NULL argument");
    if (!h->d_prof) return set_err(-1, "profiling was never enabled (PQ_OPT_PROFILE)");
    if (frames < 0 || frames > h->max_frames) return set_err(-1, "bad frame count");
    CUDA_TRY(cudaMemcpy(out, h->d_prof, (size_t)frames * PQ_PROF_SLOTS * 8, cudaMemcpyDeviceToHost));
    return 0;
}

int pq_decoder_get_option(const pq_decoder *h, int key)
{
    if (!h) return set_err(-1, "handle is NULL");
    switch (key) {
    case PQ_OPT_SSC: return h->ssc;
    case PQ_OPT_SUBTREE_LOG2: return h->log2S_opt;
    case PQ_OPT_FMODE: return h->fmode;
    case PQ_OPT_PROFILE: return h->profile;
    case PQ_OPT_WARP_LOG2: return h->warp_log2;
    case PQ_OPT_CLUSTER: return h->cluster_opt;
    case PQ_OPT_THREADS: return h->threads_opt;
    case PQ_OPT_TIMING: return h->timing;
    default: return set_err(-1, "unknown option %d", key);
    }
}

int pq_decoder_set_frozen_mask(pq_decoder *h, const uint8_t *mask)
{
    if (!h || !mask) return set_err(-1, "NULL argument");
    const uint32_t N = h->N;
    // node types, heap order: index (1 << d) + j for node j at depth d
    std::vector<uint8_t> ty(2 * (size_t)N, NT_MIXED);
    std::vector<uint32_t> nfrozen(2 * (size_t)N);
    std::vector<uint8_t> lastinfo(2 * (size_t)N);
    for (uint32_t i = 0; i < N; i++) {
        if (mask[i] > 1) return set_err(-1, "frozen mask entries must be 0 or 1 (index %u)", i);
        const size_t q = N + i;
        nfrozen[q] = mask[i];
        lastinfo[q] = mask[i] ? 0 : 1;
        ty[q] = mask[i] ? NT_RATE0 : NT_RATE1;
    }
    for (size_t q = N - 1; q >= 1; q--) {
        const size_t l = 2 * q, r = 2 * q + 1;
        const uint32_t W = (uint32_t)(N >> (31 - __builtin_clz((uint32_t)q)));
        nfrozen[q] = nfrozen[l] + nfrozen[r];
        lastinfo[q] = lastinfo[r];
        if (nfrozen[q] == W) ty[q] = NT_RATE0;
        else if (nfrozen[q] == 0) ty[q] = NT_RATE1;
        else if (nfrozen[q] == W - 1 && lastinfo[q]) ty[q] = NT_REP;
        else ty[q] = NT_MIXED;
    }
    ty[0] = NT_MIXED;
    std::vector<uint32_t> words(h->wpf, 0);
    for (uint32_t i = 0; i < N; i++)
        if (mask[i]) words[i >> 5] |= 1u << (i & 31);
    DEVICE_GUARD(h->device);
    CUDA_TRY(cudaMemcpy(h->d_types, ty.data(), ty.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(h->d_mask, words.data(), words.size() * 4, cudaMemcpyHostToDevice));
    h->have_mask = 1;
    return 0;
}

int pq_polar_transform(const uint32_t *in, uint32_t *out, int n, int frames, void *stream)
{
    if (n < 1 || n > 25) return set_err(-1, "n must be in [1, 25], got %d", n);
    if (frames < 0) return set_err(-1, "frames must be >= 0");
    if (frames == 0) return 0;
    if (!in || !out) return set_err(-1, "NULL pointer");
    int launches = 0;
    return launch_transform(in, out, n, frames, nullptr, nullptr, (cudaStream_t)stream, &launches);
}

static int decode_impl(pq_decoder *h, const float *llr, const uint32_t *ybits, float mag,
                       const uint32_t *frozen_u, uint32_t *u_hat, uint32_t *x_hat, float *dump,
                       int frames, void *stream, const short *llr16 = nullptr)
{
    if (!h) return set_err(-1, "handle is NULL");
    if (!h->have_mask) return set_err(-1, "frozen mask not set (pq_decoder_set_frozen_mask)");
    if (frames < 0 || frames > h->max_frames)
        return set_err(-1, "frames=%d outside [0, max_frames=%d]", frames, h->max_frames);
    if (!llr && !ybits && !llr16) return set_err(-1, "no channel input");
    if (frames == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    DEVICE_GUARD(h->device);
    int launches = 0;
    const uint32_t *cw = nullptr;
    if (frozen_u) {
        int rc = launch_transform(frozen_u, h->d_cw, h->n, frames, h->d_mask, nullptr, st, &launches);
        if (rc) return rc;
        cw = h->d_cw;
    }
    DecParams p;
    memset(&p, 0, sizeof p);
    p.n = h->n;
    int nthreads = choose_threads(h, frames);
    p.log2S = choose_log2S(h, frames, nthreads);
    p.plain = (dump || !h->ssc) ? 1 : 0;
    p.frames = frames;
    p.N = h->N;
    p.S = 1u << p.log2S;
    p.wpf = h->wpf;
    p.llr = llr;
    p.llr16 = llr16;
    p.ybits = ybits;
    p.mag = mag;
    p.cw = cw;
    p.types = h->d_types;
    p.fmask = h->d_mask;
    p.scr = h->d_scr;
    p.X = h->d_x;
    p.dump = dump;
    p.prof = h->profile ? h->d_prof : nullptr;
    p.wmax = 1u << h->warp_log2;
    p.fixed = h->fmode == PQ_F_FIXED ? 1 : 0;
    if (p.fixed) {
        int rc = ensure_fixed_tables();
        if (rc) return rc;
        p.mag = fminf(fmaxf(rintf(mag * 256.0f), -32767.0f), 32767.0f);
    }
    p.K = (uint32_t)choose_K(h, frames, p.log2S, dump != nullptr);
#ifndef PQ_NT512
#define PQ_NT512 1
#endif
    // clusters with one CTA per SM: 512 threads (production kernel only)
    if (PQ_NT512 && h->threads_opt == 0 && p.K > 1 && !p.plain && !dump && !h->profile &&
        (size_t)frames * p.K <= (size_t)h->sm_count)
        nthreads = 512;
    h->last_K = (int)p.K;
    h->last_log2S = p.log2S;
    h->last_threads = nthreads;
    const size_t smem = dec_smem_bytes(p.S);
    const int slot = h->n_timed % PQ_TIMING_SLOTS;
    if (h->timing) CUDA_TRY(cudaEventRecord(h->ev[2 * slot], st));
    int lrc;
    if (h->fmode == PQ_F_FIXED) lrc = launch_dec<PQ_F_FIXED>(p, frames, nthreads, smem, st);
#ifdef PQ_ONLY_FIXED  // A/B builds of the fixed-point kernel (tools/build_variant.sh)
    else lrc = set_err(-1, "variant build: fixed point only");
#else
    else if (h->fmode == PQ_F_MINSUM) lrc = launch_dec<PQ_F_MINSUM>(p, frames, nthreads, smem, st);
    else if (h->fmode == PQ_F_FAST) lrc = launch_dec<PQ_F_FAST>(p, frames, nthreads, smem, st);
    else lrc = launch_dec<PQ_F_EXACT>(p, frames, nthreads, smem, st);
#endif
    if (lrc) return lrc;
    if (h->timing) {
        CUDA_TRY(cudaEventRecord(h->ev[2 * slot + 1], st));
        h->n_timed++;
    }
    launches++;
    const size_t nwords = (size_t)frames * h->wpf;
    if (x_hat) {
        if (cw) {
            xor_words<<<(unsigned)((nwords + 255) / 256 < 4096 ? (nwords + 255) / 256 : 4096), 256, 0, st>>>(
                h->d_x, cw, x_hat, nwords);
            CUDA_TRY(cudaGetLastError());
        } else {
            CUDA_TRY(cudaMemcpyAsync(x_hat, h->d_x, nwords * 4, cudaMemcpyDeviceToDevice, st));
        }
        launches++;
    }
    if (u_hat) {
        // u_hat = T(x_hat') XOR (v & mask): T maps the shifted partial sums back to
        // shifted decisions (zero on the frozen set), the XOR restores the revealed values
        int rc;
        if (frozen_u) {
            rc = launch_transform(h->d_x, u_hat, h->n, frames, nullptr, nullptr, st, &launches);
            if (rc) return rc;
            const size_t g = (nwords + 255) / 256 < 4096 ? (nwords + 255) / 256 : 4096;
            xor_masked<<<(unsigned)g, 256, 0, st>>>(u_hat, frozen_u, h->d_mask, h->wpf, nwords);
            CUDA_TRY(cudaGetLastError());
            launches++;
        } else {
            rc = launch_transform(h->d_x, u_hat, h->n, frames, nullptr, nullptr, st, &launches);
            if (rc) return rc;
        }
    }
    h->last_launches = launches;
    return 0;
}

int pq_sc_decode_f32(pq_decoder *h, const float *llr, const uint32_t *frozen_u, uint32_t *u_hat,
                     uint32_t *x_hat, int frames, void *stream)
{
    if (frames == 0 && h) return 0;
    if (!llr) return set_err(-1, "llr is NULL");
    return decode_impl(h, llr, nullptr, 0.0f, frozen_u, u_hat, x_hat, nullptr, frames, stream);
}

int pq_sc_decode_q88(pq_decoder *h, const int16_t *llr_q88, const uint32_t *frozen_u, uint32_t *u_hat,
                     uint32_t *x_hat, int frames, void *stream)
{
    if (frames == 0 && h) return 0;
    if (!llr_q88) return set_err(-1, "llr_q88 is NULL");
    if (h && h->fmode != PQ_F_FIXED) return set_err(-1, "pq_sc_decode_q88 needs a PQ_F_FIXED decoder");
    return decode_impl(h, nullptr, nullptr, 0.0f, frozen_u, u_hat, x_hat, nullptr, frames, stream,
                       reinterpret_cast<const short *>(llr_q88));
}

int pq_sc_decode_f32_dump(pq_decoder *h, const float *llr, const uint32_t *frozen_u, uint32_t *u_hat,
                          uint32_t *x_hat, float *dump, int frames, void *stream)
{
    if (frames == 0 && h) return 0;
    if (!llr || !dump) return set_err(-1, "llr/dump is NULL");
    return decode_impl(h, llr, nullptr, 0.0f, frozen_u, u_hat, x_hat, dump, frames, stream);
}

int pq_debug_fmag(int f_mode, const float *a, const float *b, float *out, int n, void *stream)
{
    if (n < 0) return set_err(-1, "n must be >= 0");
    if (n == 0) return 0;
    if (!a || !b || !out) return set_err(-1, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = (n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024;
    switch (f_mode) {
    case PQ_F_EXACT: fmag_kernel<PQ_F_EXACT><<<grid, 256, 0, st>>>(a, b, out, n); break;
    case PQ_F_MINSUM: fmag_kernel<PQ_F_MINSUM><<<grid, 256, 0, st>>>(a, b, out, n); break;
    case PQ_F_FIXED: {
        int rc = ensure_fixed_tables();
        if (rc) return rc;
        fmag_kernel<PQ_F_FIXED><<<grid, 256, 0, st>>>(a, b, out, n);
        break;
    }
    case PQ_F_FAST: fmag_kernel<PQ_F_FAST><<<grid, 256, 0, st>>>(a, b, out, n); break;
    default: return set_err(-1, "unknown f mode %d", f_mode);
    }
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int pq_sc_decode_bsc(pq_decoder *h, const uint32_t *y_bits, float llr_mag, const uint32_t *frozen_u,
                     uint32_t *u_hat, uint32_t *x_hat, int frames, void *stream)
{
    if (frames == 0 && h) return 0;
    if (!y_bits) return set_err(-1, "y_bits is NULL");
    if (!(llr_mag >= 0.0f)) return set_err(-1, "llr_mag must be >= 0");
    return decode_impl(h, nullptr, y_bits, llr_mag, frozen_u, u_hat, x_hat, nullptr, frames, stream);
}

}  // extern "C"

