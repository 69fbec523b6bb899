// serial_q88.cuh -- the single-warp band of the fixed-point decoder (SPEC.md's
// sc_decode_fixed), nodes of width W <= 2048.
//
// The serial band is one dependent instruction chain per frame, so this
// engine is built to keep that chain short:
//  * Q8.8 codes live in int registers; f is the table boxplus of
//    oracle/sc_oracle.c with ONE 4095-byte symmetric table T[k] = C[|k-2047|]
//    (both lookups index it, the +2047 bias is an immediate of the load):
//      |f| = max(0, min(|a|,|b|) + T[min(|a|+|b|, 2047)] - T[clamp(|a|-|b|, +-2047)])
//    g = sat(b +- a) is one fused add-min plus a max.
//  * Node types below width 32 come from the frozen-mask word of the
//    sub-tree (no type table, no vote), and nodes of width <= 16 are decoded
//    with their values REPLICATED in every lane: f/g steps, rate-1 guards,
//    repetition sums and decisions are all in-lane register arithmetic, no
//    shuffles, ballots or votes.  Width-8 nodes are compile-time
//    specialisations per frozen pattern (straight-line SC, a handful of
//    patterns cover every mixed width-8 node of the BASELINE codes; any
//    other pattern takes a generic routine).
//  * Width-32 nodes are lane-parallel (lane l = element l): one shuffle per
//    step, then the width-16 child is gathered into every lane.  A rate-1
//    right child's two hypotheses (left partial-sum bit 0 / 1) are decided
//    while the left child decodes; the partial sums then select per bit.
//  * Widths 64..512 walk with lane l holding elements l + 32q in registers
//    (in-lane f/g steps); 1024 / 2048 step from the shared-memory stage
//    buffers (the node values arrive there as fp32 Q8.8 codes from the
//    block band and are converted on load).
// Every decision is SC's own: the rate-1 and repetition shortcuts are the
// decision-exact ones of polarsc.cu (same guards), and a failed guard
// re-decodes the node with plain SC.  tests/ and tools/ubench/serial_bench.cu
// check it bit for bit against the integer oracle.
#pragma once

#ifndef SE_SPEC_R1
#define SE_SPEC_R1 0
#endif
#ifndef SE_SPEC_REP
#define SE_SPEC_REP 0
#endif
#ifndef SE_W8_PATTERNS
#define SE_W8_PATTERNS 2
#endif
#ifndef SE_UNR
#define SE_UNR 256  // widest node of the compile-time unrolled register walk
#endif
#ifndef SE_SPEC_LP
#define SE_SPEC_LP 0
#endif
#ifndef SE_UNIFORM_MASK
#define SE_UNIFORM_MASK 1
#endif
#ifndef SE_DIVZ
#define SE_DIVZ 0
#endif



namespace se {

#ifdef SE_PROF
// cycle profile of the engine's layers (microbenchmarks only): slot sums and counts
__shared__ unsigned long long se_prof[2][16];
#define SE_T0() const long long se_t0_ = clock64()
#define SE_T1(slot)                                                        \
    do {                                                                   \
        if ((threadIdx.x & 31) == 0) {                                     \
            se_prof[0][slot] += clock64() - se_t0_;                        \
            se_prof[1][slot] += 1;                                         \
        }                                                                  \
    } while (0)
#else
#define SE_T0()
#define SE_T1(slot)
#endif

enum : int { T_MIX = 0, T_R0 = 1, T_R1 = 2, T_REP = 3 };

__host__ __device__ constexpr uint32_t lm(int w) { return w >= 32 ? 0xffffffffu : ((1u << w) - 1u); }
// node type from its frozen mask (bit i = leaf i frozen), as pq_decoder_set_frozen_mask
__host__ __device__ constexpr int ntype(uint32_t m, int W)
{
    return m == lm(W) ? T_R0 : m == 0u ? T_R1 : (W > 1 && m == lm(W - 1)) ? T_REP : T_MIX;
}
__host__ __device__ constexpr int clog2(int w) { return w <= 1 ? 0 : 1 + clog2(w / 2); }

// T[k] = C[|k - 2047|], k = 0..4094 (C = CORR_TAB_C, zero beyond 1597)
__shared__ uint8_t ctab[4096];
// integer rate-1 thresholds (RATE1_TAU_FIX, never-taken entries at INT_MAX)
__constant__ int TAUI[26];

__device__ __forceinline__ void load_tables()
{
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
        const int k = i < 2047 ? 2047 - i : i - 2047;
        ctab[i] = (uint8_t)(int)CORR_TAB_C[k < 4096 ? k : 4096];
    }
}

__device__ __forceinline__ int fq(int a, int b)
{
    const int ma = abs(a), mb = abs(b);
    const int s = min(ma + mb, 2047);
    const int d = max(min(ma - mb, 2047), -2047);
    const int r = max(min(ma, mb) + (int)ctab[s + 2047] - (int)ctab[d + 2047], 0);
    return (a ^ b) < 0 ? -r : r;
}
__device__ __forceinline__ int qa(int x, int y) { return max(min(x + y, 32767), -32767); }
__device__ __forceinline__ int gq(int a, int b, uint32_t s) { return qa(b, s ? -a : a); }
// fp32 Q8.8 code (an exact small integer) -> int
__device__ __forceinline__ int f2q(float v) { return __float2int_rn(v); }

// ---- width <= 16, values replicated in every lane

// plain SC (no shortcuts) of a node with runtime frozen mask m: the exact
// fallback after a failed rate-1 guard
template <int W>
__device__ __forceinline__ uint32_t rplain(const int (&x)[W], uint32_t m)
{
    if constexpr (W == 1) {
        return ((m & 1u) || x[0] >= 0) ? 0u : 1u;
    } else {
        constexpr int H = W / 2;
        int c[H];
#pragma unroll
        for (int i = 0; i < H; i++) c[i] = fq(x[i], x[i + H]);
        const uint32_t xl = rplain<H>(c, m & lm(H));
#pragma unroll
        for (int i = 0; i < H; i++) c[i] = gq(x[i], x[i + H], (xl >> i) & 1u);
        const uint32_t xr = rplain<H>(c, m >> H);
        return (xl ^ xr) | (xr << H);
    }
}

// SSC with compile-time frozen mask M: straight-line code, ok &= every guard
template <int W, uint32_t M>
__device__ __forceinline__ uint32_t rnode(const int (&x)[W], bool &ok)
{
    constexpr int t = ntype(M, W);
    if constexpr (W == 1) {
        return (M & 1u) ? 0u : (x[0] < 0 ? 1u : 0u);
    } else if constexpr (t == T_R0) {
        return 0u;
    } else if constexpr (t == T_R1) {
        int mn = abs(x[0]);
        uint32_t b = (uint32_t)x[0] >> 31;
#pragma unroll
        for (int i = 1; i < W; i++) {
            mn = min(mn, abs(x[i]));
            b |= ((uint32_t)x[i] >> 31) << i;
        }
        ok &= mn >= TAUI[clog2(W)];
        return b;
    } else if constexpr (t == T_REP) {
        // SC's g-chain with zero partial sums, in SC's pairing order
        int s[W];
#pragma unroll
        for (int i = 0; i < W; i++) s[i] = x[i];
#pragma unroll
        for (int hv = W / 2; hv >= 1; hv >>= 1)
#pragma unroll
            for (int q = 0; q < hv; q++) s[q] = qa(s[q + hv], s[q]);
        return s[0] < 0 ? lm(W) : 0u;
    } else {
        constexpr int H = W / 2;
        constexpr uint32_t ML = M & lm(H), MR = M >> H;
        constexpr int tl = ntype(ML, H), tr = ntype(MR, H);
        if constexpr (SE_SPEC_R1 && tr == T_R1 && tl != T_R0) {
            // rate-1 right child: its decisions under both values of each
            // left partial-sum bit, computed before (and overlapped with) the
            // left child; the left's bits then select per position.  The
            // guard over both hypotheses implies the real one.
            uint32_t dp = 0, dm = 0;
            int mn = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < H; i++) {
                const int gp = qa(x[i + H], x[i]), gm = qa(x[i + H], -x[i]);
                dp |= ((uint32_t)gp >> 31) << i;
                dm |= ((uint32_t)gm >> 31) << i;
                mn = min(mn, min(abs(gp), abs(gm)));
            }
            int c[H];
#pragma unroll
            for (int i = 0; i < H; i++) c[i] = fq(x[i], x[i + H]);
            const uint32_t xl = rnode<H, ML>(c, ok);
            uint32_t xr;
            if (mn >= TAUI[clog2(H)]) {
                xr = (dp & ~xl) | (dm & xl);
            } else {
#pragma unroll
                for (int i = 0; i < H; i++) c[i] = gq(x[i], x[i + H], (xl >> i) & 1u);
                xr = rnode<H, MR>(c, ok);
            }
            return (xl ^ xr) | (xr << H);
        } else if constexpr (SE_SPEC_REP && tl == T_REP && tr != T_R0 && H <= 4) {
            // repetition left child: its partial sums are all 0 or all 1, so
            // the right child is decoded under both and selected
            int c0[H], c1[H];
#pragma unroll
            for (int i = 0; i < H; i++) {
                c0[i] = qa(x[i + H], x[i]);
                c1[i] = qa(x[i + H], -x[i]);
            }
            bool ok0 = true, ok1 = true;
            const uint32_t r0 = rnode<H, MR>(c0, ok0), r1 = rnode<H, MR>(c1, ok1);
            int c[H];
#pragma unroll
            for (int i = 0; i < H; i++) c[i] = fq(x[i], x[i + H]);
            const uint32_t xl = rnode<H, ML>(c, ok);
            const uint32_t xr = xl ? r1 : r0;
            ok &= xl ? ok1 : ok0;
            return (xl ^ xr) | (xr << H);
        } else {
            uint32_t xl = 0, xr = 0;
            if constexpr (tl != T_R0) {
                int c[H];
#pragma unroll
                for (int i = 0; i < H; i++) c[i] = fq(x[i], x[i + H]);
                xl = rnode<H, ML>(c, ok);
            }
            if constexpr (tr != T_R0) {
                int c[H];
#pragma unroll
                for (int i = 0; i < H; i++) c[i] = gq(x[i], x[i + H], (xl >> i) & 1u);
                xr = rnode<H, MR>(c, ok);
            }
            return (xl ^ xr) | (xr << H);
        }
    }
}

// plain SC of a width-8 node with runtime frozen mask: the generic path (any
// pattern without a routine, and every failed guard).  One out-of-line copy.
__device__ __noinline__ uint32_t w8plain(int x0, int x1, int x2, int x3, int x4, int x5, int x6, int x7, uint32_t m)
{
    const int x[8] = {x0, x1, x2, x3, x4, x5, x6, x7};
    return rplain<8>(x, m);
}

template <uint32_t M>
__device__ __forceinline__ uint32_t r8(const int (&x)[8], uint32_t m)
{
    bool ok = true;
    const uint32_t b = rnode<8, M>(x, ok);
    return ok ? b : w8plain(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], m);
}

// width-8 node, any frozen pattern m (uniform).  Straight-line routines for
// the node types and the two patterns that dominate the mixed width-8 nodes
// of the BASELINE codes (SPC and F F F I F I I I: ~80 %); everything else
// takes the out-of-line generic path.  Code size is the constraint here: the
// serial band's instructions must stay within the SM's instruction caches.
__device__ __forceinline__ uint32_t d8(const int (&x)[8], uint32_t m)
{
    if (m == 0xFFu) return 0u;
    if (m == 0x00u) return r8<0x00u>(x, m);
    if (m == 0x01u) return r8<0x01u>(x, m);   // F I I I I I I I  (SPC)
    if (m == 0x7Fu) return r8<0x7Fu>(x, m);
#if SE_W8_PATTERNS >= 2
    if (m == 0x17u) return r8<0x17u>(x, m);   // F F F I F I I I
#endif
#if SE_W8_PATTERNS >= 3
    if (m == 0x1Fu) return r8<0x1Fu>(x, m);   // F F F F F I I I
    if (m == 0x07u) return r8<0x07u>(x, m);   // F F F I I I I I
#endif
    return w8plain(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], m);
}

// ---- widths 16 and 32, lane-parallel: lane l holds element l (lanes >= W
// carry don't-care values); every lane returns the same bits

// the width-8 child of a lane-parallel width-16 node: gather its 8 values
// (lanes 0..7) into every lane, then the replicated pattern routines
//
// z is a lane-dependent zero (SE_DIVZ): a shuffle from a constant lane is
// warp-uniform to ptxas, which then MAY move the whole replicated width-8
// computation to the uniform datapath (USEL / UIADD3 chains fed by R2UR
// transfers).  Whether it does depends on the uniform registers the rest of
// the kernel leaves free -- an unrelated edit of the upper band flipped w32
// from 557 to 655 instructions and cost every config 12 % -- so the source
// lane is made opaque and the replicated arithmetic stays on the vector ALUs.
__device__ __forceinline__ uint32_t child8(int c, uint32_t m8, bool plain, int z)
{
    SE_T0();
    int x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = __shfl_sync(0xffffffffu, c, i | z);
    const uint32_t r = plain ? w8plain(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], m8) : d8(x, m8);
    SE_T1(0);
    return r;
}

__device__ __forceinline__ uint32_t w16_body(int v, uint32_t m16, int z);
__device__ __forceinline__ uint32_t w16(int v, uint32_t m16, int z)
{
    SE_T0();
    const uint32_t r = w16_body(v, m16, z);
    SE_T1(1);
    return r;
}
__device__ __forceinline__ uint32_t w16_body(int v, uint32_t m16, int z)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int t = ntype(m16, 16);
    if (t == T_R0) return 0u;
    if (t == T_R1) {
        const bool ok = __all_sync(FULL, lane >= 16 || abs(v) >= TAUI[4]);
        const uint32_t neg = __ballot_sync(FULL, v < 0) & 0xffffu;
        if (ok) return neg;
    } else if (t == T_REP) {
        const int vv = lane < 16 ? v : 0;
        const int tot = __reduce_add_sync(FULL, vv);
        const int mag = __reduce_add_sync(FULL, abs(vv));
        if (mag <= 32767) return tot < 0 ? 0xffffu : 0u;
        int s = vv;
#pragma unroll
        for (int hh = 8; hh >= 1; hh >>= 1) s = qa(__shfl_down_sync(FULL, s, hh), s);
        return __shfl_sync(FULL, s, 0) < 0 ? 0xffffu : 0u;
    }
    const bool plain = t != T_MIX;
    const int b = __shfl_down_sync(FULL, v, 8);  // lanes < 8: the pair (l, l + 8)
    const uint32_t ml = m16 & 0xffu, mr = m16 >> 8;
    bool spec = false;
    uint32_t dp = 0, dm = 0;
    if (SE_SPEC_LP && !plain && mr == 0u) {  // rate-1 right child: both hypotheses now
        const int gp = qa(b, v), gm = qa(b, -v);
        spec = __all_sync(FULL, lane >= 8 || min(abs(gp), abs(gm)) >= TAUI[3]);
        dp = __ballot_sync(FULL, gp < 0) & 0xffu;
        dm = __ballot_sync(FULL, gm < 0) & 0xffu;
    }
    uint32_t xl = 0, xr = 0;
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
        const uint32_t m8 = side ? mr : ml;
        uint32_t bits = 0;
        if (side == 1 && spec) {
            bits = (dp & ~xl) | (dm & xl);
        } else if (plain || m8 != 0xffu) {
            int c;
            if (side) c = gq(v, b, (xl >> lane) & 1u);
            else c = fq(v, b);
            bits = child8(c, m8, plain, z);
        }
        if (side) xr = bits;
        else xl = bits;
    }
    return (xl ^ xr) | (xr << 8);
}

__device__ __forceinline__ uint32_t w32_body(int v, uint32_t m32);
__device__ __noinline__ uint32_t w32(int v, uint32_t m32)
{
    SE_T0();
#if SE_UNIFORM_MASK
    // The mask is warp-uniform, but as the argument of an out-of-line function
    // the compiler must treat it as divergent: every type test below became a
    // potentially divergent branch with a convergence barrier (BSSY / BSYNC /
    // BREAK) and every shuffle or vote a divergence check (BRA.DIV, WARPSYNC).
    // One redux hands it back as a uniform register: the branches on it are
    // uniform branches and the barriers and checks disappear (w32: 809 -> 555
    // SASS instructions, none of them BSSY).  c2..c5 +4.6 .. +7.3 %.  The same
    // trick on the width-8 fallback, the wide levels' types, the register
    // walk's type masks or per node costs 3-5 % (profiles/r02/ab_uniform.txt):
    // ptxas keeps a value uniform only while uniform registers are free along the
    // call chain: with the walk's type masks in uniform registers (live across
    // the w32 calls) this function falls back to the divergent form (806
    // instructions) and nothing is gained in the walk itself.
    m32 = __reduce_or_sync(0xffffffffu, m32);
#endif
    const uint32_t r = w32_body(v, m32);
    SE_T1(2);
    return r;
}
__device__ __forceinline__ uint32_t w32_body(int v, uint32_t m32)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
#if SE_DIVZ
    const int z = abs(v) >> 16;  // 0: Q8.8 codes are saturated to +-32767 (see child8)
#else
    const int z = 0;
#endif
    const int t = ntype(m32, 32);
    if (t == T_R0) return 0u;
    if (t == T_R1) {
        const bool ok = __all_sync(FULL, abs(v) >= TAUI[5]);
        const uint32_t neg = __ballot_sync(FULL, v < 0);
        if (ok) return neg;
    } else if (t == T_REP) {
        // exact sum by redux when no pairwise partial sum can saturate
        const int tot = __reduce_add_sync(FULL, v);
        const int mag = __reduce_add_sync(FULL, abs(v));
        if (mag <= 32767) return tot < 0 ? FULL : 0u;
        int s = v;
#pragma unroll
        for (int hh = 16; hh >= 1; hh >>= 1) s = qa(__shfl_down_sync(FULL, s, hh), s);
        return __shfl_sync(FULL, s, 0) < 0 ? FULL : 0u;
    }
    // mixed, or a rate-1 node whose guard failed: its rate-1 halves carry
    // their own guards (decision-exact either way)
    const int b = __shfl_down_sync(FULL, v, 16);  // lanes < 16: the pair (l, l + 16)
    const uint32_t ml = m32 & 0xffffu, mr = m32 >> 16;
    bool spec = false;
    uint32_t dp = 0, dm = 0;
    if (SE_SPEC_LP && t == T_MIX && mr == 0u) {  // rate-1 right child: both hypotheses now
        const int gp = qa(b, v), gm = qa(b, -v);
        spec = __all_sync(FULL, lane >= 16 || min(abs(gp), abs(gm)) >= TAUI[4]);
        dp = __ballot_sync(FULL, gp < 0) & 0xffffu;
        dm = __ballot_sync(FULL, gm < 0) & 0xffffu;
    }
    uint32_t xl = 0, xr = 0;
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
        const uint32_t m16 = side ? mr : ml;
        uint32_t bits = 0;
        if (side == 1 && spec) {
            bits = (dp & ~xl) | (dm & xl);
        } else if (m16 != 0xffffu) {
            int c;
            if (side) c = gq(v, b, (xl >> lane) & 1u);
            else c = fq(v, b);
            bits = w16(c, m16, z);
        }
        if (side) xr = bits;
        else xl = bits;
    }
    return (xl ^ xr) | (xr << 16);
}

// ---- widths 8..32 with a compile-time frozen pattern: a whole width-32
// sub-tree as straight-line code.  SC's control flow does not depend on the
// data, and density-evolution constructions draw their width-32 patterns from
// one small family (30 patterns cover every mixed width-32 node of the
// BASELINE codes and of the Table-1 codes for n = 14..24), so a pattern can
// have its own routine: no type tests, loops or calls inside, every guard
// folded into one flag that is tested once at the end (a failed guard
// re-decodes the sub-tree with the generic w32, which is decision-exact on
// its own).  Lane-parallel at widths 32 and 16 (lane l = element l), rate-1
// and repetition children of any width decided by ballot / redux without a
// gather, mixed width-8 children gathered into the replicated routines.
// A routine executes ~40 % fewer instructions than the generic w32 on the same
// node, but every routine is 8-19 KB of code that runs once per call, so the
// gain is bounded by instruction fetch: with all 30 patterns the serial warp
// stalls 32 % of its cycles on fetch and c3 (two CTAs per SM) loses 21 %.  The
// engine is therefore templated on SP: the routines of the SE_W32_NPAT most
// frequent patterns (2: F I^31 and 0x10117, 43 % of c3's mixed width-32
// nodes) are compiled into the clustered kernels only (one CTA per SM: c5
// +4.6 %); with two CTAs per SM the same two routines cost c3 1 %, so those
// kernels keep SP = false (profiles/r02/ab_w32_patterns.txt).

template <int W, uint32_t M>
__device__ __forceinline__ uint32_t lnode(int v, bool &ok)
{
    constexpr int t = ntype(M, W);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    if constexpr (t == T_R0) {
        return 0u;
    } else if constexpr (t == T_R1) {
        ok &= __ballot_sync(FULL, (W == 32 || lane < W) && abs(v) < TAUI[clog2(W)]) == 0u;
        return __ballot_sync(FULL, v < 0) & lm(W);
    } else if constexpr (t == T_REP) {
        // exact sum by redux when no pairwise partial sum can saturate
        const int vv = (W == 32 || lane < W) ? v : 0;
        const int tot = __reduce_add_sync(FULL, vv);
        ok &= __reduce_add_sync(FULL, abs(vv)) <= 32767;
        return tot < 0 ? lm(W) : 0u;
    } else if constexpr (W == 8) {
        int x[8];
        const int z = SE_DIVZ ? abs(v) >> 16 : 0;  // lane-dependent zero, see child8
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = __shfl_sync(FULL, v, i | z);
        return rnode<8, M>(x, ok);
    } else {
        constexpr int H = W / 2;
        constexpr uint32_t ML = M & lm(H), MR = M >> H;
        const int b = __shfl_down_sync(FULL, v, H);  // lanes < H: the pair (l, l + H)
        uint32_t xl = 0, xr = 0;
        if constexpr (ntype(ML, H) != T_R0) xl = lnode<H, ML>(fq(v, b), ok);
        if constexpr (ntype(MR, H) != T_R0) xr = lnode<H, MR>(gq(v, b, (xl >> lane) & 1u), ok);
        return (xl ^ xr) | (xr << H);
    }
}

__device__ __noinline__ uint32_t w32(int v, uint32_t m32);

template <uint32_t M>
__device__ __noinline__ uint32_t w32s(int v)
{
    bool ok = true;
    const uint32_t r = lnode<32, M>(v, ok);
    return ok ? r : w32(v, M);
}

// the width-32 patterns with a routine: X(mask), most frequent first
#ifndef SE_W32_NPAT
#define SE_W32_NPAT 2
#endif
#ifndef SE_SP_ALL
#define SE_SP_ALL 0  // 1: the pattern routines in the unclustered kernels too (measured slower)
#endif
#define SE_W32_P0(X)
#define SE_W32_P1(X) X(0x1u)
#define SE_W32_P2(X) SE_W32_P1(X) X(0x10117u)
#define SE_W32_P4(X) SE_W32_P2(X) X(0x177f7fffu) X(0x117177fu)
#define SE_W32_P8(X) SE_W32_P4(X) X(0x117u) X(0x1011fu) X(0x177fffffu) X(0x17u)
#define SE_W32_P12(X) SE_W32_P8(X) X(0x3u) X(0x11717ffu) X(0x7u) X(0x17ffffffu)
#define SE_W32_P30(X)                                                                              \
    SE_W32_P12(X) X(0x1013fu) X(0x77f7fffu) X(0x1171fffu)                                          \
    X(0x7177fu) X(0x13f7fffu) X(0x37f7fffu) X(0x1fffffffu) X(0x17177fu) X(0x11f7fffu) X(0x1037fu)  \
    X(0x17f7fffu) X(0x1017fu) X(0x1077fu) X(0x3177fu) X(0x1173fffu) X(0x3fffffffu) X(0x3077fu)    \
    X(0x11f3fffu)
#define SE_CAT_(a, b) a##b
#define SE_CAT(a, b) SE_CAT_(a, b)
#define SE_W32_PATTERNS(X) SE_CAT(SE_W32_P, SE_W32_NPAT)(X)

template <bool SP>
__device__ __forceinline__ uint32_t w32d(int v, uint32_t m32)
{
    if constexpr (SP) {
#define SE_X(mask) if (m32 == mask) return w32s<mask>(v);
        SE_W32_PATTERNS(SE_X)
#undef SE_X
    }
    return w32(v, m32);
}

// ---- widths 64..512: lane l holds elements l + 32q (q < W/32) in registers
// (in-lane f/g steps), the tree unrolled at compile time (node types as two
// uniform masks, every type test a constant shift); the width-32 leaves are
// one out-of-line w32 (out-of-line calls per width were measured ~20 % slower:
// the register values would cross every call)
struct WalkCtx {
    const uint32_t *fm;  // S-local frozen-mask words (shared memory)
    uint32_t wb0, wb1;   // type bits of relative heap positions 1..31
    uint32_t pos0;       // S-local leaf position of the walk root
};

template <int REL>
__device__ __forceinline__ int wtype(const WalkCtx &c)
{
    return (int)(((c.wb0 >> REL) & 1u) | (((c.wb1 >> REL) & 1u) << 1));
}

template <int W, int REL, bool SP>
__device__ __forceinline__ void wnode(const int (&x)[W / 32], const WalkCtx &c, uint32_t (&xo)[W / 32]);

template <int H, int REL, bool SP>
__device__ __forceinline__ void wchild(const int (&x)[H / 32], const WalkCtx &c, uint32_t (&xo)[H / 32])
{
    if constexpr (H == 32) {
        // relative heap position REL at the width-32 level: leaf offset
        constexpr int e = clog2(REL);
        const uint32_t pos = c.pos0 + 32u * (uint32_t)(REL - (1 << e));
        PQ_CHECK(e >= 0 && REL < 32);
        xo[0] = w32d<SP>(x[0], c.fm[pos >> 5]);
    } else {
        wnode<H, REL, SP>(x, c, xo);
    }
}

template <int W, int REL, bool SP>
__device__ __forceinline__ void wnode(const int (&x)[W / 32], const WalkCtx &c, uint32_t (&xo)[W / 32])
{
    constexpr int V = W / 32, Vh = V / 2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int t = wtype<REL>(c), tl = wtype<2 * REL>(c), tr = wtype<2 * REL + 1>(c);
    if (t == T_R0) {
#pragma unroll
        for (int q = 0; q < V; q++) xo[q] = 0u;
        return;
    }
    if (t == T_R1) {
        int mn = abs(x[0]);
#pragma unroll
        for (int q = 1; q < V; q++) mn = min(mn, abs(x[q]));
        if (__all_sync(FULL, mn >= TAUI[clog2(W)])) {
#pragma unroll
            for (int q = 0; q < V; q++) xo[q] = __ballot_sync(FULL, x[q] < 0);
            return;
        }
    }
    if (t == T_REP) {
        int s[V];
#pragma unroll
        for (int q = 0; q < V; q++) s[q] = x[q];
#pragma unroll
        for (int hv = V / 2; hv >= 1; hv >>= 1)
#pragma unroll
            for (int q = 0; q < hv; q++) s[q] = qa(s[q + hv], s[q]);
        const int tot = __reduce_add_sync(FULL, s[0]);
        const int mag = __reduce_add_sync(FULL, abs(s[0]));
        uint32_t bits;
        if (mag <= 32767) {
            bits = tot < 0 ? FULL : 0u;
        } else {
            int s0 = s[0];
#pragma unroll
            for (int hh = 16; hh >= 1; hh >>= 1) s0 = qa(__shfl_down_sync(FULL, s0, hh), s0);
            bits = __shfl_sync(FULL, s0, 0) < 0 ? FULL : 0u;
        }
#pragma unroll
        for (int q = 0; q < V; q++) xo[q] = bits;
        return;
    }
    // mixed, or a rate-1 node whose guard failed (its rate-1 children carry
    // their own guards, exactly as in polarsc.cu)
    int ch[Vh];
    uint32_t xl[Vh], xr[Vh];
    if (tl == T_R0) {
#pragma unroll
        for (int q = 0; q < Vh; q++) xl[q] = 0u;
    } else {
#pragma unroll
        for (int q = 0; q < Vh; q++) ch[q] = fq(x[q], x[q + Vh]);
        wchild<W / 2, 2 * REL, SP>(ch, c, xl);
    }
    if (tr == T_R0) {
#pragma unroll
        for (int q = 0; q < Vh; q++) xr[q] = 0u;
    } else {
#pragma unroll
        for (int q = 0; q < Vh; q++) ch[q] = gq(x[q], x[q + Vh], (xl[q] >> lane) & 1u);
        wchild<W / 2, 2 * REL + 1, SP>(ch, c, xr);
    }
#pragma unroll
    for (int q = 0; q < Vh; q++) {
        xo[q] = xl[q] ^ xr[q];
        xo[Vh + q] = xr[q];
    }
}

// write V uniform words: lane q < V stores word q (select chain, no branches)
template <int V>
__device__ __forceinline__ void put_words(uint32_t *xw, const uint32_t (&xo)[V])
{
    const int lane = threadIdx.x & 31;
    uint32_t w = xo[0];
#pragma unroll
    for (int q = 1; q < V; q++) w = lane == q ? xo[q] : w;
    if (lane < V) xw[lane] = w;
}

template <int W, bool SP>
__device__ __forceinline__ void walk_root(const int *nd, uint32_t *xw, const WalkCtx &c)
{
    constexpr int V = W / 32;
    const int lane = threadIdx.x & 31;
    int x[V];
    uint32_t xo[V];
#pragma unroll
    for (int q = 0; q < V; q++) x[q] = nd[32 * q + lane];
    wnode<W, 1, SP>(x, c, xo);
    put_words<V>(xw, xo);
}

// the walk from a width-W (64..512) node whose int values are at nd
template <bool SP>
__device__ __noinline__ void walk(const int *nd, uint32_t *xs, const uint8_t *ty, const uint32_t *fm, uint32_t S,
                                  int dS, int d0, uint32_t j0)
{
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t W = S >> (d0 - dS);
    const int e = d0 - dS;
    const uint32_t root = (1u << e) + (j0 & ((1u << e) - 1u));
    const int k32 = 26 - __clz(W);  // log2(W) - 5
    int tint = T_MIX;
    if (lane >= 1) {
        const int k = 31 - __clz(lane);
        if (k <= k32) tint = ty[(root << k) + (uint32_t)lane - (1u << k)];
    }
    WalkCtx c;
    c.fm = fm;
    c.wb0 = __ballot_sync(FULL, tint & 1);
    c.wb1 = __ballot_sync(FULL, tint & 2);
    c.pos0 = (j0 * W) & (S - 1);
    uint32_t *xw = xs + (c.pos0 >> 5);
    SE_T0();
#if SE_UNR >= 512
    if (W == 512) walk_root<512, SP>(nd, xw, c);
    else
#endif
#if SE_UNR >= 256
    if (W == 256) walk_root<256, SP>(nd, xw, c);
    else
#endif
    if (W == 128) walk_root<128, SP>(nd, xw, c);
    else walk_root<64, SP>(nd, xw, c);
    SE_T1(3);
}

// ---- widths 1024 / 2048 from the shared-memory stage buffers.  The node's
// values are int Q8.8 codes at st_end - 2W, except at the band's root
// (FROM_F32: fp32 codes written by the block band)
// ---- widths 1024 / 2048 from the shared-memory stage buffers: node values
// at st_end - 2W, fp32 codes at the band's root (FROM_F32, written by the
// block band) and int codes below.  Every loop loads a batch of B elements
// per lane before it computes or stores (the stage buffers are one shared
// array: without the batching each element's loads would wait for the
// previous element's store).
template <int W, bool FROM_F32, bool SP>
__device__ __forceinline__ void wide(float *st_end, uint32_t *xs, const uint8_t *ty, const uint32_t *fm, uint32_t S,
                                     int dS, int d0, uint32_t j0)
{
    constexpr int V = W / 32, Vh = V / 2, B = 8;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int e = d0 - dS;
    const uint32_t lh = (1u << e) + (j0 & ((1u << e) - 1u));
    const int *ndi = reinterpret_cast<const int *>(st_end - 2 * W);
    const float *ndf = st_end - 2 * W;
    int *ch = reinterpret_cast<int *>(st_end - W);
    uint32_t *xw = xs + (((j0 * W) & (S - 1)) >> 5);
    auto ld = [&](int i) -> int { return FROM_F32 ? f2q(ndf[i]) : ndi[i]; };
    const uint8_t t = ty[lh], tl = ty[2 * lh], tr = ty[2 * lh + 1];
    if (t == T_R0) {
        for (int q = lane; q < V; q += 32) xw[q] = 0u;
        __syncwarp();
        return;
    }
    if (t == T_R1) {
        int mn = 0x7fffffff;
#pragma unroll 1
        for (int q0 = 0; q0 < V; q0 += B) {
            int a[B];
#pragma unroll
            for (int k = 0; k < B; k++) a[k] = ld(32 * (q0 + k) + lane);
#pragma unroll
            for (int k = 0; k < B; k++) mn = min(mn, abs(a[k]));
        }
        if (__all_sync(FULL, mn >= TAUI[clog2(W)])) {
#pragma unroll 1
            for (int q0 = 0; q0 < V; q0 += B) {
                int a[B];
#pragma unroll
                for (int k = 0; k < B; k++) a[k] = ld(32 * (q0 + k) + lane);
                uint32_t w = 0;
#pragma unroll
                for (int k = 0; k < B; k++) {
                    const uint32_t b = __ballot_sync(FULL, a[k] < 0);
                    w = lane == k ? b : w;
                }
                if (lane < B) xw[q0 + lane] = w;
            }
            __syncwarp();
            return;
        }
    }
    if (t == T_REP) {
        int s0;
        if constexpr (V <= 64) {
            int acc[V];
#pragma unroll
            for (int q = 0; q < V; q++) acc[q] = ld(32 * q + lane);
#pragma unroll
            for (int hv = V / 2; hv >= 1; hv >>= 1)
#pragma unroll
                for (int q = 0; q < hv; q++) acc[q] = qa(acc[q + hv], acc[q]);
            s0 = acc[0];
        } else {
            // very wide repetition node (rare): fold in SC's pairing order
            // through the free child stage area, then in registers
#pragma unroll 1
            for (int hv = V / 2; hv >= 32; hv >>= 1)
#pragma unroll 1
                for (int q = 0; q < hv; q++) {
                    const int a = hv == V / 2 ? ld(32 * q + lane) : ch[32 * q + lane];
                    const int b = hv == V / 2 ? ld(32 * (q + hv) + lane) : ch[32 * (q + hv) + lane];
                    __syncwarp();
                    ch[32 * q + lane] = qa(b, a);
                    __syncwarp();
                }
            int acc[32];
#pragma unroll
            for (int q = 0; q < 32; q++) acc[q] = ch[32 * q + lane];
#pragma unroll
            for (int hv = 16; hv >= 1; hv >>= 1)
#pragma unroll
                for (int q = 0; q < hv; q++) acc[q] = qa(acc[q + hv], acc[q]);
            s0 = acc[0];
        }
#pragma unroll
        for (int hh = 16; hh >= 1; hh >>= 1) s0 = qa(__shfl_down_sync(FULL, s0, hh), s0);
        const uint32_t bits = __shfl_sync(FULL, s0, 0) < 0 ? FULL : 0u;
        for (int q = lane; q < V; q += 32) xw[q] = bits;
        __syncwarp();
        return;
    }
    if (tl == T_R0) {
        for (int q = lane; q < Vh; q += 32) xw[q] = 0u;
        __syncwarp();
    } else {
#pragma unroll 1
        for (int q0 = 0; q0 < Vh; q0 += B) {
            int a[B], b[B];
#pragma unroll
            for (int k = 0; k < B; k++) {
                a[k] = ld(32 * (q0 + k) + lane);
                b[k] = ld(32 * (q0 + k) + lane + W / 2);
            }
#pragma unroll
            for (int k = 0; k < B; k++) ch[32 * (q0 + k) + lane] = fq(a[k], b[k]);
        }
        __syncwarp();
        if constexpr (W / 2 > SE_UNR) wide<W / 2, false, SP>(st_end, xs, ty, fm, S, dS, d0 + 1, 2 * j0);
        else walk<SP>(reinterpret_cast<const int *>(st_end - W), xs, ty, fm, S, dS, d0 + 1, 2 * j0);
    }
    if (tr == T_R0) {
        for (int q = lane; q < Vh; q += 32) xw[Vh + q] = 0u;
        __syncwarp();
    } else {
#pragma unroll 1
        for (int q0 = 0; q0 < Vh; q0 += B) {
            int a[B], b[B];
            uint32_t sw[B];
#pragma unroll
            for (int k = 0; k < B; k++) {
                a[k] = ld(32 * (q0 + k) + lane);
                b[k] = ld(32 * (q0 + k) + lane + W / 2);
                sw[k] = xw[q0 + k];
            }
#pragma unroll
            for (int k = 0; k < B; k++) ch[32 * (q0 + k) + lane] = gq(a[k], b[k], (sw[k] >> lane) & 1u);
        }
        __syncwarp();
        if constexpr (W / 2 > SE_UNR) wide<W / 2, false, SP>(st_end, xs, ty, fm, S, dS, d0 + 1, 2 * j0 + 1);
        else walk<SP>(reinterpret_cast<const int *>(st_end - W), xs, ty, fm, S, dS, d0 + 1, 2 * j0 + 1);
    }
    for (int q = lane; q < Vh; q += 32) xw[q] ^= xw[Vh + q];
    __syncwarp();
}

// Entry: the node (d0, j0) of width W = S >> (d0 - dS), 32 <= W <= 2048, whose
// fp32 Q8.8 values are in the shared stage buffer at st_end - 2W; writes its
// partial-sum words to xs (S-local).  ty: S-local heap types; fm: the
// S-sub-tree's frozen-mask words.  One warp.
#ifndef SE_ROOT_INLINE
#define SE_ROOT_INLINE 1
#endif
// inlined into sc_decode_kernel (its only caller): c3 +5 %, c4 +6.6 %, c5 +1.8 %
// against the out-of-line call (profiles/r02/ab_uniform.txt)
#if SE_ROOT_INLINE
#define SE_ROOT_ATTR __forceinline__
#else
#define SE_ROOT_ATTR __noinline__
#endif
template <bool SP>
__device__ SE_ROOT_ATTR void root(float *st_end, uint32_t *xs, const uint8_t *ty, const uint32_t *fm, uint32_t S,
                                  int dS, int d0, uint32_t j0)
{
    const int lane = threadIdx.x & 31;
    const uint32_t W = S >> (d0 - dS);
    PQ_CHECK(W >= 32 && W <= S && d0 >= dS && ((j0 * W) & (S - 1)) + W <= S);
    PQ_JITTER();
    if (false) {
#if PQ_WIDE_WARP_LOG2 >= 14
    } else if (W == 16384) {
        wide<16384, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#endif
#if PQ_WIDE_WARP_LOG2 >= 13
    } else if (W == 8192) {
        wide<8192, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#endif
#if PQ_WIDE_WARP_LOG2 >= 12
    } else if (W == 4096) {
        wide<4096, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#endif
    } else if (W == 2048) {
        wide<2048, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
    } else if (W == 1024) {
        wide<1024, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#if SE_UNR < 512
    } else if (W == 512) {
        wide<512, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#endif
#if SE_UNR < 256
    } else if (W == 256) {
        wide<256, true, SP>(st_end, xs, ty, fm, S, dS, d0, j0);
#endif
    } else if (W >= 64) {
        // the node's fp32 codes -> int in place (batched: loads ahead of stores)
        float *nd = st_end - 2 * W;
#pragma unroll 1
        for (uint32_t i0 = 0; i0 < W; i0 += 256) {
            float a[8];
#pragma unroll
            for (int k = 0; k < 8; k++) a[k] = i0 + 32 * k < W ? nd[i0 + 32 * k + lane] : 0.0f;
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (i0 + 32 * k < W) reinterpret_cast<int *>(nd)[i0 + 32 * k + lane] = f2q(a[k]);
        }
        __syncwarp();
        walk<SP>(reinterpret_cast<const int *>(nd), xs, ty, fm, S, dS, d0, j0);
    } else {
        const uint32_t pos = (j0 * W) & (S - 1);
        const uint32_t bits = w32d<SP>(f2q((st_end - 64)[lane]), fm[pos >> 5]);
        if (lane == 0) xs[pos >> 5] = bits;
        __syncwarp();
    }
}

}  // namespace se
