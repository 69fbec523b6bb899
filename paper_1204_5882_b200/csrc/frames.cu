// frames.cu -- seeded BSC trial inputs generated on the device:
// the frames of bench.run_trials without a host pass.
//
// The input contract is the reference's numpy call sequence (channel.py:66-73,
// :116-125, with the frame seed convention of SURVEY.md 8(d)):
//   x     = make_rng(seed, 2j).integers(0, 2, N, dtype=uint8)
//   flips = make_rng(seed, 2j + 1).random(N) < p,      y = x ^ flips
// where make_rng(seed, s) = Generator(PCG64(SeedSequence((seed, s)))).  All of
// it is integer arithmetic, restated here from the published algorithms:
//   * SeedSequence (O'Neill's seed_seq_fe128 as numpy pins it): the entropy
//     words are hashed into a 4-word pool, 8 output words seed PCG64;
//   * PCG64 = PCG XSL-RR 128/64: state' = state * M + inc (mod 2^128), output
//     rotr64(hi ^ lo, state' >> 122); jump-ahead by the usual O(log k)
//     affine-power recurrence, so every thread starts at its own draw;
//   * integers(0, 2, dtype=uint8) takes one byte of the stream per element
//     (the 64-bit draws in little-endian byte order) and keeps its top bit
//     (Lemire's bounded method at range 2 never rejects);
//   * random() = (draw >> 11) * 2^-53, so "random() < p" is the integer test
//     (draw >> 11) < ceil(p * 2^53), exact for every double p.
// tests/test_frames.py pins the host seeding against numpy and the device
// frames against channel.frame() and the reference's golden vectors.
// BIAWGN noise (Generator.normal: a 256-layer ziggurat with numpy's own
// tables and libm tails) is not restated; those trials keep the threaded
// host generator (channel.frames_batch).
#include <cmath>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "polarsc.h"

int pq_set_error_text(int code, const char *msg);

namespace {

typedef unsigned __int128 u128;

__host__ __device__ inline u128 pcg_mult()
{
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

struct Pcg {
    u128 state, inc;
};

__host__ __device__ inline uint64_t pcg_next(Pcg &g)
{
    g.state = g.state * pcg_mult() + g.inc;
    const uint64_t hi = (uint64_t)(g.state >> 64), lo = (uint64_t)g.state;
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// state after `delta` further steps
__host__ __device__ inline void pcg_advance(Pcg &g, uint64_t delta)
{
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = g.inc;
    while (delta) {
        if (delta & 1u) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    g.state = acc_mult * g.state + acc_plus;
}

// SeedSequence(entropy words).generate_state(8 x uint32) -> PCG64 (state, inc)
Pcg pcg_seed_words(const uint32_t *entropy, int n_entropy)
{
    const uint32_t MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
    const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
    uint32_t hc = 0x43b0d7e5u;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= MULT_A;
        v *= hc;
        v ^= v >> 16;
        return v;
    };
    auto mix = [&](uint32_t x, uint32_t y) {
        uint32_t r = MIX_L * x - MIX_R * y;
        r ^= r >> 16;
        return r;
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < n_entropy ? entropy[i] : 0u);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (int s = 4; s < n_entropy; s++)
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(entropy[s]));
    uint32_t w[8], hb = INIT_B;
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3] ^ hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    uint64_t v64[4];
    for (int i = 0; i < 4; i++) v64[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const u128 initstate = ((u128)v64[0] << 64) | v64[1], initseq = ((u128)v64[2] << 64) | v64[3];
    Pcg g;
    g.inc = (initseq << 1) | 1u;
    g.state = 0;
    g.state = g.state * pcg_mult() + g.inc;
    g.state += initstate;
    g.state = g.state * pcg_mult() + g.inc;
    return g;
}

// numpy's coercion of a non-negative integer to uint32 words (at least one)
int int_words(uint64_t v, uint32_t *out)
{
    out[0] = (uint32_t)v;
    if ((v >> 32) == 0) return 1;
    out[1] = (uint32_t)(v >> 32);
    return 2;
}

Pcg pcg_seed(uint64_t seed, uint64_t stream)
{
    uint32_t e[4];
    int k = int_words(seed, e);
    k += int_words(stream, e + k);
    return pcg_seed_words(e, k);
}

struct FrameSeeds {  // per frame: the bit stream's and the noise stream's generators
    Pcg bits, noise;
};

constexpr int WPT = 4;  // output words per thread

__global__ void __launch_bounds__(256) bsc_frames_kernel(const FrameSeeds *seeds, uint32_t N, uint32_t wpf,
                                                         uint64_t thresh, uint32_t *xw, uint32_t *yw)
{
    const uint32_t frame = blockIdx.y;
    const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) * WPT;
    if (w0 >= wpf) return;
    Pcg gb = seeds[frame].bits, gn = seeds[frame].noise;
    pcg_advance(gb, (uint64_t)w0 * 4u);   // one byte per bit: 8 bits per draw
    pcg_advance(gn, (uint64_t)w0 * 32u);  // one draw per flip
    for (uint32_t w = w0; w < w0 + WPT && w < wpf; w++) {
        uint32_t x = 0, e = 0;
        for (int q = 0; q < 4; q++) {
            if (32u * w + 8u * q >= N) break;
            // bytes of the draw in little-endian order, top bit of each
            const uint64_t v = pcg_next(gb) & 0x8080808080808080ull;
            x |= (uint32_t)((v * 0x0002040810204081ull) >> 56) << (8 * q);
        }
        for (int b = 0; b < 32; b++) {
            if (32u * w + b >= N) break;
            e |= (uint32_t)((pcg_next(gn) >> 11) < thresh) << b;
        }
        if (N < 32u * (w + 1)) x &= (1u << (N & 31u)) - 1u;
        xw[(size_t)frame * wpf + w] = x;
        yw[(size_t)frame * wpf + w] = x ^ e;
    }
}

}  // namespace

extern "C" int pq_pcg64_seed(uint64_t seed, uint64_t stream, uint64_t out[4])
{
    if (!out) return pq_set_error_text(-1, "pq_pcg64_seed: null output");
    const Pcg g = pcg_seed(seed, stream);
    out[0] = (uint64_t)(g.state >> 64);
    out[1] = (uint64_t)g.state;
    out[2] = (uint64_t)(g.inc >> 64);
    out[3] = (uint64_t)g.inc;
    return 0;
}

extern "C" int pq_bsc_frames(int n, uint64_t seed, uint64_t j0, int frames, double p, uint32_t *x_words,
                             uint32_t *y_words, void *stream)
{
    if (n < 0 || n > 30) return pq_set_error_text(-1, "pq_bsc_frames: n out of range");
    if (frames < 1 || !x_words || !y_words) return pq_set_error_text(-1, "pq_bsc_frames: bad arguments");
    if (!(p >= 0.0 && p <= 0.5)) return pq_set_error_text(-1, "pq_bsc_frames: p must be in [0, 0.5]");
    if (j0 + (uint64_t)frames > (1ull << 62)) return pq_set_error_text(-1, "pq_bsc_frames: frame index out of range");
    const uint32_t N = 1u << n, wpf = N >= 32 ? N / 32 : 1;
    cudaStream_t st = (cudaStream_t)stream;
    if (frames > 65535) return pq_set_error_text(-1, "pq_bsc_frames: at most 65535 frames per call");
    std::vector<FrameSeeds> h(frames);
    FrameSeeds *d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, sizeof(FrameSeeds) * frames, st);
    if (e != cudaSuccess) return pq_set_error_text((int)e, cudaGetErrorString(e));
    for (int f = 0; f < frames; f++) {
        h[f].bits = pcg_seed(seed, 2 * (j0 + f));
        h[f].noise = pcg_seed(seed, 2 * (j0 + f) + 1);
    }
    // random() < p  <=>  (draw >> 11) < ceil(p * 2^53)   (p * 2^53 is exact)
    const uint64_t thresh = (uint64_t)std::ceil(std::ldexp(p, 53));
    // pageable source: the call returns once the block is staged, so h may go
    e = cudaMemcpyAsync(d, h.data(), sizeof(FrameSeeds) * frames, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        const uint32_t threads = 256, per_block = threads * WPT;
        dim3 grid((wpf + per_block - 1) / per_block, (unsigned)frames);
        bsc_frames_kernel<<<grid, threads, 0, st>>>(d, N, wpf, thresh, x_words, y_words);
        e = cudaGetLastError();
    }
    cudaFreeAsync(d, st);
    return e == cudaSuccess ? 0 : pq_set_error_text((int)e, cudaGetErrorString(e));
}
