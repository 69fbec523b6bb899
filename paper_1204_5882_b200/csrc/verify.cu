// verify.cu -- the verification step of bob_decode on the device (
// SURVEY.md 8(f) f3): x-hat = T(u-hat) comes out of the decoder, then a
// seed-keyed 64-bit hash of every frame's x-hat is compared with Alice's.
//
// Hash: XXH64 (SPEC.md:353's design decision: "a fixed, well-known 64-bit
// non-cryptographic hash, seed-keyed per session"), over the frame's packed
// words as little-endian bytes (4 * max(1, N/32) bytes: bit i = byte i>>3,
// bit i&7).  XXH64's four stripe accumulators are independent: lanes 0..3 of
// one warp each run one of them over the frame's 32-byte stripes (8 stripes of
// loads in flight per lane), lane 0 finishes (merge, length, tail, avalanche).
// One warp per frame; all frames of a batch in one launch.
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "polarsc.h"

// error text shared with the decoder's pq_last_error (polarsc.cu)
int pq_set_error_text(int code, const char *msg);

namespace {

constexpr uint64_t P1 = 0x9E3779B185EBCA87ull, P2 = 0xC2B2AE3D27D4EB4Full, P3 = 0x165667B19E3779F9ull,
                   P4 = 0x85EBCA77C2B2AE63ull, P5 = 0x27D4EB2F165667C5ull;

__host__ __device__ inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__host__ __device__ inline uint64_t xx_round(uint64_t acc, uint64_t in) { return rotl64(acc + in * P2, 31) * P1; }
__host__ __device__ inline uint64_t xx_merge(uint64_t h, uint64_t v) { return (h ^ xx_round(0, v)) * P1 + P4; }
__host__ __device__ inline uint64_t xx_avalanche(uint64_t h)
{
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}
// length, 8/4/1-byte tail and avalanche after the stripes (p: the tail bytes)
__host__ __device__ inline uint64_t xx_finish(uint64_t h, uint64_t len, const unsigned char *p, size_t rem)
{
    h += len;
    size_t i = 0;
    for (; i + 8 <= rem; i += 8) {
        uint64_t k = 0;
        for (int b = 7; b >= 0; b--) k = (k << 8) | p[i + b];
        h ^= xx_round(0, k);
        h = rotl64(h, 27) * P1 + P4;
    }
    if (i + 4 <= rem) {
        const uint64_t k = (uint64_t)p[i] | ((uint64_t)p[i + 1] << 8) | ((uint64_t)p[i + 2] << 16) |
                           ((uint64_t)p[i + 3] << 24);
        h ^= k * P1;
        h = rotl64(h, 23) * P2 + P3;
        i += 4;
    }
    for (; i < rem; i++) {
        h ^= (uint64_t)p[i] * P5;
        h = rotl64(h, 11) * P1;
    }
    return xx_avalanche(h);
}

__global__ void __launch_bounds__(128) xxh64_frames_kernel(const uint32_t *x, uint32_t wpf, int frames, uint64_t seed,
                                                           uint64_t *hash_out, const uint64_t *expect,
                                                           uint8_t *verified, unsigned int *n_discarded)
{
    const int warp = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    const int lane = threadIdx.x & 31;
    if (warp >= frames) return;
    const uint32_t *fw = x + (size_t)warp * wpf;
    const uint64_t len = 4ull * wpf;
    const uint32_t nstripes = (uint32_t)(len / 32);
    uint64_t v = 0;
    if (lane < 4 && nstripes > 0) {
        v = lane == 0 ? seed + P1 + P2 : lane == 1 ? seed + P2 : lane == 2 ? seed : seed - P1;
        const uint2 *src = reinterpret_cast<const uint2 *>(fw) + lane;  // 8-byte lane of stripe 0
        uint32_t s = 0;
        for (; s + 8 <= nstripes; s += 8) {
            uint2 w[8];
#pragma unroll
            for (int q = 0; q < 8; q++) w[q] = __ldg(src + 4 * (s + q));
#pragma unroll
            for (int q = 0; q < 8; q++) v = xx_round(v, ((uint64_t)w[q].y << 32) | w[q].x);
        }
        for (; s < nstripes; s++) {
            const uint2 w = __ldg(src + 4 * s);
            v = xx_round(v, ((uint64_t)w.y << 32) | w.x);
        }
    }
    const uint64_t v1 = __shfl_sync(0xffffffffu, v, 0), v2 = __shfl_sync(0xffffffffu, v, 1);
    const uint64_t v3 = __shfl_sync(0xffffffffu, v, 2), v4 = __shfl_sync(0xffffffffu, v, 3);
    if (lane != 0) return;
    uint64_t h;
    if (nstripes > 0) {
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xx_merge(h, v1);
        h = xx_merge(h, v2);
        h = xx_merge(h, v3);
        h = xx_merge(h, v4);
    } else {
        h = seed + P5;
    }
    const size_t done = 32ull * nstripes;
    h = xx_finish(h, len, reinterpret_cast<const unsigned char *>(fw) + done, (size_t)(len - done));
    if (hash_out) hash_out[warp] = h;
    if (expect) {
        const bool ok = h == expect[warp];
        if (verified) verified[warp] = ok ? 1 : 0;
        if (!ok && n_discarded) atomicAdd(n_discarded, 1u);
    }
}

int launch_hash(const uint32_t *x, int n, int frames, uint64_t seed, uint64_t *hash_out, const uint64_t *expect,
                uint8_t *verified, unsigned int *n_discarded, void *stream)
{
    if (n < 1 || n > 30) return pq_set_error_text(-1, "n outside 1..30");
    if (frames < 0) return pq_set_error_text(-1, "frames < 0");
    if (!x && frames > 0) return pq_set_error_text(-1, "x_words is NULL");
    if (frames == 0) return 0;
    const uint32_t wpf = n >= 5 ? (1u << n) / 32u : 1u;
    const int warps_per_block = 4;
    const int blocks = (frames + warps_per_block - 1) / warps_per_block;
    xxh64_frames_kernel<<<blocks, 32 * warps_per_block, 0, (cudaStream_t)stream>>>(x, wpf, frames, seed, hash_out,
                                                                                  expect, verified, n_discarded);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return pq_set_error_text(1 + (int)e, cudaGetErrorString(e));
    return 0;
}

}  // namespace

extern "C" {

uint64_t pq_xxh64(const void *data, size_t len, uint64_t seed)
{
    const unsigned char *p = static_cast<const unsigned char *>(data);
    uint64_t h;
    size_t i = 0;
    if (len >= 32) {
        uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
        for (; i + 32 <= len; i += 32) {
            uint64_t k[4];
            for (int q = 0; q < 4; q++) {
                k[q] = 0;
                for (int b = 7; b >= 0; b--) k[q] = (k[q] << 8) | p[i + 8 * q + b];
            }
            v1 = xx_round(v1, k[0]);
            v2 = xx_round(v2, k[1]);
            v3 = xx_round(v3, k[2]);
            v4 = xx_round(v4, k[3]);
        }
        h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
        h = xx_merge(h, v1);
        h = xx_merge(h, v2);
        h = xx_merge(h, v3);
        h = xx_merge(h, v4);
    } else {
        h = seed + P5;
    }
    return xx_finish(h, (uint64_t)len, p + i, len - i);
}

int pq_hash_frames(const uint32_t *x_words, int n, int frames, uint64_t seed, uint64_t *hash_out, void *stream)
{
    if (!hash_out && frames > 0) return pq_set_error_text(-1, "hash_out is NULL");
    return launch_hash(x_words, n, frames, seed, hash_out, nullptr, nullptr, nullptr, stream);
}

int pq_verify_frames(const uint32_t *x_words, int n, int frames, uint64_t seed, const uint64_t *expect,
                     uint8_t *verified, unsigned int *n_discarded, void *stream)
{
    if (!expect && frames > 0) return pq_set_error_text(-1, "expected hashes are NULL");
    return launch_hash(x_words, n, frames, seed, nullptr, expect, verified, n_discarded, stream);
}

}  // extern "C"
