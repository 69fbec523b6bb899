// codetable.cu -- the reference's binary code-table format (PQCT) read on the
// host side of the C ABI: construction.py:483-507 read_code_table with its
// checksum construction.py:458-459 (_checksum = BLAKE2b, 8-byte digest,
// little-endian).  The reference writes the file (write_code_table,
// construction.py:464-480); a C caller of the decoder reads it here and feeds
// the mask to pq_decoder_set_frozen_mask.
//
// Layout: "PQCT" | <HBBddI: version u16, n u8, channel tag u8, param f64,
// target FER f64, DE bins u32 | frozen mask, ceil(2^n / 8) bytes packed
// LSB-first (np.packbits bitorder="little") | u64 BLAKE2b-64 of everything
// before it.
//
// BLAKE2b is restated from its public specification (RFC 7693), unkeyed,
// digest length 8.

#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/polarsc.h"

int pq_set_error_text(int code, const char *msg);  // polarsc.cu

namespace {

const uint64_t B2_IV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                           0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                           0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

const uint8_t B2_SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr64(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }

inline void b2_g(uint64_t *v, int a, int b, int c, int d, uint64_t x, uint64_t y)
{
    v[a] = v[a] + v[b] + x;
    v[d] = rotr64(v[d] ^ v[a], 32);
    v[c] = v[c] + v[d];
    v[b] = rotr64(v[b] ^ v[c], 24);
    v[a] = v[a] + v[b] + y;
    v[d] = rotr64(v[d] ^ v[a], 16);
    v[c] = v[c] + v[d];
    v[b] = rotr64(v[b] ^ v[c], 63);
}

void b2_compress(uint64_t h[8], const uint8_t block[128], uint64_t t, bool last)
{
    uint64_t m[16], v[16];
    for (int i = 0; i < 16; i++) {
        uint64_t w = 0;
        for (int k = 7; k >= 0; k--) w = (w << 8) | block[8 * i + k];
        m[i] = w;
    }
    for (int i = 0; i < 8; i++) {
        v[i] = h[i];
        v[i + 8] = B2_IV[i];
    }
    v[12] ^= t;  // byte counter (messages < 2^64 bytes: high word stays 0)
    if (last) v[14] = ~v[14];
    for (int r = 0; r < 12; r++) {
        const uint8_t *s = B2_SIGMA[r];
        b2_g(v, 0, 4, 8, 12, m[s[0]], m[s[1]]);
        b2_g(v, 1, 5, 9, 13, m[s[2]], m[s[3]]);
        b2_g(v, 2, 6, 10, 14, m[s[4]], m[s[5]]);
        b2_g(v, 3, 7, 11, 15, m[s[6]], m[s[7]]);
        b2_g(v, 0, 5, 10, 15, m[s[8]], m[s[9]]);
        b2_g(v, 1, 6, 11, 12, m[s[10]], m[s[11]]);
        b2_g(v, 2, 7, 8, 13, m[s[12]], m[s[13]]);
        b2_g(v, 3, 4, 9, 14, m[s[14]], m[s[15]]);
    }
    for (int i = 0; i < 8; i++) h[i] ^= v[i] ^ v[i + 8];
}

// BLAKE2b, unkeyed, 8-byte digest, as a little-endian u64
uint64_t blake2b64(const uint8_t *data, size_t len)
{
    uint64_t h[8];
    memcpy(h, B2_IV, sizeof h);
    h[0] ^= 0x01010000ull ^ 8ull;  // param block: digest length 8, key length 0, fanout 1, depth 1
    uint8_t block[128];
    size_t off = 0;
    while (len - off > 128) {
        b2_compress(h, data + off, (uint64_t)(off + 128), false);
        off += 128;
    }
    memset(block, 0, sizeof block);
    if (len > off) memcpy(block, data + off, len - off);
    b2_compress(h, block, (uint64_t)len, true);
    return h[0];
}

int err(int code, const char *msg) { return pq_set_error_text(code, msg); }

}  // namespace

extern "C" {

uint64_t pq_blake2b64(const void *data, size_t len)
{
    return blake2b64(static_cast<const uint8_t *>(data), len);
}

int pq_read_code_table(const char *path, int *n_out, int *channel_tag, double *channel_param, double *target_fer,
                       int *bins, uint8_t *mask_out, size_t mask_len)
{
    if (!path) return err(-1, "path is NULL");
    FILE *f = fopen(path, "rb");
    if (!f) return err(-2, (std::string("cannot open code table: ") + path).c_str());
    std::vector<uint8_t> blob;
    uint8_t buf[65536];
    size_t got;
    while ((got = fread(buf, 1, sizeof buf, f)) > 0) blob.insert(blob.end(), buf, buf + got);
    fclose(f);
    const size_t head = 2 + 1 + 1 + 8 + 8 + 4;  // struct "<HBBddI"
    if (blob.size() < 4 + head + 8) return err(-3, "code table truncated");
    if (memcmp(blob.data(), "PQCT", 4) != 0) return err(-4, "bad code-table magic");
    const size_t body = blob.size() - 8;
    uint64_t stored = 0;
    for (int k = 7; k >= 0; k--) stored = (stored << 8) | blob[body + k];
    if (blake2b64(blob.data(), body) != stored) return err(-5, "code-table checksum mismatch");
    const uint8_t *p = blob.data() + 4;
    uint16_t version;
    uint8_t n, tag;
    double param, fer;
    uint32_t nbins;
    memcpy(&version, p, 2);
    n = p[2];
    tag = p[3];
    memcpy(&param, p + 4, 8);
    memcpy(&fer, p + 12, 8);
    memcpy(&nbins, p + 20, 4);
    if (version != 1) {
        char m[64];
        snprintf(m, sizeof m, "unsupported code-table version %u", (unsigned)version);
        return err(-6, m);
    }
    if (n > 30) return err(-3, "code table truncated");
    const size_t size = (size_t)1 << n, nbytes = (size + 7) / 8;
    if (4 + head + nbytes > body) return err(-3, "code table truncated");
    if (n_out) *n_out = n;
    if (channel_tag) *channel_tag = tag;
    if (channel_param) *channel_param = param;
    if (target_fer) *target_fer = fer;
    if (bins) *bins = (int)nbins;
    if (mask_out) {
        if (mask_len < size) return err(-1, "mask buffer shorter than 2^n");
        const uint8_t *mb = p + head;
        for (size_t i = 0; i < size; i++) mask_out[i] = (mb[i >> 3] >> (i & 7)) & 1u;
    }
    return 0;
}

}  // extern "C"
