/*
 * polarsc.h -- C ABI of the B200-native polar-code SC decoder.
 *
 * Plain pointers and sizes only; no torch types.  Every device pointer is
 * caller-owned CUDA device memory; every call is stream-ordered and
 * asynchronous (no implicit device synchronisation).  A handle owns its
 * device scratch (allocated once in pq_decoder_create, never inside decode)
 * and is not thread-safe: use one handle per host thread / stream
 * ("a decoder instance owns its scratch buffers and is
 * single-threaded; instances are independent").
 *
 * Bit vectors (u-domain and x-domain BitBlocks) are packed
 * uint32 words, bit i of a frame at word i>>5, bit position i&31 (LSB first),
 * the same order as the reference's code-table mask packing
 * (np.packbits(..., bitorder="little"), construction.py:476 / :668).
 * Frames are stored frame-major: frame f's words start at f * (N/32)
 * (N >= 32; for N < 32 each frame still occupies one word).
 *
 * Return codes: 0 = ok; negative = invalid argument (Python: ValueError);
 * positive = CUDA/runtime failure (Python: RuntimeError).  pq_last_error()
 * returns the text of the most recent failure on the calling thread.
 *
 * Reference interfaces replaced (the reference's polar_core is specified in
 * /root/reference/SPEC.md but not implemented; its construction->decoding
 * contract is PolarCode in pkg/src/polarqkd/construction.py):
 */
#ifndef POLARSC_H
#define POLARSC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQ_ABI_VERSION 1

/* f-function modes.  EXACT is the SPEC's phi-form boxplus (SPEC.md:243,
 * SPEC.md:270 "exact phi-based form, not min-sum"); MINSUM is the opt-in
 * approximation named by the north star (no reference counterpart).        */
#define PQ_F_EXACT 0
#define PQ_F_MINSUM 1
/* FAST: the same exact boxplus evaluated with the SFU's ex2/lg2/rcp
 * approximations (max relative error ~1e-6 vs f64; ~1.7x cheaper); its parity
 * is the north star's tolerance rule against the f64 oracle, not bit-exactness
 * with the fp32 mirror.                                                    */
#define PQ_F_FAST 2
/* FIXED: SPEC.md's sc_decode_fixed -- the reference's
 * default decode path: saturating Q8.8 LLRs (raw = sat(rint(256
 * L)) of the fp32 channel LLR), f = the exact boxplus by lookup in a 4097-entry
 * table uniform on [0, 16]: sgn a sgn b max(0, min(|a|,|b|) + C[|a|+|b|] -
 * C[||a|-|b||]), C[k] = rint(256 ln(1 + e^(-k/256))) (oracle/sc_oracle.c says
 * why not the literal double phi lookup), saturating g.  Integer-exact: the
 * GPU reproduces the C oracle's decisions and stage values bit for bit.     */
#define PQ_F_FIXED 3

/* options for pq_decoder_set_option */
#define PQ_OPT_SSC 1          /* 1 (default): skip rate-0/rate-1/repetition sub-trees
                                 (decision-exact); 0: plain SC          */
#define PQ_OPT_SUBTREE_LOG2 2 /* log2 of the shared-memory sub-tree width S; 0 = auto  */
#define PQ_OPT_FMODE 3        /* PQ_F_EXACT / PQ_F_MINSUM / PQ_F_FAST / PQ_F_FIXED     */
#define PQ_OPT_PROFILE 4      /* 1: record per-frame clock64 cycles per step class      */
#define PQ_OPT_WARP_LOG2 5    /* log2 of the widest node decoded by one warp (5..9, default 9) */
#define PQ_OPT_CLUSTER 6      /* CTAs per frame for the upper band (a thread-block cluster):
                                 0 = auto (more when frames < SMs), or 1, 2, 4, 8; it only
                                 applies when the block has an upper band and S >= 2048   */
#define PQ_OPT_THREADS 7      /* threads per CTA: 0 = auto (256 up to 2 frames per SM, else
                                 128 so that 4 frames share an SM; 512 when a clustered
                                 batch leaves one CTA per SM), or 64 / 128 / 256          */

#define PQ_OPT_TIMING 8       /* 1: bracket every decode's sc_decode_kernel launch with CUDA
                                 events on the launching stream (a ring of the last 64
                                 decodes, read with pq_decoder_kernel_times); 0: off     */

/* slots of the per-frame profile record (pq_decoder_read_profile) */
#define PQ_PROF_SLOTS 16

typedef struct pq_decoder pq_decoder;

/* Create a decoder for block length N = 2^n (1 <= n <= 25) and up to
 * max_frames frames per call on CUDA device `device`.
 * Replaces: constructing a polar_core decoder instance.  */
int pq_decoder_create(pq_decoder **out, int n, int max_frames, int f_mode, int device);

/* Install the frozen set: mask_host[i] = 1 if position i is frozen, length
 * 2^n bytes -- exactly PolarCode.frozen_mask (construction.py:96-108).
 * The mask is copied; the handle is immutable w.r.t. the code afterwards. */
int pq_decoder_set_frozen_mask(pq_decoder *h, const uint8_t *mask_host);

int pq_decoder_set_option(pq_decoder *h, int key, int value);
int pq_decoder_get_option(const pq_decoder *h, int key);

/* Batched float SC decode.
 * Replaces: sc_decode(code, llrs, frozen_values) -> u_hat,
 *           applied to `frames` independent blocks.
 *   llr       [frames][N] fp32 channel LLRs (positive favours 0, channel.py:14)
 *   frozen_u  [frames][N/32] packed u-domain words whose bits at frozen
 *             positions are the revealed frozen values;
 *             bits at information positions are ignored.  NULL = all zero.
 *   u_hat     [frames][N/32] out: decoded u (frozen positions carry exactly
 *             the revealed values).  May be NULL.
 *   x_hat     [frames][N/32] out: x_hat = polar_transform(u_hat) (what
 *             bob_decode re-encodes).  May be NULL.
 *   stream    cudaStream_t (NULL = legacy default stream).                 */
int pq_sc_decode_f32(pq_decoder *h, const float *llr, const uint32_t *frozen_u,
                     uint32_t *u_hat, uint32_t *x_hat, int frames, void *stream);

/* Same, plain SC (no sub-tree shortcuts) with every stage LLR written to
 * dump [frames][n+1][N]: dump[f][d][j*W + t] = element t of node j at depth
 * d, W = N >> d (the canonical stage dump of SURVEY.md App. A.6), in the
 * coset-shifted domain (each node's LLRs are sign-flipped by
 * the node-level codeword of the frozen values).  Parity/debug only.     */
int pq_sc_decode_f32_dump(pq_decoder *h, const float *llr, const uint32_t *frozen_u,
                          uint32_t *u_hat, uint32_t *x_hat, float *dump, int frames,
                          void *stream);

/* SPEC.md's sc_decode_fixed(code, llrs-fixed, frozen_values):
 * channel LLRs given as saturating Q8.8 raw codes (int16, |raw| <= 32767,
 * e.g. sat(rint(256 L))), [frames][N] frame-major.  Needs a PQ_F_FIXED
 * decoder; otherwise as pq_sc_decode_f32 (half its input bytes).          */
int pq_sc_decode_q88(pq_decoder *h, const int16_t *llr_q88, const uint32_t *frozen_u,
                     uint32_t *u_hat, uint32_t *x_hat, int frames, void *stream);

/* BSC front end fused into the decoder's level-0 reads: y_bits are Bob's
 * received bits packed like u_hat; the channel LLR (1-2y)*llr_mag is formed
 * on the fly (channel.py:142-147 with magnitude min(30, ln((1-p)/p))).
 * Replaces: channel_llr(Bsc(p), obs) followed by sc_decode (bob_decode's
 * first two steps).                                          */
int pq_sc_decode_bsc(pq_decoder *h, const uint32_t *y_bits, float llr_mag,
                     const uint32_t *frozen_u, uint32_t *u_hat, uint32_t *x_hat, int frames,
                     void *stream);

/* x = u F^{(x)n} over GF(2), natural order, involution, on packed frames.
 * in and out may alias.  Replaces: polar_transform(u),
 * also alice_disclose's u = polar_transform(x).             */
int pq_polar_transform(const uint32_t *in, uint32_t *out, int n, int frames, void *stream);

/* Verification step of bob_decode ("returns Verified if
 * hash(x_hat) equals verification_hash, else Discarded").  The hash is
 * XXH64 ("a fixed, well-known 64-bit non-cryptographic hash,
 * seed-keyed per session") of each frame's packed words read as
 * little-endian bytes (4 * max(1, N/32) bytes), seed = the session key.
 * Replaces: the hash(...) inside alice_disclose and
 * bob_decode's comparison, batched over frames on the
 * device.
 *   pq_hash_frames:   hash_out[f] = XXH64(frame f)
 *   pq_verify_frames: verified[f] = (XXH64(frame f) == expect[f]) (nullable),
 *                     *n_discarded += #mismatches (device counter, nullable)
 *   pq_xxh64:         the same hash on the host (CPU, any byte string).   */
int pq_hash_frames(const uint32_t *x_words, int n, int frames, uint64_t seed, uint64_t *hash_out,
                   void *stream);
int pq_verify_frames(const uint32_t *x_words, int n, int frames, uint64_t seed, const uint64_t *expect,
                     uint8_t *verified, unsigned int *n_discarded, void *stream);
uint64_t pq_xxh64(const void *data, size_t len, uint64_t seed);

/* Density evolution on the GPU (the construction service's hot loop,
 * SURVEY.md 8(f) f2).  Replaces: density_evolution(ch, n, quant, prune_z_eps,
 * prune_i_eps, mass_floor) (construction.py:313-391) with its f/g transforms
 * (_f_scatter / f_self / g_self, construction.py:138-158, :206-248) and the
 * pruned-subtree fill (construction.py:302-310).  The grid tables are the
 * reference's own (_GridOps, construction.py:164-190), computed on the host
 * and passed in: f_idx / f_whi are (bins-1)^2 row-major, z_weights / i_loss
 * have bins-1 entries.  pq_de_run takes the base density (bins+1 slots:
 * -inf, interior, +inf) and writes pe[2^n] (host memory); synchronous.     */
typedef struct pq_de pq_de;
int pq_de_create(pq_de **out, int bins, double z_lo_bound, const int32_t *f_idx, const double *f_whi,
                 const double *z_weights, const double *i_loss, int device);
int pq_de_run(pq_de *h, const double *base_density, int n, double prune_z_eps, double prune_i_eps,
              double mass_floor, double *pe_out);
int pq_de_destroy(pq_de *h);

/* Read a PQCT code-table file -- the reference's binary frozen-set format.
 * Replaces: read_code_table(path) (construction.py:483-507), with its
 * BLAKE2b-64 checksum (construction.py:458-459) and the same rejections
 * (return codes: -3 "code table truncated", -4 "bad code-table magic",
 * -5 "code-table checksum mismatch", -6 "unsupported code-table version",
 * -2 unreadable file, -1 bad arguments; the text is in pq_last_error()).
 * Outputs are nullable; mask_out (mask_len >= 2^n bytes) receives
 * PolarCode.frozen_mask, 1 = frozen -- exactly what
 * pq_decoder_set_frozen_mask takes.  Host only, no device needed.         */
int pq_read_code_table(const char *path, int *n, int *channel_tag, double *channel_param,
                       double *target_fer, int *bins, uint8_t *mask_out, size_t mask_len);
/* The table's checksum: BLAKE2b (RFC 7693), unkeyed, 8-byte digest, as a
 * little-endian u64 (construction.py:458-459).                             */
uint64_t pq_blake2b64(const void *data, size_t len);

/* Seeded BSC trial inputs on the device (the frames of
 * bench.run_trials).  Frame j0 + f reproduces the reference's
 * numpy call sequence bit for bit (channel.py:66-73 make_rng, :116-125
 * transmit):
 *   x = make_rng(seed, 2j).integers(0, 2, N, dtype=uint8)
 *   y = x ^ (make_rng(seed, 2j + 1).random(N) < p)
 * packed LSB-first into x_words / y_words [frames][max(1, N/32)] (device).
 * Stream-ordered.  pq_pcg64_seed is the host half: PCG64's (state, inc) after
 * seeding from SeedSequence((seed, stream)), as {state_hi, state_lo, inc_hi,
 * inc_lo} -- numpy's bit_generator.state.  BIAWGN noise is not generated on
 * the device (see csrc/frames.cu).                                          */
int pq_bsc_frames(int n, uint64_t seed, uint64_t j0, int frames, double p, uint32_t *x_words,
                  uint32_t *y_words, void *stream);
int pq_pcg64_seed(uint64_t seed, uint64_t stream, uint64_t out_state_inc[4]);

/* Copy the per-frame cycle profile of the last decode (PQ_OPT_PROFILE=1):
 * out[frame][PQ_PROF_SLOTS] = {upper f, upper g, upper other, shared f,
 * shared g, shared other, warp sub-trees, type staging, rate-1, total,
 * #warp sub-trees, #block nodes, ...}.  Synchronous.  Diagnostics only. */
int pq_decoder_read_profile(const pq_decoder *h, unsigned long long *out, int frames);

/* Evaluate the signed f (check-node combine) of mode f_mode elementwise on
 * device arrays: out[i] = f(a[i], b[i]).  Diagnostics / parity tests.     */
int pq_debug_fmag(int f_mode, const float *a, const float *b, float *out, int n, void *stream);

/* Bytes of device scratch owned by the handle. */
size_t pq_decoder_workspace_bytes(const pq_decoder *h);

/* Durations (ms) of the sc_decode_kernel launches of the last `count` decodes
 * made with PQ_OPT_TIMING = 1 (oldest first; count <= 64 and <= the number
 * timed since the option was set).  Waits for those launches to finish.
 * Measurement only (bench.py's roofline): the events sit on the launching
 * stream right before and after the kernel.                               */
int pq_decoder_kernel_times(pq_decoder *h, float *ms_out, int count);

/* Number of kernels the last decode call launched (for bench accounting). */
int pq_decoder_last_launches(const pq_decoder *h);

/* CTAs per frame (thread-block cluster size) of the last decode launch. */
int pq_decoder_last_ctas_per_frame(const pq_decoder *h);

/* Launch shape of the last decode: log2 of the shared-memory sub-tree width
 * S, threads per CTA, CTAs per frame (any pointer may be NULL).            */
int pq_decoder_last_config(const pq_decoder *h, int *log2S, int *threads_per_cta, int *ctas_per_frame);

int pq_decoder_destroy(pq_decoder *h);

const char *pq_last_error(void);
int pq_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* POLARSC_H */
