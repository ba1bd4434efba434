/* xsum.h — C-ABI of the B200 superaccumulator reduction (libxsum.so).
 *
 * Exact summation of IEEE-754 binary64 values after Goodrich & Eldawy,
 * "Parallel Algorithms for Summing Floating-Point Numbers" (arXiv 1605.05436).
 * Citations "PAPER.md:L" are line numbers of the paper's LaTeX source.
 *
 * Problem (§1): given X = {x_1..x_n}, compute the floating-point
 * number S_n* that faithfully rounds S_n = sum x_i. This library returns the
 * round-to-nearest-even double of the EXACT sum (one of the faithful results; the
 * "correctly rounded" sum of §5) together with the exact sum
 * itself as a canonical two's-complement integer image.
 *
 * Representation (§2): a superaccumulator is a vector of signed
 * integer digits Y_j with value sum_j Y_j * R^j * 2^-1074, radix R = 2^52
 * (XSUM_RADIX_BITS), XSUM_NDIGITS = 42 digits (2184 bits >= 1074 + 1024 + 63:
 * enough for any n < 2^63). A state is (alpha,beta)-regularized
 * with alpha = beta = R-1 (|Y_j| <= R-1, Lemma 1), which makes
 * adding two states carry-free.
 *
 * Conventions (all entry points):
 *   - Pointers named d_* are DEVICE pointers (cudaMalloc'd or torch tensors) on the
 *     handle's device; h_* are HOST pointers. The caller owns every buffer passed in.
 *   - Entry points without a handle (segments, strided reductions) run on the calling
 *     thread's current CUDA device; their device pointers must be on it.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are asynchronous and stream-ordered; a buffer must stay valid until
 *     the stream passes the call. One handle is used by one stream at a time.
 *   - Functions return a status code and never abort or throw across the ABI.
 *     Argument errors are detected on the host before anything is enqueued.
 *   - NaN / +-Inf inputs are not errors: they set sticky flags (R10).
 *   - No CPU fallback exists: every arithmetic step runs in CUDA kernels built
 *     for sm_100a.
 *   - The accumulate launches (xsum_accumulate*, xsum_sum*, xsum_sum_allreduce) of less than
 *     1 GiB of input use programmatic dependent launch: their blocks may become resident while
 *     the previous kernel in the stream is finishing, but every block waits for that kernel's
 *     completion (griddepcontrol.wait) before its first input load, so data written by any
 *     preceding stream operation is complete and visible, as with ordinary stream order.
 *     XSUM_NO_PDL=1 in the environment disables it.
 */
#ifndef XSUM_H
#define XSUM_H

#if defined(__GNUC__)
#define XSUM_API __attribute__((visibility("default")))
#else
#define XSUM_API
#endif

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum xsum_status {
    XSUM_OK = 0,
    XSUM_EINVAL = 1,     /* null/misaligned pointer, bad size, wrong device, too-small buffer */
    XSUM_ECAPACITY = 2,  /* total count would exceed 2^63-1 summands */
    XSUM_ECUDA = 3,      /* a CUDA runtime call or kernel launch failed */
    XSUM_EMISMATCH = 4,  /* a merged state image had a wrong header (magic/version/radix) */
    XSUM_ENOMEM = 5      /* host allocation failed */
} xsum_status;

/* Element formats (xsum_sum_segments_ex, xsum_accumulate_host_ex). */
#define XSUM_DT_F64 0   /* IEEE binary64 */
#define XSUM_DT_F32 1   /* IEEE binary32 */
#define XSUM_DT_F16 2   /* IEEE binary16 (bit patterns) */
#define XSUM_DT_BF16 3  /* bfloat16 (bit patterns) */

#define XSUM_RADIX_BITS 52          /* w: R = 2^52 */
#define XSUM_NDIGITS 42             /* D */
#define XSUM_STATE_BYTES 384        /* packed state image, see below */
#define XSUM_CANON_LIMBS 34         /* canonical image: 34 x u64 = 2176-bit two's complement */
#define XSUM_MAGIC 0x4D555358u      /* "XSUM" little-endian */
#define XSUM_VERSION 1u

/* Result / state flag bits (xsum_result.flags, state header flags). */
#define XSUM_F_NAN 1u        /* a NaN was summed */
#define XSUM_F_PINF 2u       /* +Inf was summed */
#define XSUM_F_NINF 4u       /* -Inf was summed */
#define XSUM_F_OVERFLOW 8u   /* the finite exact sum rounds beyond DBL_MAX (result +-Inf) */
#define XSUM_F_INEXACT 16u   /* the finite exact sum is not representable */
#define XSUM_F_MISMATCH 32u  /* a merged state image was rejected (header mismatch) */
#define XSUM_F_OVERFLOW32 64u /* the binary32 rounding (value_f32) overflowed to +-Inf */
#define XSUM_F_INEXACT32 128u /* the binary32 rounding differs from the exact finite sum */
#define XSUM_F_PEER_TIMEOUT 256u /* fused multi-GPU step: a peer's state did not arrive within ~2 s;
                                   the value is NOT the group's sum (xsum_sum_allreduce) */
#define XSUM_F_CAPACITY 512u /* a merge (or an accumulate after a merge whose count the host had not
                                yet seen) took the summand count past 2^63-1: the count saturates at
                                2^63-1 and the state is no longer a valid checkpoint image; the
                                digits stay exact (int64 top digit) */
#define XSUM_TOP_DIGIT_MAX (1ll << 29) /* |digit[41]| bound: |A| < 2^(1074+1024+63) = 2^2161 and
                                          R^41 = 2^2132 (R7) */

/* Packed state image (XSUM_STATE_BYTES, little-endian). Exactly mergeable in any
 * order; it is also the checkpoint format and what ranks exchange.
 *   offset 0  u32 magic = XSUM_MAGIC      offset 4  u16 version = XSUM_VERSION
 *   offset 6  u8  w = 52                  offset 7  u8  ndigits = 42
 *   offset 8  u32 flags (XSUM_F_NAN|PINF|NINF|MISMATCH; CAPACITY / PEER_TIMEOUT make the image
 *             invalid as a checkpoint)
 *   offset 12 u32 reserved (0)            offset 16 u64 count (summands so far)
 *   offset 24 i64 digit[42], digit j worth R^j * 2^-1074, |digit| <= R-1 (j < 41),
 *             |digit[41]| <= XSUM_TOP_DIGIT_MAX (merges reject images outside these bounds)
 *   offset 360..383 zero padding */
typedef struct xsum_state_image {
    uint32_t magic;
    uint16_t version;
    uint8_t w;
    uint8_t ndigits;
    uint32_t flags;
    uint32_t reserved;
    uint64_t count;
    int64_t digit[XSUM_NDIGITS];
    uint8_t pad[XSUM_STATE_BYTES - 24 - 8 * XSUM_NDIGITS];
} xsum_state_image;

/* Sparse state image: the paper's sparse superaccumulator keeps only the
 * active (non-zero) components. Header (24 bytes, little-endian) followed by
 * nnz u64 records (digit << 6) | index in strictly ascending index order, digit the
 * regularized component (|digit| <= R-1; the top digit's magnitude is bounded by the value),
 * stored two's complement in the top 58 bits. Size 24 + 8*nnz <= XSUM_SPARSE_MAX_BYTES; narrow
 * exponent ranges give a few records. */
#define XSUM_SPARSE_MAGIC 0x41505358u   /* "XSPA" little-endian */
#define XSUM_SPARSE_MAX_BYTES (24 + 8 * XSUM_NDIGITS)
typedef struct xsum_sparse_header {
    uint32_t magic;      /* XSUM_SPARSE_MAGIC */
    uint16_t version;    /* XSUM_VERSION */
    uint8_t w;           /* 52 */
    uint8_t nnz;         /* records that follow, <= XSUM_NDIGITS */
    uint32_t flags;      /* XSUM_F_NAN | PINF | NINF | MISMATCH */
    uint32_t reserved;   /* 0 */
    uint64_t count;      /* summands */
} xsum_sparse_header;

/* Result record written by xsum_finalize_round / xsum_sum (48 bytes, device memory).
 * PAPER.md:787-795 (§3 step 7): locate the most significant non-zero component,
 * combine it with its neighbours and round on the truncated bits. */
typedef struct xsum_result {
    double value;        /* RN-even of the exact sum; +0.0 for an exact zero; NaN / +-Inf per flags */
    int32_t direction;   /* sign(value - exact) of the finite part: -1, 0, +1 (0 if a special is returned) */
    uint32_t flags;      /* XSUM_F_* */
    int32_t msb_exp;     /* floor(log2 |exact|), INT32_MIN if the exact sum is zero */
    int32_t sign;        /* 1 if the exact finite sum is negative */
    uint64_t count;      /* summands accumulated */
    uint64_t sig53;      /* unbounded-exponent rounding: |exact| ~= sig53 * 2^exp2 (RN-even, 53 bits) */
    int32_t exp2;
    uint32_t value_f32;  /* bits of the RN-even binary32 rounding of the exact sum (one rounding, no
                            double rounding; a negative sum that rounds to 0 gives -0.0f) */
} xsum_result;

/* Outcome of the condition-number-sensitive sum (xsum_sum_condsens), device memory, 152 bytes. */
typedef struct xsum_condsens_info {
    uint32_t r;          /* truncation parameter of the last iteration: 2, 4, 16, or 256 (the exact pass) */
    uint32_t iterations; /* 1..4 (r = 2, 4, 16, 256) */
    int32_t e_cut;       /* largest truncation index of the last iteration; -1 if nothing was truncated */
    uint32_t exact;      /* 1: the last iteration truncated nothing, value = RN-even of the exact sum */
    uint32_t rule;       /* stopping condition used: 1 or 2 */
    uint32_t nnz;        /* entries of the root (truncated iterations; 0 for the exact pass) */
    uint64_t root[16];   /* the root's r-truncated sparse superaccumulator, records (digit << 6) | index in
                            descending index order (the sparse image record format), zero-padded */
} xsum_condsens_info;

typedef struct xsum_ctx xsum_ctx;

/* Sizes of the caller-provided device buffers. */
XSUM_API size_t xsum_state_bytes(void);                 /* = XSUM_STATE_BYTES */
XSUM_API size_t xsum_scratch_bytes(int device);         /* scratch a handle needs on `device` (1 KiB: grid accumulator) */
XSUM_API size_t xsum_result_bytes(void);                /* = sizeof(xsum_result) = 48 */

/* Create a handle bound to `device` whose exact state lives in d_state (XSUM_STATE_BYTES,
 * 8-B aligned) and whose kernels use d_scratch (>= xsum_scratch_bytes(device), 256-B
 * aligned). The state is initialised to zero (header written) on `stream`.
 * Errors: XSUM_EINVAL (null pointers, misalignment, scratch too small, bad device),
 * XSUM_ECUDA, XSUM_ENOMEM. On error *h is NULL. */
XSUM_API xsum_status xsum_create(xsum_ctx **h, int device, void *d_state, void *d_scratch,
                        size_t scratch_bytes, void *stream);

/* State := 0 (count 0, flags 0), stream-ordered. */
XSUM_API xsum_status xsum_reset(xsum_ctx *h, void *stream);

/* Checkpoint / resume (the paper's external-memory scan PAPER.md:1095-1108:
 * the whole superaccumulator is the only state, so a long or out-of-core summation can stop
 * and resume). The checkpoint is the 384-byte state image above.
 * xsum_save_state: copies the handle's state image into host_image (>= XSUM_STATE_BYTES bytes,
 *   caller-owned) after everything enqueued on `stream`; synchronizes `stream`.
 *   Errors: XSUM_EINVAL (null), XSUM_ECUDA.
 * xsum_check_state_image: host-side validation of an image: magic, version, w = 52, 42 digits,
 *   zero reserved word and padding, known flag bits, count <= 2^63-1, every digit regularized
 *   (|digit| <= R-1; the top digit |d| <= 2^29, the bound the value range gives).
 *   Returns XSUM_OK or XSUM_EMISMATCH (XSUM_EINVAL for null).
 * xsum_load_state: state := the image (validated as above; nothing is written on error),
 *   stream-ordered; the host-side count becomes the image's count. host_image may be pageable
 *   and freed when the call returns. Errors: XSUM_EINVAL, XSUM_EMISMATCH, XSUM_ECUDA. */
XSUM_API xsum_status xsum_save_state(xsum_ctx *h, void *host_image, void *stream);
XSUM_API xsum_status xsum_check_state_image(const void *host_image);
XSUM_API xsum_status xsum_load_state(xsum_ctx *h, const void *host_image, void *stream);

/* State += sum of d_x[0..n) EXACTLY (§5: the whole superaccumulator
 * stays in fast memory and components are added in any order; PAPER.md:744-750 step 2
 * decomposition; PAPER.md:559-628 carry-free regularization; PAPER.md:768-776 bottom-up
 * merge). d_x needs only 8-byte alignment; n = 0 is a no-op. May be called repeatedly
 * (chunked / streaming sums). One kernel launch.
 * Errors: XSUM_EINVAL (h or d_x null with n > 0, d_x not 8-B aligned),
 * XSUM_ECAPACITY (total count > 2^63-1), XSUM_ECUDA (launch failure). */
XSUM_API xsum_status xsum_accumulate(xsum_ctx *h, const double *d_x, uint64_t n, void *stream);

/* Binary32 inputs: state += sum of the binary32 values d_x[0..n) EXACTLY
 * (IEEE binary32, t = 23 / l = 8; every binary32 is a multiple of 2^-149,
 * inside the same 2^-1074 fixed-point window). d_x 4-byte aligned. Same errors as
 * xsum_accumulate. Results round to binary64 (value) and binary32 (value_f32). */
XSUM_API xsum_status xsum_accumulate_f32(xsum_ctx *h, const float *d_x, uint64_t n, void *stream);

/* One-shot fused binary32 path (reset + accumulate_f32 + finalize in one launch). */
XSUM_API xsum_status xsum_sum_f32(xsum_ctx *h, const float *d_x, uint64_t n, void *d_res, uint64_t *d_canon,
                                  void *stream);

/* 16-bit inputs, given as bit patterns: state += sum of the IEEE binary16
 * (t = 10, l = 5) or bfloat16 (t = 7, l = 8) values d_x[0..n) EXACTLY (the paper's t-bit fraction /
 * l-bit exponent format; every such value is an integer multiple of 2^-24 resp.
 * 2^-133, inside the 2^-1074 fixed-point window). d_x 2-byte aligned. NaN / +-Inf patterns set
 * the sticky flags (R10). Results round to binary64 (value) and binary32 (value_f32).
 * Errors: as xsum_accumulate. One launch per 2^40 summands. */
XSUM_API xsum_status xsum_accumulate_f16(xsum_ctx *h, const uint16_t *d_x, uint64_t n, void *stream);
XSUM_API xsum_status xsum_accumulate_bf16(xsum_ctx *h, const uint16_t *d_x, uint64_t n, void *stream);

/* One-shot fused 16-bit paths (reset + accumulate + finalize; one launch for n < 2^40). */
XSUM_API xsum_status xsum_sum_f16(xsum_ctx *h, const uint16_t *d_x, uint64_t n, void *d_res, uint64_t *d_canon,
                                  void *stream);
XSUM_API xsum_status xsum_sum_bf16(xsum_ctx *h, const uint16_t *d_x, uint64_t n, void *d_res, uint64_t *d_canon,
                                   void *stream);

/* State += sum of h_x[0..n) for a HOST buffer (pinned memory overlaps best): chunks are
 * copied into the caller's device staging buffer d_stage (two halves, double-buffered,
 * stage_bytes >= 2 MiB) and accumulated while the next chunk is in flight. This is the
 * paper's O(scan(n)) external-memory algorithm with sigma(n) <= M.
 * Returns after enqueueing; h_x and d_stage must stay valid until `stream` completes.
 * Errors: as xsum_accumulate, plus XSUM_EINVAL for a null / too-small staging buffer. */
XSUM_API xsum_status xsum_accumulate_host(xsum_ctx *h, const double *h_x, uint64_t n, void *d_stage,
                                 size_t stage_bytes, void *stream);

/* The same for a host buffer of any element format (dtype XSUM_DT_*; the element size sets the
 * chunking). Errors: as xsum_accumulate_host, plus XSUM_EINVAL for a bad dtype. */
XSUM_API xsum_status xsum_accumulate_host_ex(xsum_ctx *h, const void *h_x, uint64_t n, int dtype, void *d_stage,
                                             size_t stage_bytes, void *stream);

/* State += sum of `count` packed state images at d_states (count * XSUM_STATE_BYTES bytes,
 * 8-B aligned): the MapReduce post-process / all-gather merge (§6.1),
 * a Lemma-1 pairwise tree of carry-free additions. Images with a bad
 * header are skipped and set XSUM_F_MISMATCH in the state (reported by finalize). A merged
 * summand count beyond 2^63-1 saturates and sets XSUM_F_CAPACITY (known only on the device, so
 * no status code reports it). Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_merge(xsum_ctx *h, const void *d_states, uint32_t count, void *stream);

/* Fused post-process ("reads back the p sparse superaccumulators ...
 * add all of them into one ... converted to a correctly-rounded floating point value"):
 * state := sum of the `count` images (Lemma-1 tree, as xsum_merge), then the rounding of
 * xsum_finalize_round into d_res / d_canon, in ONE launch. Used after the all-gather of the
 * per-GPU states. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_merge_round(xsum_ctx *h, const void *d_states, uint32_t count, void *d_res,
                                      uint64_t *d_canon, void *stream);

/* Sparse image of the state: writes the header and one
 * record per non-zero digit to d_out (device, 8-B aligned, >= XSUM_SPARSE_MAX_BYTES) and the
 * image's byte size to *d_nbytes (device u32). Non-destructive. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_to_sparse(xsum_ctx *h, void *d_out, uint32_t *d_nbytes, void *stream);

/* State += sum of `count` sparse images; image s starts at byte d_images + d_offsets[s]
 * (d_offsets: device u64[count], multiples of 8). Carry-free Lemma-1 merge tree as
 * xsum_merge (the paper's sparse merges of PAPER.md:851-873 without the
 * sort: the indices address the dense window directly). Images with a bad header, misaligned
 * offset, unsorted / out-of-range indices or unregularized digits are skipped and set
 * XSUM_F_MISMATCH. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_merge_sparse(xsum_ctx *h, const void *d_images, const uint64_t *d_offsets, uint32_t count,
                                       void *stream);

/* Non-destructive rounding of the state: writes *d_res (device, 8-B aligned) and, if
 * d_canon != NULL, the canonical image (XSUM_CANON_LIMBS little-endian u64 limbs of the
 * two's complement integer A = exact_sum * 2^1074; the "non-overlapping" form of
 * PAPER.md:777-786 / :1058-1064, R4). Signed-carry propagation is a parallel
 * prefix over {-1,0,+1} carries; rounding is RN-even.
 * Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_finalize_round(xsum_ctx *h, void *d_res, uint64_t *d_canon, void *stream);

/* One-shot fused path: state := sum d_x[0..n) exactly, then finalize into d_res / d_canon.
 * Equivalent to reset + accumulate + finalize_round in ONE kernel launch (the last block
 * to finish merges the block partials and rounds). */
XSUM_API xsum_status xsum_sum(xsum_ctx *h, const double *d_x, uint64_t n, void *d_res, uint64_t *d_canon,
                     void *stream);

/* Fused multi-GPU step (SURVEY.md §8(e) fused option; the MapReduce post-process of
 * PAPER.md:1151-1163 done over NVLink peer memory inside the accumulate kernel):
 * every one of `world` ranks calls xsum_sum_allreduce with its own shard; in ONE launch per rank
 * the shard is summed, the last block publishes the rank's state into every rank's exchange
 * buffer (P2P stores), release-increments every rank's arrival counter, waits (acquire) for all
 * world contributions and merges them in rank order with Lemma-1 adds, so every rank's state is
 * the group's exact sum (bit-identical digits) and d_res / d_canon its rounding.
 * d_bufs: DEVICE array of `world` pointers, d_bufs[r] = rank r's exchange buffer as mapped in
 * this process (symmetric memory / CUDA IPC), each >= xsum_peer_buffer_bytes(world) bytes,
 * 8-B aligned, zero-initialised before the first call. epoch: 1 for the first call on these
 * buffers, then +1 per call (the same on every rank). All ranks must make the call (it is a
 * collective); a peer that does not arrive within ~2 s sets XSUM_F_PEER_TIMEOUT instead of
 * hanging. Errors: XSUM_EINVAL (rank >= world, world == 0, epoch == 0, null / misaligned
 * pointers), XSUM_ECAPACITY, XSUM_ECUDA. */
XSUM_API size_t xsum_peer_buffer_bytes(uint32_t world);
XSUM_API xsum_status xsum_sum_allreduce(xsum_ctx *h, const double *d_x, uint64_t n, void *const *d_bufs,
                                        uint32_t rank, uint32_t world, uint64_t epoch, void *d_res,
                                        uint64_t *d_canon, void *stream);

/* Self-test of the exchange protocol on ONE GPU: `world` (<= 64) virtual ranks, one thread block
 * each, run the same device exchange as xsum_sum_allreduce in one cooperative launch (so all are
 * co-resident): rank r publishes state image d_states[r] (regularized), waits and merges;
 * writes the merged image d_out[r] and its rounding d_res[r] (xsum_result). d_bufs as above, on
 * this device. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_peer_selftest(const void *d_states, void *const *d_bufs, uint32_t world, uint64_t epoch,
                                        void *d_res, void *d_out, void *stream);

/* Cap the number of thread blocks an accumulate launch of this handle may use
 * (0 = one per SM, the default; values above 1024 are clamped). Lets a caller leave
 * SMs to concurrent work; tests use it to force many flush windows per lane.
 * Errors: XSUM_EINVAL (null handle). */
XSUM_API xsum_status xsum_set_grid_limit(xsum_ctx *h, uint32_t max_blocks);

/* Release the host handle (never frees caller memory). */
XSUM_API xsum_status xsum_destroy(xsum_ctx *h);

/* Summands in the handle's state: the host-side counter of what was accumulated through the
 * handle since the last reset / sum / load, plus, after a merge, the merged state's count (the
 * merge enqueues a copy of it; the first xsum_count after a merge waits for that copy, i.e. for
 * the stream to pass the merge). Saturates at 2^63-1 (then the state carries XSUM_F_CAPACITY).
 * UINT64_MAX if that wait fails; 0 for a null handle. */
XSUM_API uint64_t xsum_count(const xsum_ctx *h);

/* Segmented exact sums (BASELINE.json config 5): for s < nseg, d_out[s] = RN-even of the
 * exact sum of d_x[s*seg_len .. (s+1)*seg_len). Optional outputs: d_canon[s*34 .. s*34+34)
 * canonical images, d_flags[s] XSUM_F_* flags. d_x 8-B aligned, any seg_len >= 0.
 * Each segment is reduced by one warp (the paper's per-block "combine");
 * equal segments of length <= 256 by one lane each (its own superaccumulator and rounding), and
 * equal 16-B-aligned segments whose length is a multiple of 512 by half a warp each.
 * Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_sum_segments(const double *d_x, uint64_t nseg, uint64_t seg_len, double *d_out,
                              uint64_t *d_canon, uint32_t *d_flags, void *stream);

/* Segmented exact sums of any input format (SURVEY.md §8(f) f1 x f2): segment s is
 * d_x[s*seg_len .. (s+1)*seg_len) or, if d_offsets != NULL, d_x[d_offsets[s] .. d_offsets[s+1])
 * (elements of `dtype`, d_x aligned to the element size). Per segment, optional outputs: d_out[s]
 * the RN-even binary64 and d_out32[s] the RN-even binary32 of the exact sum (each rounded once
 * from the exact value), d_canon[s*34 ..] the canonical image, d_flags[s]. One warp per segment.
 * Errors: XSUM_EINVAL (bad dtype, null / misaligned pointers, no output requested), XSUM_ECUDA. */
XSUM_API xsum_status xsum_sum_segments_ex(const void *d_x, int dtype, uint64_t nseg, uint64_t seg_len,
                                          const uint64_t *d_offsets, double *d_out, float *d_out32,
                                          uint64_t *d_canon, uint32_t *d_flags, void *stream);

/* Variable-length segments (CSR offsets): segment s is
 * d_x[d_offsets[s] .. d_offsets[s+1]), offsets non-decreasing device u64 array of nseg+1.
 * Outputs as xsum_sum_segments. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_sum_segments_csr(const double *d_x, const uint64_t *d_offsets, uint64_t nseg,
                                  double *d_out, uint64_t *d_canon, uint32_t *d_flags, void *stream);

/* Condition-number-sensitive exact-or-faithful sum (§4):
 * the paper's iteration r = 2, 4, 16 (r <- r^2) over the complete binary
 * summation tree of d_x[0..n) in index order (reading C2), every internal node the
 * r-truncated Lemma-1 sum (Lemma 2 :859-872) of its children;
 * after each iteration the root is rounded to nearest even (y) and the iteration stops when the
 * stopping condition `rule` holds - 1: y = y (+) n eps_min = y (+) -n eps_min,
 * 2: the least significant bit of y is >= ceil(log2 n) + 2 binary orders above eps_min
 * (reading C4) - with eps_min = R^E_cut 2^-1074 from the largest truncation
 * index over all nodes (reading C3), or when nothing was truncated. If r = 16 does not stop, the
 * exact dense sum (r = 256 truncates nothing) runs. Then *d_res holds y (a FAITHFUL rounding of
 * the exact sum, the RN-even rounding when info.exact; direction / INEXACT refer to the
 * truncated root T), *d_info the iteration record, d_canon (optional, 34 limbs) the canonical
 * image of T. NaN / +-Inf inputs set flags and the value per R10. Stream-ordered, no host
 * synchronization: every iteration is enqueued and an iteration after a stop exits at entry.
 * d_work: device scratch of xsum_condsens_work_bytes(n) bytes, 256-B aligned, no initialization,
 * not shared by concurrent calls. d_x 8-B aligned. Errors: XSUM_EINVAL (null / misaligned
 * pointers, rule not 1 or 2, d_work too small), XSUM_ECUDA. */
XSUM_API size_t xsum_condsens_work_bytes(uint64_t n);
XSUM_API xsum_status xsum_sum_condsens(const double *d_x, uint64_t n, int rule, void *d_work, size_t work_bytes,
                                       void *d_res, void *d_info, uint64_t *d_canon, void *stream);

/* Static string for a status code. */
XSUM_API const char *xsum_status_str(xsum_status s);

/* Number of kernel launches the library enqueued since load (for bench.py's gpu_launches). */
XSUM_API uint64_t xsum_launch_count(void);

/* xsum_sum_segments_ex with a work-balancing ticket: d_ticket (optional, 8-B aligned, caller-owned)
 * is one 64-bit device word that must be ZERO when the call's work starts on `stream` (e.g. zeroed
 * by a stream-ordered memset just before) and is left non-zero. With CSR offsets the warps then
 * draw the next unclaimed segment from it atomically instead of taking the static order s,
 * s + nw, ... - ragged lengths otherwise leave the busiest warp with well above the mean work
 * (c5csr: 1.36x). Used for binary64 CSR segments; ignored otherwise. A ticket word must not be
 * shared by calls whose work may overlap. Errors: as xsum_sum_segments_ex. */
XSUM_API xsum_status xsum_sum_segments_ws(const void *d_x, int dtype, uint64_t nseg, uint64_t seg_len,
                                          const uint64_t *d_offsets, double *d_out, float *d_out32,
                                          uint64_t *d_canon, uint32_t *d_flags, void *d_ticket, void *stream);

/* CSR segments that are mostly short (SURVEY.md §8(f) f1 batched sums; e.g. sparse-matrix rows):
 * same arguments and outputs as xsum_sum_segments_ws with d_offsets required. Warps take groups of
 * 32 consecutive segments; a segment of <= 256 elements is summed by one lane in its own
 * superaccumulator and rounded by it (one thread), longer ones of the group by
 * the whole warp. d_ticket (optional, zero at the call's start, as in xsum_sum_segments_ws)
 * balances the groups dynamically. Faster than the warp-per-segment path when most segments are
 * short; the binding picks it when the mean length is <= 256. Errors: XSUM_EINVAL, XSUM_ECUDA. */
XSUM_API xsum_status xsum_sum_segments_csr_lanes(const void *d_x, int dtype, uint64_t nseg, const uint64_t *d_offsets,
                                                 double *d_out, float *d_out32, uint64_t *d_canon, uint32_t *d_flags,
                                                 void *d_ticket, void *stream);

/* Exact reduction along a strided dimension (a reproducible sum over one
 * tensor dimension without a transposing copy): d_x is a contiguous [outer][len][inner] array of
 * `dtype` elements (XSUM_DT_*; element-size aligned); for every o < outer, i < inner
 *   d_out64[o*inner + i] and/or d_out32[o*inner + i] = RN-even (binary64 / binary32) of the exact
 *   sum over r < len of d_x[(o*len + r)*inner + i]   (len = 0 gives +0.0),
 * d_flags[o*inner + i] (optional) the XSUM_F_* flags of that sum (NaN/Inf seen, and OVERFLOW /
 * INEXACT for the binary64 rounding, OVERFLOW32 / INEXACT32 for the binary32 one, per the outputs
 * requested). Specials follow R10 (NaN, +Inf, -Inf). Each lane sums one fibre in its own shared
 * superaccumulator and rounds it itself. When the fibres
 * cannot fill the GPU the rows are split into parts whose exact partial superaccumulators are
 * merged by a second launch, or (binary64, when the fibre groups fill the resident warps unevenly)
 * every warp takes an equal share of all rows and the pieces of a fibre meet in a per-fibre
 * accumulator (stream-K; the call clears it first); either needs d_work of
 * xsum_sum_strided_work_bytes(...) bytes (8-B aligned, caller-owned, no initialization); with a
 * smaller or NULL d_work neither is used (same results, fewer SMs busy). inner = 1 is served by the segment kernels
 * (xsum_sum_segments_ex; its flags carry both roundings' bits). At least one of d_out64 /
 * d_out32. Stream-ordered, no host synchronization. Errors: XSUM_EINVAL (bad dtype, no output,
 * misalignment, sizes overflowing 2^63), XSUM_ECUDA. */
XSUM_API size_t xsum_sum_strided_work_bytes(uint64_t outer, uint64_t len, uint64_t inner, int device);
XSUM_API xsum_status xsum_sum_strided(const void *d_x, int dtype, uint64_t outer, uint64_t len, uint64_t inner,
                                      double *d_out64, float *d_out32, uint32_t *d_flags, void *d_work,
                                      size_t work_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* XSUM_H */
