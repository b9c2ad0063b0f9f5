/*
 * vsaogm.h -- C ABI of the B200-native VSA-OGM hot path (arXiv 2408.09066).
 *
 * The library computes, on an sm_100a GPU, the data-parallel hot path of
 * VSA-OGM (Snyder et al., "Brain Inspired Probabilistic Occupancy Grid
 * Mapping with Vector Symbolic Architectures"):
 *
 *   encode/bundle  m_{c,k} += sum_{i: psi_i = c} exp(i (thx_k x_i + thy_k y_i) / l)
 *                  PAPER.md:252-258 (Eq. 9), :216-219 (Eq. 5), :260-285 (Alg. 1, delta = 1)
 *   normalise      m_c / ||m_c||                      PAPER.md:292-295 (Eq. 10)
 *   decode         q_c(x,y) = Re <m_c/||m_c||, phi(x,y)> / sqrt(D)
 *                                                     PAPER.md:297-301 (Eq. 11)
 *   Born rule      p_c = q_c^2
 *   local entropy  S_c = window mean of H_b(p_c); S = S_1 - S_0
 *                                                     PAPER.md:318, :330-356 (Alg. 2)
 *   classify       occupied if S >= rho_occ, empty if S < rho_emp, else unknown
 *                                                     PAPER.md:320-328 (Eq. 12) + DESIGN.md L14
 *
 * Conventions: D independent complex phasors per
 * vector, phases uniform on (-pi, pi] drawn by splitmix64 (x axis then y
 * axis, u = (z >> 11) 2^-53, theta = pi (1 - 2u)); class 0 = empty,
 * class 1 = occupied; grid cell (r, c) has centre (x0 + (c + .5) res,
 * y0 + (r + .5) res), row r grows along +y.
 *
 * Memory and streams.  Every pointer named *_dev is a device pointer owned by
 * the caller (e.g. a torch CUDA tensor) that must stay valid until the work
 * queued on the context's stream has reached it; *_host pointers are host
 * memory (pinned memory gives asynchronous copies).  All calls enqueue work on
 * the context's stream and return without synchronising unless they say so.
 * A context is bound to the CUDA device current at vsaogm_create and is not
 * thread-safe: use one context per (device, thread).
 *
 * Errors.  Every int-returning call returns VSAOGM_OK (0) or a negative code
 * below; vsaogm_strerror() names it.  Argument errors are detected on the host
 * before any work is queued (the call then has no effect).  Invalid points
 * (label not in {0,1}, non-finite coordinate) are detected on the device,
 * skipped, and reported by the next vsaogm_sync() (deferred error).
 */
#ifndef VSAOGM_H
#define VSAOGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSAOGM_OK 0
#define VSAOGM_EINVAL_DIM (-1)   /* D < 1 (SPEC.md:47 analogue for complex phasors)      */
#define VSAOGM_EINVAL_ARG (-2)   /* bad length scale, bounds, grid, band, window or rho   */
#define VSAOGM_EEMPTY (-3)       /* n < 1 points                      */
#define VSAOGM_ELABEL (-4)       /* deferred: a label not in {0,1}          */
#define VSAOGM_ENONFINITE (-5)   /* deferred: a non-finite coordinate       */
#define VSAOGM_ENOMEM (-6)       /* device or host allocation failed                      */
#define VSAOGM_ECUDA (-7)        /* a CUDA runtime / driver call failed                   */
#define VSAOGM_ESTATE (-8)       /* call not valid in the current state (see each call)   */

/* Opaque per-(device, rank) context: owns theta, the memories, tables, scratch. */
typedef struct vsaogm_ctx vsaogm_ctx;

/* World bounds in metres (x_max > x_min, y_max > y_min, all finite).  Their
 * centre is the phase origin of the device tables; results do not depend on
 * it (a common phase rotation cancels in Eq. 11), but every rank of a
 * multi-GPU job must pass the same bounds (Alg. 3 preconditions). */
typedef struct {
    double x_min, y_min, x_max, y_max;
} vsaogm_bounds;

/* Query grid.  Full grid rows x cols, cell size res > 0, lower-left corner
 * (x0, y0).  This rank owns rows [row_begin, row_end) (0 <= row_begin <
 * row_end <= rows); the decode also evaluates `halo` extra rows on each side
 * (clipped to [0, rows)) so that vsaogm_entropy can use window half-widths up
 * to `halo` without communication (row-band sharding). */
typedef struct {
    double x0, y0, res;
    int32_t rows, cols;
    int32_t row_begin, row_end;
    int32_t halo;
} vsaogm_grid;

/* Tensor-core operand precision of the decode contraction (fp32 accumulate). */
typedef enum { VSAOGM_F16 = 0, VSAOGM_BF16 = 1 } vsaogm_precision;

/* Alg. 2 window + Eq. 12 thresholds.  Class 1 (occupied) uses half-width
 * half_occ, class 0 (empty) half_emp; window (2h+1)^2 box if disk == 0, the
 * paper's disk u^2 + v^2 <= h^2 if disk == 1; 1 <= h <= 16.  Windows are
 * clipped to the full grid and averaged over the clipped count. */
typedef struct {
    int32_t half_occ, half_emp;
    int32_t disk;
    float rho_occ, rho_emp;   /* rho_emp <= rho_occ; equal values give the binary Eq. 12 */
} vsaogm_entropy_params;

/* Create a context on the current CUDA device: draws theta (D phases per axis,
 * seed as above), allocates zeroed memories.  l = length scale in metres
 * (Eq. 8), l > 0.  *out receives the context.
 * Errors: EINVAL_DIM (D < 1), EINVAL_ARG (l, bounds, out == NULL), ENOMEM, ECUDA. */
int vsaogm_create(int32_t D, uint64_t seed, double length_scale, vsaogm_bounds bounds,
                  vsaogm_ctx **out);

/* Space discretisation (sec. III-B-4; Alg. 1 :260-285): as
 * vsaogm_create with delta x delta equal quadrants of `bounds` (1 <= delta <=
 * VSAOGM_MAX_DELTA) and 2 delta^2 memories, slot 2 beta + psi.  A point goes to
 * the quadrant beta = j delta + i whose centre (x_min + (i + 1/2) W / delta,
 * y_min + (j + 1/2) H / delta) is nearest (fp64 squared distance, ties to the
 * lowest index; out-of-bounds points to the nearest centre);
 * a grid cell queries the two memories of the quadrant nearest its centre.
 * Memories, pending memories and counts are then [2 delta^2] slots instead of
 * [2] classes in every call below.  vsaogm_create(...) == delta 1. */
#define VSAOGM_MAX_DELTA 8
int vsaogm_create_quadrants(int32_t D, uint64_t seed, double length_scale, vsaogm_bounds bounds,
                            int32_t delta, vsaogm_ctx **out);

/* Release every resource of the context (synchronises its stream). NULL is a no-op. */
void vsaogm_destroy(vsaogm_ctx *ctx);

/* Queue all later work on `stream` (a cudaStream_t; NULL = the legacy default stream). */
int vsaogm_set_stream(vsaogm_ctx *ctx, void *stream);

/* Bundle n labelled points into the pending memories (Eq. 9 + Eq. 5, Alg. 1
 * with delta = 1: the slot is the label).  xy_dev: float32 [n][2] metres
 * (x, y interleaved), labels_dev: uint8 [n] in {0 empty, 1 occupied}.  Points
 * with another label or a non-finite coordinate are skipped and raise the
 * deferred ELABEL / ENONFINITE.  Errors: EINVAL_ARG (NULL), EEMPTY (n < 1). */
int vsaogm_encode_bundle(vsaogm_ctx *ctx, const float *xy_dev, const uint8_t *labels_dev,
                         int64_t n);

/* As vsaogm_encode_bundle, from host arrays: the host->device copies are
 * queued on the context's stream into context-owned staging buffers. */
int vsaogm_encode_bundle_host(vsaogm_ctx *ctx, const float *xy_host, const uint8_t *labels_host,
                              int64_t n);

/* Expose the pending (not yet committed) memories for a multi-rank all-reduce
 * (Alg. 3 fusion): *dev_ptr = ONE contiguous fp64 buffer of
 * *n_doubles = 2 S Dp + S values: the pending memories [S][Dp][2] (slot, k,
 * re/im; S = 2 delta^2 slots 2 beta + psi, S = 2 classes for delta = 1) in the
 * context's centred-phase convention, Dp = D rounded up to a multiple of 32
 * (padding entries stay zero), followed by the S pending point counts as
 * integer-valued doubles (exact below 2^53).  A multi-rank job sums the whole
 * buffer with a single all-reduce (sum) and then calls vsaogm_commit.  After
 * this call the context is in multi-rank mode: vsaogm_decode no longer commits
 * implicitly and returns ESTATE while pending work is uncommitted.  The
 * pointer stays valid for the life of the context; the buffer is ordered on
 * the context stream (encodes queued on an encode stream are joined first). */
int vsaogm_pending(vsaogm_ctx *ctx, double **dev_ptr, int64_t *n_doubles);

/* m += pending; pending = 0 (and the counts). */
int vsaogm_commit(vsaogm_ctx *ctx);

/* Zero the memories, pending memories and counts. */
int vsaogm_reset(vsaogm_ctx *ctx);

/* Decode every cell of this rank's band (plus halo rows) into signed
 * similarities (Eq. 10 normalisation, Eq. 11 query), and
 * the per-cell binary entropy H_b(q^2) kept in the context for
 * vsaogm_entropy.  Two methods compute the same sums (tuning key
 * "dec_method"): a dense tcgen05 GEMM over separable phasor tables (precision
 * selects its 16-bit operand type; fp32 accumulation), and a type-1 NUFFT
 * (fp32 Gaussian gridding + FFTs, nudecode.cu; delta = 1, grid spacing below
 * l / 2, `precision` unused).  The default picks the NUFFT where it applies
 * and its modelled time is lower.  q_dev: NULL, or float32 [2][row_end-row_begin][cols]
 * (class 0 empty, 1 occupied) receiving q for the band's own rows.  In
 * single-rank mode pending memories are committed first.
 * Errors: EINVAL_ARG (grid), ESTATE (multi-rank mode with uncommitted
 * pending), ENOMEM, ECUDA. */
int vsaogm_decode(vsaogm_ctx *ctx, const vsaogm_grid *grid, vsaogm_precision precision,
                  float *q_dev);

/* Local-entropy estimator used by the following decodes and entropy calls
 * (L10):
 *   0 (default) the window mean of the per-cell binary entropy H_b(p), in bits;
 *   1 the Shannon entropy, in bits, of the 8-bit grey-level histogram of p in the
 *     window (p quantised as floor(255 p + 1/2) in fp32) -- the image-processing
 *     reading of "passing a disk filter ... applying Shannon entropy".
 * Errors: EINVAL_ARG. */
int vsaogm_set_estimator(vsaogm_ctx *ctx, int32_t estimator);

/* Tuning variants (measurement and test hook; the defaults are the measured best and no
 * environment variable changes them).  Sets the integer knob `key` of this context for
 * later calls: "enc_method" (-1 auto, the default: the type-3 NUFFT for delta = 1 and D >= 2048 when its
 * modelled time is below the direct kernel's; 0 direct pair kernels; 1 NUFFT), "enc_x2" (direct encode kernel family; 4 = the pair kernel, the default),
 * "enc_pairs_npoly", "enc_pairs_minb", "enc_pairs_split", "enc_x2_npoly", "enc_x2_minb",
 * "enc_x2_waves", "enc_npoly", "enc_minb", "enc_kt", "enc_path", "enc_waves",
 * "enc_runs_waves" (encode variants), "gemm_variant" (-1 auto, 0
 * CTA pair, 1 single CTA, 2 two CTA pairs per cluster with B multicast), "gemm_bn" (0 auto, else the tile width), "gemm_splits" (0 auto,
 * else the split-K factor), "gemm_l2_hints" (0 none, the default; 1 A evict-first + B evict-last; 2 B evict-last), "pipe_early" (0/1), "entropy_kernel"
 * (0 auto: the column-walk box kernel for labels-only equal-radius box windows h <= 4, else the
 * generic staged kernel; 1 the generic kernel; 2 the TMA-streamed box kernel), "entropy_rw" (0 auto,
 * else output rows per thread chunk / work item of the box kernels), "table_rows" (1..256, default 32:
 * phasor-table rows per thread of the table kernels), "dec_method" (-1 auto, the default; 0 the
 * tcgen05 GEMM; 1 the NUFFT where it applies, else the GEMM), "pdl" (1, the default: the step's
 * kernels are chained by programmatic dependent launches; 0 ordinary launches), "nd_bps" (0, the
 * default: the NUFFT decode's FFT kernels fill the SMs; else a cap on their resident blocks per SM).
 * Errors: EINVAL_ARG (unknown key or value out of range; nothing changes). */
int vsaogm_set_tuning(vsaogm_ctx *ctx, const char *key, int64_t value);

/* Read a tuning knob of this context into *value (the same keys).  Errors: EINVAL_ARG. */
int vsaogm_get_tuning(vsaogm_ctx *ctx, const char *key, int64_t *value);

/* Local entropy (Alg. 2), global entropy S = S_occ - S_emp, 3-way labels
 * (Eq. 12 + L14) over the band of the last vsaogm_decode.  s_dev: NULL or
 * float32 [3][band][cols] = (S_occ, S_emp, S); labels_dev: NULL or uint8
 * [band][cols] with 0 empty, 1 occupied, 2 unknown.
 * Errors: ESTATE (no decode yet), EINVAL_ARG (params, or a half-width larger
 * than the decode halo where the band has neighbours). */
int vsaogm_entropy(vsaogm_ctx *ctx, const vsaogm_entropy_params *params, float *s_dev,
                   uint8_t *labels_dev);

/* As vsaogm_entropy, returning to host memory: s_host NULL or float32
 * [3][band][cols], labels_host uint8 [band][cols].  Synchronises the stream. */
int vsaogm_entropy_host(vsaogm_ctx *ctx, const vsaogm_entropy_params *params, float *s_host,
                        uint8_t *labels_host);

/* Encode stream (streaming pipeline): with a non-NULL
 * `stream` (a cudaStream_t), vsaogm_encode_bundle runs its kernels there
 * instead of on the context stream.  Ordering stays that of the calls: an
 * encode waits for the last commit / reset / import / decode's table build
 * queued on the context stream (so it overlaps the rest of that decode: the
 * tensor-core GEMM and the entropy), and the next operation on the context
 * stream that touches the pending memories (decode, commit, reset, pending,
 * export, sync ...) waits for the encodes queued before it.  The caller orders
 * the encode inputs against `stream`.  NULL restores single-stream operation.
 * Errors: EINVAL_ARG, ECUDA. */
int vsaogm_set_encode_stream(vsaogm_ctx *ctx, void *stream);

#define VSAOGM_IO_SLOTS 4

/* Pipelined host I/O for streaming mapping (one batch per step, Alg. 1 then
 * Alg. 2): the host<->device copies of step k run on two
 * internal copy streams and overlap the kernels of steps k-1 and k+1.
 *
 * vsaogm_encode_bundle_host_async: as vsaogm_encode_bundle_host, but the
 * host->device copy of (xy_host float32 [n][2], labels_host uint8 [n]) goes to
 * one of VSAOGM_IO_SLOTS device staging slots on the upload stream, and the encode on the
 * context stream (or the encode stream, when one is set) waits for it.  The host
 * arrays must be page-locked for the
 * copy to be asynchronous, and must stay unmodified until the ticket of the
 * vsaogm_entropy_host_async that follows this call has been waited for.
 *
 * vsaogm_entropy_host_async: as vsaogm_entropy_host, into one of VSAOGM_IO_SLOTS
 * device output slots, then a device->host copy on the download stream (it
 * overlaps the next step's kernels); returns at once with *ticket.  s_host /
 * labels_host (page-locked for overlap) are written when vsaogm_wait(ctx, *ticket)
 * returns.  There are VSAOGM_IO_SLOTS (4) staging and output slots; a slot is reused that
 * many calls later (the device orders the reuse after its previous download), so
 * up to VSAOGM_IO_SLOTS - 1 steps may be in flight: the caller waits for ticket
 * k - 3 after queuing step k (at C4 the 75 us label download of a step is half a step long: with
 * fewer steps in flight the host queues the next encode too late to overlap the running decode).
 *
 * vsaogm_wait: block until step `ticket` has been downloaded; returns a deferred
 * device error like vsaogm_sync (the error bits are sticky until vsaogm_sync and are
 * snapshotted after the step's entropy; with an encode stream set, the next step's
 * encode may already have run, so an error can be reported one step early).
 * Errors: EINVAL_ARG (unknown ticket), ECUDA.  Switching the encode stream
 * (vsaogm_set_encode_stream) synchronises the copy streams of this pipeline. */
int vsaogm_encode_bundle_host_async(vsaogm_ctx *ctx, const float *xy_host, const uint8_t *labels_host, int64_t n);
int vsaogm_entropy_host_async(vsaogm_ctx *ctx, const vsaogm_entropy_params *params, float *s_host,
                              uint8_t *labels_host, int64_t *ticket);
int vsaogm_wait(vsaogm_ctx *ctx, int64_t ticket);

/* Wait for the context's stream; return a deferred device error (ELABEL or
 * ENONFINITE, first one seen since the last sync) or ECUDA, else OK. */
int vsaogm_sync(vsaogm_ctx *ctx);

/* Test hook (synchronises): committed + pending memories as fp64 [S][D][2]
 * (S = 2 delta^2 slots) in the raw-coordinate convention of Eq. 9 (the
 * centring rotation undone on the host in fp64), and counts[S].  Either
 * pointer may be NULL. */
int vsaogm_get_memory(vsaogm_ctx *ctx, double *host, int64_t *counts);

/* Test hook: theta as fp64 [2][D] (x axis, then y axis). */
int vsaogm_get_phases(vsaogm_ctx *ctx, double *host);

/* Kernel-level timing.  While enabled, the library brackets each of its
 * kernel launches with CUDA events on the context's stream.  read: waits for
 * the stream, writes the summed milliseconds and launch counts per kernel id
 * (ms[VSAOGM_NKERNELS], launches[VSAOGM_NKERNELS]; either may be NULL) since
 * the last read, then clears them. */
#define VSAOGM_K_ENCODE 0
#define VSAOGM_K_REDUCE 1
#define VSAOGM_K_COMMIT 2
#define VSAOGM_K_NORMS 3
#define VSAOGM_K_TABLE_B 4
#define VSAOGM_K_TABLE_A 5
#define VSAOGM_K_DECODE_GEMM 6
#define VSAOGM_K_ENTROPY 7
#define VSAOGM_K_ND_SPREAD 8   /* NUFFT decode: point strengths + Gaussian gather (nudecode.cu) */
#define VSAOGM_K_ND_COLFFT 9   /* NUFFT decode: transforms along y of the band columns */
#define VSAOGM_K_ND_ROWFFT 10  /* NUFFT decode: transforms along x of the decoded rows + epilogue */
#define VSAOGM_NKERNELS 11
int vsaogm_profile_enable(vsaogm_ctx *ctx, int enable);
int vsaogm_profile_read(vsaogm_ctx *ctx, double *ms, int64_t *launches);

/* Total number of kernels this context has launched (all ids). */
int64_t vsaogm_launch_count(const vsaogm_ctx *ctx);

/* Test hook: the decode GEMM kernel alone.  C[M][N] (float32, row-major) =
 * A[M][K] . B[N][K]^T with A, B 16-bit (precision) K-major device arrays,
 * K a multiple of 64, 1 <= M, N.  kernel: -1 library default, 0 the CTA-pair
 * (cta_group::2) kernel, 1 the single-CTA kernel, 2 the CTA-pair kernel in clusters
 * of two pairs with B multicast; bn (0 auto, else 128..256 in
 * steps of 32) and splits (0 auto, else the split-K factor) pin the CTA-pair
 * kernel's tile width and split-K.  Runs on `stream` and synchronises it. */
int vsaogm_test_gemm(const void *A_dev, const void *B_dev, int32_t M, int32_t N, int32_t K,
                     vsaogm_precision precision, int32_t kernel, int32_t bn, int32_t splits, float *C_dev,
                     void *stream);

/* Multi-agent fusion (Alg. 3).
 * vsaogm_export writes the context's state -- committed + pending memories in
 * the raw-coordinate convention of Eq. 9, per-slot counts, and the fusion
 * preconditions (D, theta seed, length scale, delta, bounds) -- into `buf` as a
 * self-describing little-endian container: the 8-byte magic "VSAOGM1\0", a
 * `key=value` text header terminated by "\n\n", then int64 counts[S] and fp64
 * memories [S][D][2].  buf == NULL: only *size is set (the bytes needed).
 * Synchronises the stream.  Errors: EINVAL_ARG (size NULL, or *size too small). */
int vsaogm_export(vsaogm_ctx *ctx, void *buf, int64_t *size);

/* Fuse an exported state into this context: its memories and counts are ADDED
 * to this context's committed memories (mode 1; Alg. 3 bundles same-index
 * memories, Eq. 5) or REPLACE them (mode 0, e.g. a checkpoint restore; pending
 * work is discarded).  The three fusion conditions (same axis
 * vectors, same classes, same delta) plus the same D, length scale and bounds
 * are checked first.  Errors: EINVAL_ARG (malformed container, mode),
 * EPRECOND (a condition differs; nothing is changed). */
#define VSAOGM_EPRECOND (-9)     /* fusion precondition violated (Alg. 3)  */
int vsaogm_import(vsaogm_ctx *ctx, const void *buf, int64_t size, int32_t mode);

/* Name of an error code. */
const char *vsaogm_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* VSAOGM_H */
