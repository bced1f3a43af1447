/*
 * sqf2k_b200.h -- C ABI of the B200 hot path of the sqf2k verifier
 * (Hercher, arXiv 2411.01964: every odd n > 1 is m + 2^k with m squarefree).
 *
 * The reference (`/root/reference/pkg/src/sqf2k`, pure Python + numpy) has no
 * FFI.  Each entry point below replaces one reference Python function on the
 * hot path; the reference-side ctypes binding is shown in INTEGRATION.md.
 * The Python package `paper_2411_01964_b200` keeps the reference signatures
 * and calls these symbols.
 *
 * Conventions
 *   - Every function returns SQF2K_OK (0) or a negative SQF2K_E* code; no C++
 *     exception crosses the ABI.  sqf2k_last_error() gives the message of the
 *     last failure on the calling thread.
 *   - Output buffers are caller-allocated host memory (numpy via ctypes).
 *   - The library owns device memory, its CUDA stream and cached buffers;
 *     calls are serialised by an internal mutex.  One process drives one GPU
 *     (the device chosen by sqf2k_init); multi-GPU runs are one process per
 *     GPU, reduced by the caller (torch.distributed / NCCL).
 *   - Integers are odd n in [start, end), end - start even (the reference's
 *     normalised range, runner.py:57-61).  The GPU domain is end <= 2^62
 *     (so p <= 2^31 and p^2 < 2^62); larger ends are SQF2K_EINVAL.
 *   - Bit layout of segment bitmaps is the reference's: slot i = (n-start)/2,
 *     bit i lives in byte i>>3 at position i&7 (LSB first), 1 = squarefree,
 *     buffers padded with zero bits to a multiple of 8 bytes (sieve.py:13-16,
 *     sieve.py:60-69).
 */
#ifndef SQF2K_B200_H
#define SQF2K_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SQF2K_ABI_VERSION 1

/* histogram index k = 0..64, slot 0 unused (aggregate.py:10-12) */
#define SQF2K_HIST_LEN 65
#define SQF2K_NONE UINT64_MAX

enum {
    SQF2K_OK = 0,
    SQF2K_EINVAL = -1,    /* bad argument: the Python layer raises ValueError   */
    SQF2K_ECUDA = -2,     /* CUDA runtime / kernel failure: RuntimeError          */
    SQF2K_ENOMEM = -3,    /* device allocation failed: MemoryError                */
    SQF2K_ECAPACITY = -4, /* caller's failure buffer too small; *n_failures holds
                             the required size, retry with a larger buffer        */
    SQF2K_ENODEV = -5     /* no CUDA device / library not initialised             */
};

/*
 * Mergeable scan summary -- the device-side form of SegmentSummary
 * (aggregate.py:25-62).  The GPU produces hist[] and min_n[]; the library
 * derives k_sum, k_max_observed and the record candidates from them exactly
 * as the reference's per-block loop does (search.py:187-200):
 *   cand[m] = least n in the range whose smallest exponent exceeds m
 *           = min( min_{m < k <= k_max} min_n[k], least failure ),
 *   defined for 1 <= m <= k_max whenever such an n exists.
 */
typedef struct sqf2k_summary {
    uint64_t start;                   /* hull of the scanned odd n: [start, end) */
    uint64_t end;
    uint64_t hist[SQF2K_HIST_LEN];    /* hist[k] = #{n : k(n) = k}                */
    uint64_t min_n[SQF2K_HIST_LEN];   /* least n with k(n) = k, SQF2K_NONE if none */
    uint64_t cand[SQF2K_HIST_LEN];    /* record candidates, SQF2K_NONE if absent  */
    uint64_t k_sum;                   /* sum of k(n)                              */
    uint64_t n_failures;              /* n unresolved at k_max (may exceed cap)   */
    uint32_t k_max_observed;
    uint32_t k_max;                   /* exponent limit the scan used             */
} sqf2k_summary_t;

/* Options of sqf2k_verify.  Zero-initialised = defaults. */
typedef struct sqf2k_verify_opts {
    uint32_t pipeline;     /* 0: fused tile kernel (sieve + min-k scan in shared
                                 memory, no bitmap in HBM) -- default
                              1: two-pass: sieve -> packed bitmap in HBM ->
                                 128-bit-load scan kernel                       */
    uint32_t tile_depth;   /* exponents resolved inside a tile (halo 2^(d-1)
                              slots); 0 = default 16.  Anything unresolved at
                              the tile depth but k_max > depth escalates to the
                              exact trial-division kernel.  Tests force tiny
                              depths to exercise escalation.                   */
    uint64_t batch_slots;  /* odd slots per device batch; 0 = default 2^37, max 2^40 */
    uint32_t flags;        /* SQF2K_EXACT_BUCKETS: exact (count + scan) large-
                              prime lists from the start instead of the fixed-
                              capacity lists with exact fallback (tests)      */
    uint32_t reserved;
} sqf2k_verify_opts_t;

#define SQF2K_EXACT_BUCKETS 1u

/* Per-kernel device-time statistics (CUDA events on the library's stream). */
typedef struct sqf2k_kstat {
    char name[32];
    uint64_t launches;
    double total_ms;
} sqf2k_kstat_t;

/* ---- lifetime ---------------------------------------------------------- */

/* Bind the calling process to CUDA device `device` and create the stream.
 * Idempotent for the same device.  SQF2K_ENODEV when no GPU is visible.   */
int sqf2k_init(int device);
int sqf2k_device_count(int *count);
const char *sqf2k_last_error(void);
void sqf2k_shutdown(void);
int sqf2k_abi_version(void);

/* ---- L0: prime table  (replaces primes.py:26-40 generate_primes) ------- */

/* Number of primes <= limit (limit >= 1; limit < 2 -> 0).                 */
int sqf2k_prime_count(uint64_t limit, uint64_t *count);
/* All primes <= limit, ascending, as int64 (PrimeTable.primes dtype).
 * cap = capacity of out; *count = number written (== pi(limit)).          */
int sqf2k_primes(uint64_t limit, int64_t *out, uint64_t cap, uint64_t *count);

/* ---- L1: segment sieve  (replaces sieve.py:72-111 sieve_segment) ------ */

/* Squarefree flags of the odd n in [start, end) packed LSB-first into
 * nbytes = ceil(n_slots/64)*8 bytes, using the caller's prime table
 * (ascending int64, must cover isqrt(end-1): sieve.py:86-88).          */
int sqf2k_sieve_bits(uint64_t start, uint64_t end, const int64_t *primes,
                     uint64_t n_primes, uint8_t *out, uint64_t nbytes);

/* ---- L2: min-k scan over a two-segment window
 *      (replaces search.py:219-252 scan_segment and search.py:255-279
 *       scan_exponents; window rules of search.py:97-135) --------------- */

/* prev_bits == NULL means "no predecessor" (start of a run at n = 1).
 * Bit buffers use the Segment layout above.  failures receives the n left
 * unresolved at k_max in ascending order (up to fail_cap of them).        */
int sqf2k_scan_window(const uint8_t *prev_bits, uint64_t prev_start,
                      uint64_t prev_end, const uint8_t *cur_bits,
                      uint64_t cur_start, uint64_t cur_end, uint32_t k_max,
                      sqf2k_summary_t *out, uint64_t *failures,
                      uint64_t fail_cap);
/* Per-slot smallest exponent (uint8, 0 = unresolved or n = 1).           */
int sqf2k_scan_exponents(const uint8_t *prev_bits, uint64_t prev_start,
                         uint64_t prev_end, const uint8_t *cur_bits,
                         uint64_t cur_start, uint64_t cur_end, uint32_t k_max,
                         uint8_t *kvals, uint64_t n_slots);

/* ---- L4 hot loop: verify a whole range on the GPU
 *      (replaces the segment loop of runner.py:216-252: prime table,
 *       predecessor seeding, sieve, scan and merge of every segment) ----- */

/* Smallest exponent of every odd n in [start, end), n = 1 excluded, up to
 * k_max (1..63).  Equivalent to merging scan_segment over any segmentation
 * of the range with true predecessors (runner.py:93-102).  failures gets
 * the n unresolved at k_max, ascending (before the k <= 63 recheck).    */
int sqf2k_verify(uint64_t start, uint64_t end, uint32_t k_max,
                 const sqf2k_verify_opts_t *opts, sqf2k_summary_t *out,
                 uint64_t *failures, uint64_t fail_cap);

/* ---- failure recheck  (replaces runner.py:105-114 _recheck_failure) ---- */

/* For each n[i]: least k in [1, 63] with n - 2^k >= 1 squarefree, decided by
 * exact trial division by p^2 for the primes <= isqrt(prime_limit) (the run's
 * prime table, runner.py:192); 0 when none.  prime_limit >= isqrt(n[i]). */
int sqf2k_recheck(const uint64_t *n, uint64_t count, uint64_t prime_limit,
                  int32_t *k_out);

/* Squarefree flag of each n[i] >= 1 by exact trial division on the GPU
 * (replaces sieve.py:114-131 is_squarefree_oracle); same prime rule.   */
int sqf2k_is_squarefree(const uint64_t *n, uint64_t count, uint64_t prime_limit,
                        uint8_t *out);

/* ---- profiling -------------------------------------------------------- */

/* When enabled every library kernel launch is bracketed by CUDA events on
 * the library stream; sqf2k_profile_read returns the accumulated device
 * time per kernel name.                                                  */
int sqf2k_profile_enable(int on);
int sqf2k_profile_reset(void);
int sqf2k_profile_read(sqf2k_kstat_t *out, int cap, int *n);
/* Synchronise the library stream.                                        */
int sqf2k_sync(void);
/* The library's cudaStream_t (as void*), for callers that time on it with
 * their own CUDA events (bench.py wraps it in torch.cuda.ExternalStream). */
void *sqf2k_stream(void);
/* Host<->device bytes the library copied since the last profile reset.   */
int sqf2k_copy_stats(uint64_t *h2d_bytes, uint64_t *d2h_bytes);

#ifdef __cplusplus
}
#endif

#endif /* SQF2K_B200_H */
