/*
 * aa_testing.h — libaa hooks for tests and benchmarks (not part of the solver API).
 * Same conventions as aa.h.
 */
#ifndef AA_TESTING_H
#define AA_TESTING_H

#include <stdint.h>
#include "aa.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Append an arbitrary column v (device, n_local fp64) to the QR factorisation with
 * the handle's QRAdd variant, exactly as aa_step appends Delta f (QRDelete first if
 * the window is full), without touching x / G state.  Needed by the orthogonality
 * stress test (config 5a): forming v as a difference of iterates would cancel. */
int aa_test_qradd(aa_handle_t h, const double* v);

/* Copy the replicated small factors to host memory (synchronises):
 * R (m x m, column-major, only the leading m_i x m_i block is meaningful), T (m x m,
 * column-major, ICWY only), gamma (m_i), scale (m: lazy 1/R_kk per Q slot). */
int aa_get_small(aa_handle_t h, double* R, double* T, double* gamma, double* scale);

/* Copy the normalised active Q columns (n_local x m_i, column-major, ld = n_local)
 * to a device buffer (applies the lazy per-column scale).  Synchronises. */
int aa_get_q(aa_handle_t h, double* q_out_dev);

/* Per-class kernel timings (ms, accumulated since the last reset) when
 * AA_OPT_PROFILE = 1.  Classes: 0 pass1 (K1), 1 project (K2), 2 update (K4),
 * 3 allreduce, 4 whole aa_step.  counts[c] = number of events. Synchronises. */
int aa_timings(aa_handle_t h, double* ms_out5, int64_t* counts5, int reset);

/* Number of libaa kernels launched since the handle was created. */
int64_t aa_kernel_launches(aa_handle_t h);

/* Counter-based SplitMix64 uniform generator on the device:
 * out[i] = lo + (hi - lo) * u(seed + stream * 2^48 + offset + i), u in [0, 1),
 * computed with __dmul_rn / __dadd_rn so it is bitwise equal to aa_inputs.uniform. */
int aa_fill_uniform(double* out_dev, int64_t n, int64_t offset, uint64_t seed, uint64_t stream,
                    double lo, double hi, void* cuda_stream);

/* Test-only phase timeline: enable = 1 allocates a 384-word device buffer; every kernel's
 * CTA 0 (slots op*16 + 0..5, K4 after its head: slot 8) and last CTA (slots 6, 7) record
 * %globaltimer (ns) at: entry, after staging, after the head, first tile ready, tiles done,
 * partials written, reduction begin, end; words 128 + slot hold clock64 at the same points.
 * out384 (host, may be NULL) receives the buffer (synchronises).  Enabled, the marks
 * themselves lengthen short phases (timer reads and global stores on the critical path):
 * use it to order phases, and ncu launch lists / PC sampling for durations. */
int aa_test_timeline(aa_handle_t h, int enable, uint64_t* out384);

/* Per-exchange latency of one global reduction, collective:
 * `iters` back-to-back exchanges of `words` fp64 words (1 <= words <= 2304).  us_fused: the
 * one-shot NVLink exchange (AA_OPT_FUSED_ALLREDUCE must be on; else -1), timed inside one
 * kernel with %globaltimer; us_nccl: ncclAllReduce on the handle's communicator, timed with
 * CUDA events on the handle's stream (one untimed call first).  Either pointer may be NULL.
 * nranks == 1: both -1. */
int aa_test_exchange(aa_handle_t h, int words, int iters, double* us_fused, double* us_nccl);

/* Build-time facts: sm target, tile rows, stages, block size (for the report). */
int aa_build_info(char* buf, int len);

#ifdef __cplusplus
}
#endif
#endif
