/*
 * aa.h — C ABI of libaa: the Anderson-acceleration hot path of
 * Lockhart, Gardner, Woodward, Thomas, Olson, "Performance of Low
 * Synchronization Orthogonalization Methods in Anderson Accelerated Fixed
 * Point Solvers" (arXiv 2110.09667), built for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n.
 *
 * One AA iteration (Alg. 1 l.3-7, with Alg. 2, inside):
 *   f_i = G(x_i) - x_i;  Delta f_{i-1} = f_i - f_{i-1};  Delta g_{i-1} = G(x_i) - G(x_{i-1})
 *   if the window is full: QRDelete (Givens)
 *   QRAdd_{MGS | ICWY | CGS2 | DCGS2} (Algs. 3-6)
 *   solve R gamma = Q^T f_i (Alg. 2 l.9)
 *   x_{i+1} = G(x_i) - G_i gamma (Alg. 1 l.7)
 * Every step runs in libaa's CUDA kernels; each global reduction of a
 * distributed run is exactly one ncclAllReduce (sum, fp64) of an O(m)-word
 * vector.  Numbers are IEEE fp64 throughout.
 *
 * CONVENTIONS
 *  - Vector arguments named x*, gx*, v are DEVICE pointers to n_local fp64
 *    values, 16-byte aligned (else AA_ERR_ARG).  The caller owns them; libaa
 *    reads/writes them only inside the stream-ordered work of the call and
 *    never retains them.  Output vectors may alias inputs of the same call
 *    (every row is read before it is written).
 *  - libaa owns Q, R, T, the Delta G window, f_{i-1}, G(x_{i-1}) and all
 *    scratch: (2m+2) vectors of n_local (padded to a multiple of 256 rows) plus
 *    O(m^2) words, allocated once in aa_create.
 *  - aa_init / aa_step / aa_delete_oldest only ENQUEUE on the handle's stream
 *    and return without a host synchronisation.  aa_stats synchronises.
 *  - A handle belongs to the CUDA device that was current at aa_create; call
 *    it with that device current (one process per GPU is the intended use).
 *  - Host control flow depends only on (i, m_i, variant, options), all known
 *    on the host; no device->host transfer happens per iteration.
 *  - Errors: argument errors return immediately with no state change.  A CUDA
 *    or NCCL failure makes the handle sticky-failed: every later call except
 *    aa_stats / aa_destroy / aa_status_string returns the same error.
 *  - Collective calls (nranks > 1): aa_create, aa_step, aa_delete_oldest,
 *    aa_stats, aa_destroy must be called by every rank in the same order with
 *    the same m / variant / options.  n_local may differ per rank (contiguous
 *    row blocks).
 *  - Handles are not thread-safe.  One handle per solve.
 *
 * BREAKDOWN (reading A12: the paper is silent on linear dependence in the window; SPEC
 * S:145).  K4 tests the step's new column on the
 * device: R_kk <= eps_a ||Delta f_{i-1}|| (eps_a = 10 eps sqrt(n_global) by default,
 * n_global = the sum of every rank's n_local, so all ranks use the same threshold; the two
 * norms are global reduction results, so all ranks take the same decision).  Then:
 *  - that step degrades to gamma = 0: x_{i+1} = G(x_i) exactly (Alg. 1 l.1 restarted from
 *    x_i; no damping term), and a flag is set that stays set until aa_reset or aa_init;
 *  - while the flag is set every further aa_step also degrades to x_{i+1} = G(x_i) (the
 *    window holding the dependent column is never used again; it keeps f_{i-1}, G(x_{i-1})
 *    current, so aa_reset restarts Alg. 2 at the right place);
 *  - the flag is surfaced by aa_stats (returns AA_ERR_BREAKDOWN with the stats filled)
 *    and, with nranks == 1, at aa_step entry: a mapped pinned word written by K4 is polled
 *    without blocking and aa_step returns AA_ERR_BREAKDOWN without enqueuing anything
 *    (steps enqueued before K4 ran are the degraded steps above);
 *  - the caller applies SPEC's policy: aa_reset once; a breakdown again on the first
 *    step after the reset is a hard error.  The handle is not failed by a breakdown.
 *  - AA_OPT_BREAKDOWN_EPS = 0 disables the test except for R_kk = 0 or NaN (stress runs).
 */
#ifndef AA_H
#define AA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aa_ctx* aa_handle_t;

/* QRAdd variants (Algs. 3-6). */
enum aa_variant {
    AA_QR_MGS = 0,   /* Alg. 3: m_i dependent reductions per add (baseline)            */
    AA_QR_ICWY = 1,  /* Alg. 4: inverse compact WY MGS, 2 reductions (+1 after delete)  */
    AA_QR_CGS2 = 2,  /* Alg. 5: CGS with reorthogonalisation, 3 reductions              */
    AA_QR_DCGS2 = 3  /* Alg. 6: delayed CGS-2, 2 reductions                             */
};

enum aa_status {
    AA_OK = 0,
    AA_ERR_ARG = 1,        /* bad pointer / size / option / call order                  */
    AA_ERR_STATE = 2,      /* call not allowed in the current state                     */
    AA_ERR_CUDA = 3,       /* CUDA runtime failure (sticky)                              */
    AA_ERR_NCCL = 4,       /* NCCL failure or NCCL library unavailable (sticky)         */
    AA_ERR_NOMEM = 5,      /* device allocation failed in aa_create                     */
    AA_ERR_BREAKDOWN = 6   /* a new column was (numerically) linearly dependent:
                              R_kk <= eps_a ||Delta f|| (or NaN), reading A12 (S:145,
                              S:215).  NOT sticky-failed: see "BREAKDOWN" below          */
};

/* Options for aa_set_option (call after aa_create, before aa_init). */
enum aa_option {
    AA_OPT_DAMPING_BETA = 0,   /* beta in (0,1]; default 1 = Alg. 1 exactly.  beta != 1:
                                  x_{i+1} = G(x_i) - G_i gamma - (1-beta)(f_i - Q Q^T f_i)
                                  (not in the paper; reading A13)                */
    AA_OPT_ICWY_DELETE = 1,    /* 0 = SEPARATE (paper: T update after QRDelete is its own
                                  reduction; 3 allreduces per recycle iteration);
                                  1 = MERGED into QRAdd's first reduction (2 allreduces);
                                  2 = SMALL: T' = I + strict_lower(W^T (T + T^T - I) W) from
                                  the QRDelete rotations W, no Gram pass and no reduction
                                  (2 allreduces; NOT in the paper: SURVEY.md §8(f) row 1,
                                  DESIGN.md A6b).  Choosing SMALL after aa_init returns
                                  AA_ERR_STATE; aa_delete_oldest always uses the rebuild. */
    AA_OPT_DCGS2_COND = 2,     /* reorthogonalise when m_i > val; paper: 3 (Alg. 6 l.2);
                                  2 is the shape-allowed alternative (reading A2)          */
    AA_OPT_DCGS2_RSCALE = 3,   /* 0 = R += s verbatim (Alg. 6 l.5); 1 = R += R_kk s (A3)  */
    AA_OPT_BREAKDOWN_EPS = 4,  /* eps_a; default 10 * DBL_EPSILON * sqrt(n_global)        */
    AA_OPT_PROFILE = 5,        /* 1 = record per-kernel CUDA events (aa_timings)           */
    AA_OPT_N_GLOBAL = 6,       /* global vector length (for the default eps_a)             */
    AA_OPT_FUSED_ALLREDUCE = 7, /* 1 = every global reduction is a one-shot exchange done by
                                  the producing kernel's last CTA over NVLink peer memory
                                  (CUDA IPC, same node) instead of ncclAllReduce; collective
                                  (all ranks set it); 0 = ncclAllReduce (default).  If the
                                  IPC setup fails the call returns its error and the handle
                                  keeps using ncclAllReduce (not sticky)                    */
    AA_OPT_CONV_NORM = 8,      /* ||x_{i+1} - x_i|| of Alg. 1 l.8:
                                  0 = LAGGED (default): the local partial rides in the next
                                  step's first reduction; aa_stats sums it over ranks on
                                  demand (one extra allreduce per aa_stats call if p > 1).
                                  1 = IMMEDIATE: aa_step performs that allreduce itself
                                  (one more physical reduction per iteration, as the paper's
                                  loop checks the norm every iteration).
                                  2 = OFF: not reported (aa_stats dx_norm = -1), no
                                  norm_check in the ledger.                                 */
    AA_OPT_DETERMINISTIC = 9   /* 0 (default): reductions are summed in a fixed order
                                  (per-CTA partials in CTA order, ranks in rank order), so
                                  results are bitwise reproducible for a given n_local, m,
                                  variant and rank count.
                                  1: also bitwise identical ACROSS rank counts (SURVEY.md
                                  §8(e)): every kernel sums its rows in fixed chunks of 65536
                                  rows (one CTA per chunk, rows in a fixed order inside), the
                                  chunk partials in a power-of-two-aligned pairwise tree over
                                  the chunk index, and the ranks' sums in the same tree over
                                  the rank index (fused exchange: in the kernel; NCCL: one
                                  ncclAllGather + a summing kernel instead of ncclAllReduce).
                                  The iterates and factors of p ranks then equal those of one
                                  GPU bit for bit when every rank holds the same power-of-two
                                  number of chunks.  Requires n_local % 65536 == 0 (else
                                  AA_ERR_ARG); allocates n_local / 65536 partial slots
                                  (AA_ERR_NOMEM).  Collective (all ranks set it).  aa_stats'
                                  norms are still summed by ncclAllReduce.                   */
};

/* aa_stats flags */
#define AA_STATS_LOO 1     /* also compute ||I - Q^T Q||_F (one Gram pass + 1 allreduce) */
#define AA_STATS_RESET 2   /* reset cumulative counters after reading                    */

/* Ledger phases (logical synchronisations of the paper's counting). */
enum aa_phase { AA_PH_QRADD = 0, AA_PH_QRDELETE = 1, AA_PH_LSP_RHS = 2, AA_PH_NORM = 3,
                AA_PH_OTHER = 4 };

struct aa_stats {
    int64_t iter;              /* AA iterations done (Alg. 1 loop index i)                  */
    int32_t m_i;               /* active window columns                                     */
    int32_t sync_points_last;  /* global reduction points in the last aa_step              */
    int32_t allreduce_last;    /* physical ncclAllReduce calls in the last aa_step (0 if p=1)*/
    int32_t pad0;
    int64_t allreduce_total;
    int64_t logical_sync[5];   /* cumulative, by aa_phase (paper ledger)                    */
    int64_t logical_sync_last[5];
    double f_norm;             /* ||f_i||_2 of the last step (global)                       */
    double dx_norm;            /* ||x_{i+1} - x_i||_2 of the last step (global)             */
    double r_ratio_min;        /* min over the run of R_kk / ||Delta f|| (breakdown margin)  */
    double loo;                /* ||I - Q^T Q||_F if AA_STATS_LOO, else -1                  */
    int32_t breakdown;         /* breakdown flag, sticky until aa_reset / aa_init           */
    int32_t breakdown_count;   /* steps that broke down since aa_init                       */
};

/* NCCL rendezvous: rank 0 calls this, broadcasts the 128 bytes (e.g. with
 * torch.distributed), every rank passes them to aa_create.  Needs libnccl.so.2
 * at run time (dlopen); AA_ERR_NCCL if unavailable. */
int aa_comm_unique_id(void* id128);

/* Create a solver for n_local local rows, window depth m (1 <= m <= 64), QRAdd
 * variant (enum aa_variant).  nranks == 1: no communicator (id128 may be NULL).
 * cuda_stream: the cudaStream_t every call enqueues on; NULL = the CUDA legacy
 * default stream (so work is ordered with a caller that uses stream 0).
 * Collective over the ranks when nranks > 1. */
int aa_create(aa_handle_t* h, int64_t n_local, int m, int qr_variant, int rank, int nranks,
              const void* id128, void* cuda_stream);
/* Same as aa_create with nranks > 1, but BORROWS an already-initialised NCCL
 * communicator (ncclComm_t of nranks ranks, this process = rank), e.g. the one a
 * torch.distributed NCCL process group owns.  libaa never frees it; the caller must
 * not destroy it before aa_destroy and must not run other collectives on it
 * concurrently with libaa calls. */
int aa_create_with_comm(aa_handle_t* h, int64_t n_local, int m, int qr_variant, int rank, int nranks,
                        void* nccl_comm, void* cuda_stream);
int aa_set_option(aa_handle_t h, int opt, double val);

/* Alg. 1 l.1: f_0 = G(x_0) - x_0, remember G(x_0) and f_0, x1_out = G(x_0).
 * x1_out may alias gx0.  Resets the window. */
int aa_init(aa_handle_t h, const double* x0, const double* gx0, double* x1_out);

/* One AA iteration (Alg. 1 l.3-7 with Alg. 2): given x_i and G(x_i) produce x_{i+1}.
 * QRDelete is fused in automatically when the window is full (m_i == m).  The library
 * asserts its reduction schedule: if a step issued a number of global reductions other than
 * the paper's count (plus ICWY's separate delete reduction, A6, and the
 * IMMEDIATE norm), it returns AA_ERR_STATE (sticky) and prints the two counts. */
int aa_step(aa_handle_t h, const double* x_i, const double* gx_i, double* x_next);
/* (aa_step returns AA_ERR_BREAKDOWN, enqueuing nothing, when nranks == 1 and an earlier step
 * broke down and aa_reset has not been called since; see BREAKDOWN above.) */

/* Same computation with HOST buffers (pinned or pageable): copies in, runs aa_step,
 * copies x_next back and synchronises.  x_i_host may be NULL: then x_i is the x_{i+1} the
 * previous aa_step_host call of this handle returned (kept on the device; AA_ERR_STATE if
 * there was none since aa_init, or an aa_step came in between), so a host-side loop
 * x -> G(x) uploads only G(x_i) per iteration.  At n_local >= 4M rows the copies go in row
 * chunks overlapped with K1 (uploads) and K4 (downloads).  Like aa_step it returns
 * AA_ERR_BREAKDOWN at entry (nranks == 1) before touching anything, so after aa_reset the
 * same call -- x_i_host = NULL included -- can be repeated. */
int aa_step_host(aa_handle_t h, const double* x_i_host, const double* gx_i_host,
                 double* x_next_host);

/* Stand-alone Givens QRDelete of the oldest window column:
 * rotates Q and R, drops the oldest Delta G column; ICWY also rebuilds T with
 * one reduction.  aa_step calls the fused form automatically. */
int aa_delete_oldest(aa_handle_t h);

/* Synchronises the stream and reports counters; see struct aa_stats.  Returns
 * AA_ERR_BREAKDOWN if the breakdown flag is set (stats still filled).  Collective when
 * nranks > 1: every call does ONE allreduce of {this rank's lagged ||x_{i+1}-x_i||^2
 * partial, an error flag}, so the ranks agree: if any rank's handle failed (e.g. a fused
 * exchange timed out) every rank returns AA_ERR_NCCL.  AA_STATS_LOO adds one more. */
int aa_stats(aa_handle_t h, struct aa_stats* out, int flags);

/* Empty the window and clear the breakdown flag (restart policy after a breakdown,
 * S:256).  The next aa_step behaves like Alg. 2's i = 1 branch with
 * Delta f = f_i - f_{i-1} of the last two iterates.  Synchronises the stream. */
int aa_reset(aa_handle_t h);

int aa_destroy(aa_handle_t h);
const char* aa_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* AA_H */
