// aa_device.cuh — libaa device-side data structures, PTX wrappers (TMA bulk copy,
// mbarrier, fp64 DMMA) and the O(m^2) small-factor routines (K3) of the AA hot
// path of arXiv 2110.09667.  P:n = PAPER.md line n.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace aa {

constexpr int MMAX = 64;                 // largest window depth m
constexpr int NT = 256;                  // threads per CTA (8 warps)
constexpr int NWARP = NT / 32;
constexpr int NIN_MAX = 2 * MMAX + 4;    // input column streams of one kernel
constexpr int LRED = 2304;               // words per reduction slot (>= 4+3*63+63*62/2)
constexpr int NSLOT = MMAX + 2;          // reduction slots per iteration
constexpr int PB_COLS_PER_WARP = 9;      // ceil((MMAX+2)/NWARP)

enum Op : int {
  OP_K1 = 0,        // prologue (Delta f / Delta g) + streaming Givens + block multi-dot
  OP_K2_ICWY = 1,   // Alg. 4 l.5: Delta f - Q T^{-1} r, norms
  OP_K2_DCGS2 = 2,  // Alg. 6 l.4 + l.7: delayed reorthogonalisation + projection, norms
  OP_K2A_CGS2 = 3,  // Alg. 5 l.2-3: y = Delta f - Q s, z = Q^T y
  OP_K2B_CGS2 = 4,  // Alg. 5 l.4: Delta f = y - Q z, norms
  OP_K2_MGS = 5,    // Alg. 3 l.3 + next l.2: one axpy + one dot (or the norm)
  OP_K4 = 6,        // Alg. 2 l.9 + Alg. 1 l.7: gamma, x_{i+1} = G(x_i) - G_i gamma; commit
  OP_GRAM = 7       // diagnostic: lower triangle of Q^T Q (loss of orthogonality)
};

enum Variant : int { V_MGS = 0, V_ICWY = 1, V_CGS2 = 2, V_DCGS2 = 3 };

enum Flags : int {
  F_EXT_DF = 1,       // K1: the new column is caller-provided (aa_test_qradd)
  F_DELETE_ONLY = 2,  // K1/K4: stand-alone QRDelete (aa_delete_oldest)
  F_COMMIT_ONLY = 4   // K4: no rows, only the small-factor commit
};

// Replicated small factors (identical on every rank: every rank recomputes them from the
// same allreduce results).  Double-buffered: every kernel of a step reads version `ver`;
// CTA 0 of the step's last kernel (K4) writes version `ver ^ 1` straight from its head
// (no other CTA reads it during that kernel), so nothing is recomputed at commit time.
// Each version also carries the QRDelete of its own R precomputed (Givens coefficients
// and the re-triangularised R), so the next recycle step's heads only load them.
struct Factors {
  double R[MMAX * MMAX];     // column-major, leading dim MMAX, K x K valid
  double T[MMAX * MMAX];     // ICWY: I + L (reading A5), column-major
  double Rdel[MMAX * MMAX];  // R after QRDelete: (K-1) x (K-1)
  double Tdel[MMAX * MMAX];  // ICWY_DELETE = SMALL: T after QRDelete, rows 0..K-3 (variant, A6b)
  double scale[MMAX];        // lazy normalisation: Q_j(true) = scale[j] * Q_j(stored)
  double gamma[MMAX];
  double cs[MMAX], sn[MMAX]; // Givens coefficients of QRDelete(R)
  int K;                     // columns of R
  int has_del;
};

struct SmallState {
  Factors f[2];
  // QRDelete precompute, early part (written by this step's K1 spare CTA, read by its K4):
  // rotations 0..k-3 of the next QRDelete depend only on the factor before this step's
  // QRAdd, so they are computed while K1 streams; R' columns 0..k-3 (upper triangles)
  double gpre_R[MMAX * MMAX];
  double gpre_cs[MMAX], gpre_sn[MMAX];
  // ---- scalar tail (aa_stats copies only this part)
  double dx2_local;          // this rank's ||x_{i+1} - x_i||^2 from the last update
  double dx2_global;         // CONV_NORM = IMMEDIATE: the same, summed over ranks by aa_step
  double dx2_acc;            // chunked K4: ||x_{i+1} - x_i||^2 accumulated over row chunks
  double f2;                 // ||f_i||^2 (global) of the last step
  double rratio_min;         // min R_kk / ||Delta f||
  double last_rkk;
  int breakdown;             // sticky until aa_reset: a step broke down (reading A12); while set,
                             // every step degrades to gamma = 0 (x_{i+1} = G(x_i))
  unsigned int counter;      // cross-CTA arrival ticket
  int xchg_timeout;          // sticky: a fused peer exchange timed out
  int breakdown_count;       // steps that broke down since aa_create (kept by aa_reset)
};

// K1 reduction-slot layout (words), identical on host and device.
struct K1Layout {
  int off_df, off_f, off_x, n_x, off_gram, n_gram, words;
  __host__ __device__ static K1Layout make(int k, bool has_x, bool has_gram) {
    K1Layout L;
    L.off_df = 4;
    L.off_f = 4 + k;
    L.off_x = 4 + 2 * k;
    L.n_x = (has_x && k >= 2) ? k - 1 : 0;
    L.off_gram = L.off_x + L.n_x;
    L.n_gram = (has_gram && k >= 3) ? (k - 1) * (k - 2) / 2 : 0;
    L.words = L.off_gram + L.n_gram;
    return L;
  }
};

constexpr int NVEC_MAX = 8;   // 1-D vector streams per kernel
// AA_OPT_DETERMINISTIC: rows are summed in fixed chunks of DET_ROWS rows
// (one CTA per chunk, a fixed order inside), chunk partials in a power-of-two-aligned
// pairwise tree over the chunk index, ranks in the same tree over the rank index
constexpr long long DET_ROWS = 65536;
constexpr int MAX_RANKS = 8;  // fused NVLink exchange: ranks of one node
constexpr int NBLK_MAX = 3;   // 2-D column blocks (tensor maps) per kernel

// Kernel parameters.  Inputs of one tile are staged in shared memory as columns:
// first the nvec vectors (1-D bulk copies), then the nblk column blocks (one 2-D
// tensor-map TMA each, box = TR rows x blk_ncols columns).  Column c of a stage
// lives at stage + c*TR.
struct alignas(64) KParams {
  CUtensorMap tm[NBLK_MAX];   // 2-D maps over Q or the Delta G ring (rows x m columns)
  int blk_gcol[NBLK_MAX];     // first global column of each block
  int blk_which[NBLK_MAX];    // host bookkeeping: 0 = Q, 1 = Delta G ring
  int blk_ncols[NBLK_MAX];
  int nblk, nvec;
  const double* vec[NVEC_MAX];
  unsigned exact_vec;         // bit i: vec[i] is a caller buffer (exactly n rows)
  int op, variant, flags;
  int m;            // window capacity
  int k;            // existing columns after QRDelete (new column index)
  int c_in;         // K1: Q columns read (m at recycle, k at start-up); GRAM: columns
  int recycle;      // QRDelete fused into this step
  int has_x;        // K1: Q_{0:k-2}^T q_{k-1} needed (ICWY T row / DCGS-2 s)
  int gram;         // 0 none, 1 strict lower k x k (ICWY after delete), 2 lower incl. diag
  int reortho;      // DCGS-2 delayed reorthogonalisation active this step
  int rscale;       // DCGS-2 R update reading A3
  int icwy_merged;  // ICWY T update after QRDelete: 0 separate, 1 merged, 2 small-matrix (no Gram)
  int mgs_j;        // MGS pass index j (1..k)
  int final_slot;   // reduction slot holding (||v'||^2, v'^T f)
  int red_slot;     // slot this kernel writes
  int words;        // words this kernel reduces
  int red_words0;   // words of reduction slot 0 the heads stage into shared memory
  long long rbeg;   // first row of this launch (rows [rbeg, n)); 0 except chunked aa_step_host
  int chunk_first;  // first / last row-chunk launch of this op in the step (both 1 unchunked):
  int chunk_last;   // reductions accumulate over chunks; side effects happen once
  int pre_cta;      // K4 at small n: CTA 0 only writes the next factors + QRDelete precompute
                    // (no tiles); tiles go to CTAs 1..gridDim-1.  K1 at small n: CTA 0 only
                    // computes the early rotations of the next QRDelete (k1_delete_pre)
  int k1_pre;       // K1: compute the early rotations if a spare CTA exists; K4: K1 did (use them)
  unsigned long long* tl;   // test-only phase timeline (CTA 0 / last CTA, %globaltimer ns), or null
  int nin, tr, stages;
  int vb;           // first vector column (= sum of block columns)
  int tm3d;         // column blocks use 3-D maps (TR a multiple of 256)
  int k1_tmastore;  // K1: full tiles write their outputs with TMA stores from the stage
                    // (rotated Q block + Delta f in one tensor store; f, G(x), Delta g 1-D)
  int beta_on;
  long long n;      // local rows
  double beta, eps_a;
  double* Q;        // Q base (column j at Q + j*ld)
  long long ld;
  double* fp;       // f_{i-1} -> f_i
  double* gp;       // G(x_{i-1}) -> G(x_i)
  double* dg_out;   // Delta G ring slot written by K1
  double* x_out;    // K4 output
  SmallState* st;
  int ver;          // factor version read by this step (written: ver ^ 1, by K4)
  // fused one-shot allreduce over NVLink peer memory (AA_OPT_FUSED_ALLREDUCE): the last
  // CTA exchanges words [xoff[e], xoff[e]+xcnt[e]) of its reduction slot, e < nxchg,
  // with sequence numbers xseq + 1 + e (the counter is advanced by that CTA)
  int nxchg, nranks, rank;
  int xoff[2], xcnt[2];
  unsigned long long* xseq;               // this rank's exchange sequence counter (device word in
                                          // the mailbox buffer's header; never reset, so tags stay
                                          // fresh across graph replays and aa_reset)
  double* pmbox[MAX_RANKS];               // peer q's mailbox (q == rank: local)
  double* lmbox;
  double* red;      // reduction slots (slot s at red + s*LRED)
  double* part;     // per-CTA partials (CTA b at part + b*LRED)
  int* bd_host;     // device alias of the handle's mapped pinned breakdown word (polled by aa_step)
  int det_tpc;      // deterministic mode: tiles per DET_ROWS chunk (CTA b = chunk b); 0 = off
  long long scr_off; // head scratch at stage0 + scr_off doubles (0: aliases the stage ring)
  int early_tma;    // the first tiles' loads may be issued before the heads (AA_NO_EARLY_TMA=1: off)
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA 2-D tensor copy global -> shared (box at coordinates {row, col}); rows past the
// tensor's extent are zero-filled.
__device__ __forceinline__ void tma_2d_g2s(void* dst, const CUtensorMap* map, int row, int col, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(row), "r"(col), "r"(smem_u32(bar))
      : "memory");
}
// TMA 3-D tensor copy: Q viewed as {256 rows, row block, column}; one box brings TR =
// 256*k rows x ncols columns into the [column][TR] stage layout.
__device__ __forceinline__ void tma_3d_g2s(void* dst, const CUtensorMap* map, int rblk, int col, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(rblk), "r"(col), "r"(smem_u32(bar))
      : "memory");
}
// TMA stores shared -> global (bulk-group completion): a 3-D / 2-D tensor box of Q (the same
// maps as the loads), and 1-D bulk copies for vectors.  Rows outside the tensor are not
// written.  The smem source must have been made visible to the async proxy
// (fence.proxy.async by the writing threads, then a barrier) before the issue.
__device__ __forceinline__ void tma_3d_s2g(const CUtensorMap* map, int rblk, int col, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(0), "r"(rblk), "r"(col), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_2d_s2g(const CUtensorMap* map, int row, int col, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(row), "r"(col), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem sources of every committed store have been read (the stage may be refilled)
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed store has been performed (global writes complete)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// fp64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col)
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ K3: small factors
// All routines run on ONE warp (lanes cooperate over columns / rows) with operands
// in shared memory, leading dimension MMAX, and end with __syncwarp().

// Leading dimension of R staged in shared memory: MMAX + 1, so that lane = column accesses
// (R[i + l LDR] for l = lane) hit at most 2 banks instead of 32 (SHFL and LDS/STS share the
// MIO pipe: conflicted accesses delay the shuffles on the serial chain).
constexpr int LDR = MMAX + 1;

// QRDelete on R (reading A7): drop column 0 of the mold x mold
// factor, re-triangularise the upper-Hessenberg remainder H = R[:, 1:] with mold-1 Givens
// rotations of adjacent rows, rho = hypot(a,b) >= 0.  IN PLACE in shared memory (leading
// dimension LD): on return R's columns 0..mold-2 hold R' in their upper triangle (entries
// below the diagonal are left stale; callers copy the triangle), and cs/sn (shared) the
// rotation coefficients (applied to Q's columns by K1).
// Register form: lane l owns Hessenberg columns l and l+32; "carry" is the column's entry
// in the row being rotated (row j at step j), row j+1 is still the original R and is
// prefetched one step ahead, so the serial chain per step is one shuffle, one reciprocal
// square root and a few products.  Step j writes row j of columns j+1.. and rho into
// (j, j): no lane reads those again, and with LD = MMAX + 1 the column-per-lane stores
// hit at most two banks (they share the MIO pipe with the shuffle).
// rho = t * t^{-1/2}, c = a t^{-1/2}, s = b t^{-1/2} with t = a^2 + b^2 after an exact
// power-of-two scaling (one MUFU-seeded rsqrt instead of sqrt + reciprocal, no branches).
// Givens coefficients zeroing b against a: rho = hypot(a, b) >= 0, c = a / rho, s = b / rho
// (c = 1, s = 0 when a = b = 0).  (a, b) are scaled by an exact power of two so that
// max(|a|,|b|) is in [1, 2): t = a'^2 + b'^2 in [1, 8) needs no over/underflow branch; one
// rsqrt gives c, s and rho = t^{1/2} / 2^e.
__device__ __forceinline__ void givens_coef(double a, double b, double& c, double& s, double& rho) {
  const double mx = fmax(fabs(a), fabs(b));
  const int ex = (__double2hiint(mx) >> 20) & 0x7ff;             // biased exponent of mx
  const int es = ex == 0 ? 1 : (ex == 0x7ff ? 0x7fe : ex);        // zero / denormal / inf guard
  const double sc = __hiloint2double((2046 - es) << 20, 0);       // 2^(1023 - es), exact
  const double usc = __hiloint2double(es << 20, 0);               // 2^(es - 1023), exact
  const double as = a * sc, bs = b * sc;
  const double t = fma(as, as, bs * bs);
  const bool nz = mx > 0.0;
  const double ri = rsqrt(nz ? t : 1.0);
  rho = nz ? (t * ri) * usc : 0.0;
  c = nz ? as * ri : 1.0;
  s = nz ? bs * ri : 0.0;
}

template <int LD>
__device__ void k3_givens_delete(double* R, int mold, double* cs, double* sn, int* progress = nullptr) {
  const int lane = threadIdx.x & 31;
  const int nc = mold - 1;  // columns of the Hessenberg matrix
  const int l0 = lane, l1 = lane + 32;
  // H[i][l] = R[i + (l+1) LD] for i <= l+1 (R upper triangular), else 0
  auto h = [&](int i, int l) -> double { return (l < nc && i <= l + 1) ? R[i + (l + 1) * LD] : 0.0; };
  double carry0 = h(0, l0), carry1 = h(0, l1);
  double h20 = h(1, l0), h21 = h(1, l1);
  double bn = (nc > 0) ? R[1 + 1 * LD] : 0.0;
  __syncwarp();
#pragma unroll 1
  for (int j = 0; j < nc; ++j) {
    const double b = bn;                        // H[j+1][j], original
    const double n20 = h(j + 2, l0), n21 = h(j + 2, l1);   // next step's row j+2
    bn = (j + 1 < nc) ? R[(j + 2) + (j + 2) * LD] : 0.0;
    const double a = __shfl_sync(0xffffffffu, j < 32 ? carry0 : carry1, j & 31);
    double c, s, rho;
    givens_coef(a, b, c, s, rho);
    const bool act0 = l0 > j && l0 < nc, act1 = l1 > j && l1 < nc;
    const double o0 = __dadd_rn(__dmul_rn(c, carry0), __dmul_rn(s, h20));
    const double o1 = __dadd_rn(__dmul_rn(c, carry1), __dmul_rn(s, h21));
    carry0 = act0 ? __dadd_rn(__dmul_rn(-s, carry0), __dmul_rn(c, h20)) : carry0;
    carry1 = act1 ? __dadd_rn(__dmul_rn(-s, carry1), __dmul_rn(c, h21)) : carry1;
    if (act0) R[j + l0 * LD] = o0;              // R'[j][l] (R' column l = R column l)
    if (act1) R[j + l1 * LD] = o1;
    if (lane == 0) {
      R[j + j * LD] = rho;
      cs[j] = c;
      sn[j] = s;
      if (progress) {   // publish rotation j to a consumer warp (k3_rotate_sym)
        __threadfence_block();
        *reinterpret_cast<volatile int*>(progress) = j + 1;
      }
    }
    h20 = n20;
    h21 = n21;
  }
  __syncwarp();
}

// Two-sided application of the QRDelete rotations to a symmetric P x P matrix S in shared
// memory (leading dimension LDS, both triangles stored): S <- G_j^T S G_j for j = 0..P-2,
// where G_j mixes columns (then rows) j and j+1 as K1 mixes Q's columns.  Entries with both
// indices <= P-2 are then W^T S W restricted to them (rotation P-1 would only touch row /
// column P-1).  One pass per rotation: lane i (i != j, j+1) rotates (S[i][j], S[i][j+1]) and
// writes both symmetric copies; one lane updates the 2 x 2 diagonal block in closed form.
// With progress != nullptr the rotations are consumed as another warp publishes them.
template <int LDS>
__device__ void k3_rotate_sym(double* S, int P, const double* cs, const double* sn,
                              const int* progress = nullptr) {
  const int lane = threadIdx.x & 31;
  const int i0 = lane, i1 = lane + 32;
#pragma unroll 1
  for (int j = 0; j + 1 < P; ++j) {
    if (progress) {   // rotation j is produced by another warp (k3_givens_delete)
      if (lane == 0)
        while (*reinterpret_cast<const volatile int*>(progress) <= j) {
        }
      __syncwarp();
      __threadfence_block();
    }
    const double c = *reinterpret_cast<const volatile double*>(cs + j);
    const double s = *reinterpret_cast<const volatile double*>(sn + j);
    double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
    const bool u0 = i0 < P && i0 != j && i0 != j + 1, u1 = i1 < P && i1 != j && i1 != j + 1;
    if (u0) { a0 = S[i0 + j * LDS]; b0 = S[i0 + (j + 1) * LDS]; }
    if (u1) { a1 = S[i1 + j * LDS]; b1 = S[i1 + (j + 1) * LDS]; }
    double p = 0.0, q = 0.0, r = 0.0;
    if (lane == 0) { p = S[j + j * LDS]; q = S[(j + 1) + j * LDS]; r = S[(j + 1) + (j + 1) * LDS]; }
    __syncwarp();
    if (u0) {
      const double na = c * a0 + s * b0, nb = -s * a0 + c * b0;
      S[i0 + j * LDS] = na;  S[i0 + (j + 1) * LDS] = nb;
      S[j + i0 * LDS] = na;  S[(j + 1) + i0 * LDS] = nb;
    }
    if (u1) {
      const double na = c * a1 + s * b1, nb = -s * a1 + c * b1;
      S[i1 + j * LDS] = na;  S[i1 + (j + 1) * LDS] = nb;
      S[j + i1 * LDS] = na;  S[(j + 1) + i1 * LDS] = nb;
    }
    if (lane == 0) {   // [p q; q r] -> G^T [p q; q r] G
      const double cc = c * c, ss = s * s, cs2 = 2.0 * c * s;
      const double pn = cc * p + cs2 * q + ss * r;
      const double rn = ss * p - cs2 * q + cc * r;
      const double qn = (cc - ss) * q + c * s * (r - p);
      S[j + j * LDS] = pn;
      S[(j + 1) + (j + 1) * LDS] = rn;
      S[(j + 1) + j * LDS] = qn;
      S[j + (j + 1) * LDS] = qn;
    }
    __syncwarp();
  }
}

// Forward substitution with a unit lower-triangular T (Alg. 4 l.4 "T^{-1} R"; A5):
// r <- T^{-1} r in place, r has k entries in shared memory.  Lane j holds r_j (and
// r_{j+32}); step l broadcasts r_l with one shuffle; T's column l+1 is prefetched.
__device__ void k3_forward_unit_lower(const double* T, double* r, int k) {
  const int lane = threadIdx.x & 31;
  const int j0 = lane, j1 = lane + 32;
  double r0 = (j0 < k) ? r[j0] : 0.0, r1 = (j1 < k) ? r[j1] : 0.0;
  double t0 = (j0 < k && k > 0) ? T[j0] : 0.0, t1 = (j1 < k && k > 0) ? T[j1] : 0.0;
#pragma unroll 1
  for (int l = 0; l < k; ++l) {
    const double tn0 = (j0 < k && l + 1 < k) ? T[j0 + (l + 1) * MMAX] : 0.0;
    const double tn1 = (j1 < k && l + 1 < k) ? T[j1 + (l + 1) * MMAX] : 0.0;
    const double rl = __shfl_sync(0xffffffffu, l < 32 ? r0 : r1, l & 31);
    if (j0 > l && j0 < k) r0 -= t0 * rl;
    if (j1 > l && j1 < k) r1 -= t1 * rl;
    t0 = tn0;
    t1 = tn1;
  }
  if (j0 < k) r[j0] = r0;
  if (j1 < k) r[j1] = r1;
  __syncwarp();
}

// Back substitution R gamma = c (Alg. 2 l.9), R upper triangular K x K (leading dimension
// LD); c overwritten.
// Lane i holds c_i (and c_{i+32}) and 1/R_ii; step j: lane j forms gamma_j, one shuffle
// broadcasts it, every lane updates its c_i with R's column j (prefetched a step ahead).
template <int LD>
__device__ void k3_back_subst(const double* R, double* c, double* gamma, int K) {
  const int lane = threadIdx.x & 31;
  const int i0 = lane, i1 = lane + 32;
  double c0 = (i0 < K) ? c[i0] : 0.0, c1 = (i1 < K) ? c[i1] : 0.0;
  // reciprocals of the diagonal in parallel, so the serial chain has no division
  const double rinv0 = (i0 < K) ? 1.0 / R[i0 + i0 * LD] : 0.0;
  const double rinv1 = (i1 < K) ? 1.0 / R[i1 + i1 * LD] : 0.0;
  double r0 = (i0 < K && K > 0) ? R[i0 + (K - 1) * LD] : 0.0;
  double r1 = (i1 < K && K > 0) ? R[i1 + (K - 1) * LD] : 0.0;
#pragma unroll 1
  for (int j = K - 1; j >= 0; --j) {
    const double rn0 = (i0 < j && j >= 1) ? R[i0 + (j - 1) * LD] : 0.0;
    const double rn1 = (i1 < j && j >= 1) ? R[i1 + (j - 1) * LD] : 0.0;
    const double mine = (j < 32) ? c0 * rinv0 : c1 * rinv1;
    const double gj = __shfl_sync(0xffffffffu, mine, j & 31);
    if (lane == 0) gamma[j] = gj;
    if (i0 < j) c0 -= r0 * gj;
    if (i1 < j) c1 -= r1 * gj;
    r0 = rn0;
    r1 = rn1;
  }
  if (i0 < K) c[i0] = c0;
  if (i1 < K) c[i1] = c1;
  __syncwarp();
}

}  // namespace aa
