// aa_kernels.cuh — the streaming kernels of libaa (sm_100a).
//
// One templated persistent kernel per op.  Every op is a pass over row tiles of TR
// rows.  The op's inputs are staged in a ring of shared-memory stages by TMA: column
// blocks of Q or of the Delta G ring with ONE 2-D tensor-map copy per block per tile,
// and plain vectors (x_i, G(x_i), f_{i-1}, G(x_{i-1})) with 1-D bulk copies; the copies
// of a tile are spread over the warps (lane 0 of warp w issues copies w, w+8, ...)
// because one issuing thread sustains only ~1 copy per ~150 cycles
// (tools/stream_bench.cu).  All threads then run the op's row-wise work (phase A) out
// of shared memory and, where the op needs many dot products, a block multi-dot over
// the staged tile (phase B: lane = row, warp = column set, templated on the number of
// columns per warp; or fp64 DMMA 8x8x4 for the Gram blocks of ICWY's T rebuild).
// Per-CTA partial sums are reduced across CTAs in a fixed order by the last CTA to
// finish (deterministic), which also commits the replicated small factors.
//
// Small-factor work (K3: Givens on R, T^{-1}, back-substitution) is recomputed at the
// head of every CTA from the replicated state and the latest allreduce results, so no
// extra launch and no device->host copy is needed between reductions.
//
// Stage layout: [block 0][block 1][block 2][vectors], column c at stage + c*TR.
// Blocks start at 128-byte aligned addresses (TMA tensor copies need it).  Kernels with
// a Gram use TR in {252,124,60,28}: TR*8 bytes = 24 banks (mod 32) per column, so the
// 8-column x 4-row DMMA fragment loads are conflict-free.
#pragma once
#include "aa_device.cuh"

namespace aa {

constexpr int MAXSTAGES = 8;

// test-only phase timeline: slot s of the op's 16-slot row gets %globaltimer
#define AA_TL(s)                                                                                   \
  do {                                                                                             \
    if (p.tl && threadIdx.x == 0) {                                                                \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      p.tl[OP * 16 + (s)] = t_;                                                                    \
      p.tl[128 + OP * 16 + (s)] = (unsigned long long)clock64();                                   \
    }                                                                                              \
  } while (0)

// the same from lane 0 of the calling warp (warp-specialised sections)
#define AA_TLW(s)                                                                                  \
  do {                                                                                             \
    if (p.tl && (threadIdx.x & 31) == 0) {                                                         \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                       \
      p.tl[OP * 16 + (s)] = t_;                                                                    \
      p.tl[128 + OP * 16 + (s)] = (unsigned long long)clock64();                                   \
    }                                                                                              \
  } while (0)

struct HeadArea {
  double coef[NIN_MAX];
  double coef2[MMAX + 2];
  double sc[NIN_MAX];
  double cs[MMAX];
  double sn[MMAX];
  double2 rot[2 * MMAX];   // K1: {c_j, s_j*sc_{j+1}}, {-s_j, c_j*sc_{j+1}} (scale folded in)
  double scal[8];
  double redw[NWARP][4];
  int lcol[MMAX + 2];
  int rcol[4];
  int na, nr, is_last, gdone;   // gdone: Givens rotations published (K4, ICWY SMALL)
  int bd;                       // K4: this step degrades to gamma = 0 (breakdown, reading A12)
  int K4_K;                     // K4 CTA 0: columns of the new factor (warp 0 -> warp 1)
  double K4_rkk;                // K4 CTA 0: R_kk of the new column
  unsigned long long xbase;     // last CTA: sequence number before this kernel's exchanges
};

__host__ __device__ constexpr size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
__host__ __device__ constexpr size_t head_bytes() { return align_up(sizeof(HeadArea), 128); }
__host__ __device__ constexpr size_t bar_bytes() { return 128; }
// scratch for the head / commit (aliases the stage ring before and after the pipeline)
// scratch (aliases the stage ring before / after the pipeline):
// [Rw MMAX x LDR][Tw MMAX^2][v1, cvec, cvec2, spare: 4 x MMAX][R0: copy of reduction slot 0]
// [RF: 8 words]
constexpr size_t SCR_TW = (size_t)MMAX * LDR;
constexpr size_t SCR_V = SCR_TW + MMAX * MMAX;
constexpr size_t SCR_R0 = SCR_V + 4 * MMAX;
constexpr size_t SCR_RF = SCR_R0 + LRED;
__host__ __device__ constexpr size_t scratch_bytes() { return (SCR_RF + 8) * sizeof(double); }
// K4's CTA 0: the Givens workspace Rg (copy of the new R, m x LDR), then for ICWY SMALL the
// symmetric S of k4_tdel (m x LDR)
constexpr size_t SCR_RG = SCR_RF + 8;
__host__ __device__ constexpr size_t scr_s(int m) { return SCR_RG + (size_t)m * LDR; }
__host__ __device__ constexpr size_t scratch_bytes_k4(int m, bool tdel) {
  return (scr_s(m) + (tdel ? (size_t)m * LDR : 0)) * sizeof(double);
}

// Copy n elements src[si(e)] -> dst[di(e)], e = t0, t0 + stride, ..., with U independent loads
// in flight per thread (all loads of a round before its stores: src and dst may both be
// global, and a load-store loop would otherwise serialise on possible aliasing -- at small n
// these copies sit on the step's critical path).  idx(e, si, di) maps an element.
template <int U, class Idx>
__device__ __forceinline__ void gather_copy(double* dst, const double* src, int n, int t0, int stride, Idx idx) {
#pragma unroll 1
  for (int e0 = t0; e0 < n; e0 += stride * U) {
    double v[U];
    int dd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * stride;
      dd[u] = -1;
      if (e < n) {
        int si, di;
        idx(e, si, di);
        v[u] = __ldcg(src + si);
        dd[u] = di;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dd[u] >= 0) dst[dd[u]] = v[u];
  }
}

// FUSED K1 (NCW <= 3, no Gram): shared memory of its end-of-kernel reduction table
__host__ __device__ constexpr size_t fused_k1_table_bytes(int ncw) {
  return (size_t)NT * (size_t)((3 * (8 * ncw - 2) + 3) | 1) * sizeof(double);
}

__device__ __forceinline__ double cur_scale(const KParams& p, int j) {
  // scale of stored Q column j as seen after this step's K1: rotated columns (QRDelete)
  // were written as true values.
  return p.recycle ? 1.0 : p.st->f[p.ver].scale[j];
}

// ---------------------------------------------------------------------------- heads
// All threads: copy what the head's serial K3 math reads into shared memory in one round
// of parallel loads (columns per warp, no index divisions): reduction slot 0 (R0), the final
// reduction words (RF), R or QRDelete(R) (Rw, K4), and ICWY's T' (Tw: rows 0..k-2 from the
// stored T (start-up) or the post-delete Gram (recycle / delete-only), row k-1 from Alg. 4
// l.1, unit diagonal).
template <int OP>
__device__ void stage_small(const KParams& p, double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = p.k;
  double* Rw = scratch;
  double* Tw = scratch + SCR_TW;
  double* R0 = scratch + SCR_R0;
  double* RF = scratch + SCR_RF;
  const int nw = (OP == OP_K4 || OP == OP_K2_ICWY) ? p.red_words0 : 0;
  gather_copy<4>(R0, p.red, nw, tid, NT, [](int e, int& si, int& di) { si = e; di = e; });
  if (tid < 2) RF[tid] = p.red[(size_t)p.final_slot * LRED + tid];
  const Factors& F = p.st->f[p.ver];
  if constexpr (OP == OP_K4) {
    const double* Rsrc = p.recycle ? F.Rdel : F.R;
    gather_copy<4>(Rw, Rsrc, k * k, tid, NT, [k](int e, int& si, int& di) {
      const int j = e / k, i = e - j * k;
      si = i + j * MMAX;
      di = i + j * LDR;
    });
    // the head's other global operands, in the same round of loads: the sticky breakdown flag
    // (RF[2]), the current scales (spare words of SCR_V) and MGS / CGS-2's R-column words
    // from the later reduction slots (v1)
    double* v1 = scratch + SCR_V;
    double* scl = scratch + SCR_V + 3 * MMAX;
    if (tid == 2) RF[2] = (double)p.st->breakdown;
    for (int j = tid; j < p.m; j += NT) scl[j] = F.scale[j];
    if (p.variant == V_MGS)
      for (int j = 1 + tid; j < k; j += NT) v1[j] = p.red[(size_t)j * LRED];
    else if (p.variant == V_CGS2)
      for (int j = tid; j < k; j += NT) v1[j] = p.red[LRED + j];
  }
  if (p.variant == V_ICWY && (OP == OP_K4 || OP == OP_K2_ICWY)) {
    __syncthreads();   // R0 complete
    const K1Layout L = K1Layout::make(k, true, p.gram != 0);
    const bool del_only = p.flags & F_DELETE_ONLY;
    for (int j = warp; j < k; j += NWARP)
      for (int i = lane; i < k; i += 32) {
        double v;
        if (i == j) v = 1.0;
        else if (j > i) v = 0.0;
        else if (del_only) v = R0[i * (i - 1) / 2 + j];
        else if (i == k - 1) v = R0[L.off_x + j];
        else if (p.recycle && p.icwy_merged == 2) v = F.Tdel[i + j * MMAX];
        else if (p.recycle) v = R0[L.off_gram + i * (i - 1) / 2 + j];
        else v = F.T[i + j * MMAX];
        Tw[i + j * MMAX] = v;
      }
  }
}

struct K4Head {
  int K;          // columns of the updated factor
  double rkk, df2;
};

// Everything Alg. 2 does after the reductions, part 1: the new R column per variant, R_kk,
// Q^T f_i (merged into the existing reductions; A14) and the breakdown test.
// Writes Rw (K x K), c into cvec, H.bd.  Part 2 (k4_gamma): gamma by back-substitution.
__device__ K4Head k4_rcol(const KParams& p, HeadArea& H, double* scratch) {
  const int lane = threadIdx.x & 31;
  double* Rw = scratch;                 // R' (staged by stage_small), leading dimension LDR
  double* Tw = scratch + SCR_TW;        // ICWY T' (staged)
  double* v1 = scratch + SCR_V;         // MMAX words
  double* cvec = v1 + MMAX;             // MMAX
  const double* red0 = scratch + SCR_R0;
  const double* fin = scratch + SCR_RF;
  const int k = p.k;
  K4Head out{};
  if (p.flags & F_DELETE_ONLY) {
    out.K = k;
    return out;
  }
  const K1Layout L = K1Layout::make(k, p.has_x, p.gram != 0);
  const double vv = (k == 0) ? red0[1] : fin[0];
  const double vf = (k == 0) ? red0[3] : fin[1];
  const double rkk = sqrt(vv);
  // new R column (rows 0..k-1 of column k)
  if (p.variant == V_ICWY && k >= 1) {
    for (int j = lane; j < k; j += 32) v1[j] = red0[L.off_df + j];
    __syncwarp();
    k3_forward_unit_lower(Tw, v1, k);
    for (int j = lane; j < k; j += 32) Rw[j + k * LDR] = v1[j];
  } else {
    for (int j = lane; j < k; j += 32) {
      double r;
      if (p.variant == V_MGS) r = (j == 0) ? red0[L.off_df] : v1[j];            // staged red[j*LRED]
      else if (p.variant == V_CGS2) r = red0[L.off_df + j] + v1[j];             // s + z (Alg. 5 l.5)
      else r = red0[L.off_df + j];                                               // DCGS-2 l.1 (A4)
      Rw[j + k * LDR] = r;
    }
  }
  __syncwarp();
  if (p.variant == V_DCGS2 && p.reortho) {  // Alg. 6 l.5 (verbatim R += s, or A3)
    const double rk1 = Rw[(k - 1) + (k - 1) * LDR];
    for (int j = lane; j < k - 1; j += 32) {
      const double s = red0[L.off_x + j];
      Rw[j + (k - 1) * LDR] += p.rscale ? rk1 * s : s;
    }
  }
  if (lane == 0) Rw[k + k * LDR] = rkk;
  for (int i = lane; i < k; i += 32) Rw[k + i * LDR] = 0.0;
  // c = Q^T f_i with the final Q
  for (int j = lane; j < k; j += 32) cvec[j] = red0[L.off_f + j];
  __syncwarp();
  if (p.variant == V_DCGS2 && p.reortho) {
    double acc = 0.0;
    for (int j = lane; j < k - 1; j += 32) acc += red0[L.off_x + j] * cvec[j];
    acc = warp_sum(acc);
    if (lane == 0) cvec[k - 1] -= acc;
  }
  if (lane == 0) cvec[k] = vf / rkk;
  // breakdown (reading A12): R_kk <= eps_a ||Delta f|| (or NaN), or an
  // earlier step of this window broke down (sticky until aa_reset): the step degrades to
  // gamma = 0, x_{i+1} = G(x_i).  Every CTA (and every rank) takes the same decision: rkk
  // and ||Delta f|| are global reduction results, eps_a is the same on every rank.
  const bool bd = !(rkk > p.eps_a * sqrt(red0[1])) || fin[2] != 0.0;   // fin[2]: staged st->breakdown
  if (bd && lane == 0) H.bd = 1;
  __syncwarp();
  out.K = k + 1;
  out.rkk = rkk;
  out.df2 = red0[1];
  return out;
}

// Part 2: gamma = R^{-1} c by back-substitution (Alg. 2 l.9) into H.coef (0 on breakdown),
// and the damping coefficients.  Reads Rw, cvec, H.bd (one warp).
__device__ void k4_gamma(const KParams& p, HeadArea& H, double* scratch, const K4Head& hd) {
  const int lane = threadIdx.x & 31;
  double* Rw = scratch;
  double* cvec = scratch + SCR_V + MMAX;
  double* cvec2 = cvec + MMAX;
  const int k = p.k;
  if (p.flags & F_DELETE_ONLY) return;
  const double rkk = hd.rkk;
  for (int j = lane; j <= k; j += 32) cvec2[j] = cvec[j];
  __syncwarp();
  k3_back_subst<LDR>(Rw, cvec2, H.coef, k + 1);  // gamma -> H.coef[0..k]
  const bool bd = H.bd != 0;
  if (bd) {
    __syncwarp();
    for (int j = lane; j <= k; j += 32) H.coef[j] = 0.0;
  }
  if (p.beta_on && !bd) {
    for (int j = lane; j <= k; j += 32) {
      double fs;
      if (j == k) fs = 1.0 / rkk;
      else if (p.variant == V_DCGS2 && p.reortho && j == k - 1) fs = 1.0;
      else fs = cur_scale(p, j);
      H.coef2[j] = cvec[j] * fs;
    }
    if (lane == 0) H.scal[0] = 1.0 - p.beta;
  }
  __syncwarp();
}

__device__ K4Head k4_head(const KParams& p, HeadArea& H, double* scratch) {
  const K4Head hd = k4_rcol(p, H, scratch);
  k4_gamma(p, H, scratch, hd);
  return hd;
}

// The scalars the last CTA of K4 needs (R_kk and ||Delta f||^2) without the O(m^2) head.
__device__ K4Head k4_scalars_head(const KParams& p) {
  K4Head out{};
  const double* red0 = p.red;
  const int k = p.k;
  const double* fin = p.red + p.final_slot * LRED;
  const double vv = (k == 0) ? red0[1] : fin[0];
  out.rkk = sqrt(vv);
  out.df2 = red0[1];
  out.K = k + 1;
  return out;
}

// CTA 0 of K4 writes factor version ver^1 from the head's results in shared memory and
// precomputes QRDelete of the new R for the next step: the rotations
// (Fo.cs/sn) and R' (Fo.Rdel), so the next recycle step's heads only load them.  Two warps
// in parallel: warp 0 runs the serial Givens chain on a copy Rg of the new R while warp 1
// solves for gamma and writes R, T, the scales and gamma (ICWY SMALL: warp 2 rotates T,
// k4_tdel).
__device__ void k4_tdel(const KParams& p, HeadArea& H, double* scratch, Factors& Fo, int K);

// The commit CTA's store warps (3..7, `nt` threads from `t0`): R_new and T' -> Fo, as soon as
// warp 0 has formed R_new (they are independent of gamma); one flattened pass, so the
// stores of all five warps are in flight together (a one-warp loop of dependent
// iterations cost ~300 cycles per column at small n)
__device__ void k4_store_RT(const KParams& p, double* scratch, int K, int t0, int nt) {
  const double* Rw = scratch;
  const double* Tw = scratch + SCR_TW;
  Factors& Fo = p.st->f[p.ver ^ 1];
  const int mm = p.m;
  const bool icwy = p.variant == V_ICWY;
#pragma unroll 1
  for (int e = t0; e < mm * mm; e += nt) {
    const int jj = e / mm, ii = e - jj * mm;
    Fo.R[ii + jj * MMAX] = (ii < K && jj < K) ? Rw[ii + jj * LDR] : 0.0;
    if (icwy) {
      double v = 0.0;
      if (ii == jj) v = (ii < K) ? 1.0 : 0.0;
      else if (jj < ii && ii < p.k) v = Tw[ii + jj * MMAX];
      Fo.T[ii + jj * MMAX] = v;
    }
  }
}

// warp 1: scales, gamma, K -> Fo
__device__ void k4_write_factors(const KParams& p, HeadArea& H, double* scratch, int K, double rkk) {
  const int lane = threadIdx.x & 31;
  const double* scl = scratch + SCR_V + 3 * MMAX;   // staged F[ver].scale
  Factors& Fo = p.st->f[p.ver ^ 1];
  const int mm = p.m;
  const bool del_only = p.flags & F_DELETE_ONLY;
#pragma unroll 1
  for (int j = lane; j < mm; j += 32) {
    double s = scl[j];
    if (p.recycle && j < p.k) s = 1.0;
    if (!del_only) {
      if (j == p.k) s = 1.0 / rkk;
      if (p.variant == V_DCGS2 && p.reortho && j == p.k - 1) s = 1.0;
    }
    if (j >= K) s = 1.0;
    Fo.scale[j] = s;
    Fo.gamma[j] = del_only ? 0.0 : ((j < K) ? H.coef[j] : 0.0);
  }
  if (lane == 0) Fo.K = K;
  __syncwarp();
}

// One column of the Hessenberg matrix through rotations 0..E-1 (carry form, in place; the
// same operations, in the same order, as k3_givens_delete applies to that column): rows
// 0..E-1 become final, row E holds the carry.
__device__ __forceinline__ void rotate_column(double* col, int E, const double* cs, const double* sn) {
  double carry = col[0];
#pragma unroll 1
  for (int j = 0; j < E; ++j) {
    const double c = cs[j], s = sn[j], h2 = col[j + 1];
    col[j] = __dadd_rn(__dmul_rn(c, carry), __dmul_rn(s, h2));
    carry = __dadd_rn(__dmul_rn(-s, carry), __dmul_rn(c, h2));
  }
  col[E] = carry;
}

// warp 0: QRDelete of the new R (K = k + 1 columns): the rotations into H.cs / H.sn and R' in
// shared memory (the commit CTA's store warps write them out afterwards, k4_delete_store).
// Split form (this step's K1 had a spare CTA, p.k1_pre): rotations 0..k-3 and R' columns
// 0..k-3 depend only on the factor before QRAdd and were computed by K1 (k1_delete_pre);
// here only the last two columns of the Hessenberg matrix (R_new columns k-1, k) go
// through them, and the last two rotations are formed -- bitwise the same result as the
// full chain.  Otherwise: the full Givens chain on the copy Rg (in place).
__device__ __forceinline__ bool k4_split(const KParams& p, int K) {
  return p.k1_pre && !(p.flags & F_DELETE_ONLY) && K - 1 >= 3;
}

__device__ void k4_delete_compute(const KParams& p, HeadArea& H, double* scratch, int K) {
  const int lane = threadIdx.x & 31;
  double* Rw = scratch;
  double* Rg = scratch + SCR_RG;
  const int k = K - 1;
  int* progress = (p.variant == V_ICWY && p.icwy_merged == 2) ? &H.gdone : nullptr;
  if (k4_split(p, K)) {
    const int E = k - 2;
    const SmallState* st = p.st;
    for (int j = lane; j < E; j += 32) {
      H.cs[j] = st->gpre_cs[j];
      H.sn[j] = st->gpre_sn[j];
    }
    __syncwarp();
    if (lane == 0 && progress) {
      __threadfence_block();
      *reinterpret_cast<volatile int*>(progress) = E;
    }
    { constexpr int OP = OP_K4; AA_TLW(12); }
    // columns a = R_new[:, k-1] (rows 0..k; row k is 0) and b = R_new[:, k] (rows 0..k)
    constexpr int LC = MMAX + 1;
    double* ca = Rg;
    double* cb = Rg + LC;
    for (int i = lane; i <= k; i += 32) {
      ca[i] = Rw[i + (k - 1) * LDR];
      cb[i] = Rw[i + k * LDR];
    }
    __syncwarp();
    if (lane < 2) rotate_column(lane == 0 ? ca : cb, E, H.cs, H.sn);
    __syncwarp();
    { constexpr int OP = OP_K4; AA_TLW(13); }
    if (lane == 0) {
      double c, sn_, rho;
      givens_coef(ca[E], ca[E + 1], c, sn_, rho);      // rotation k-2: (H[k-2][k-2], R_new[k-1][k-1])
      ca[E] = rho;
      H.cs[E] = c;
      H.sn[E] = sn_;
      const double b0 = cb[E], b1 = cb[E + 1];
      cb[E] = __dadd_rn(__dmul_rn(c, b0), __dmul_rn(sn_, b1));
      const double carry = __dadd_rn(__dmul_rn(-sn_, b0), __dmul_rn(c, b1));
      if (progress) {
        __threadfence_block();
        *reinterpret_cast<volatile int*>(progress) = E + 1;
      }
      givens_coef(carry, cb[E + 2], c, sn_, rho);      // rotation k-1: (H[k-1][k-1], R_kk)
      cb[E + 1] = rho;
      H.cs[E + 1] = c;
      H.sn[E + 1] = sn_;
      if (progress) {
        __threadfence_block();
        *reinterpret_cast<volatile int*>(progress) = E + 2;
      }
    }
    __syncwarp();
  } else if (K >= 1) {
    k3_givens_delete<LDR>(Rg, K, H.cs, H.sn, progress);
  }
  { constexpr int OP = OP_K4; AA_TLW(14); }
}

// The store warps: R' and the rotations -> Fo.  Part 1 (before the Givens results): in the
// split form, R' columns 0..k-3 straight from K1's precompute.  Part 2 (after): the rest.
__device__ void k4_delete_store_early(const KParams& p, int K, int t0, int nt) {
  if (!k4_split(p, K)) return;
  const int E = K - 3;
  Factors& Fo = p.st->f[p.ver ^ 1];
  gather_copy<4>(Fo.Rdel, p.st->gpre_R, E * E, t0, nt, [E](int e, int& si, int& di) {
    const int j = e / E, i = e - j * E;
    si = i + j * MMAX;
    di = i + j * MMAX;
  });
}

__device__ void k4_delete_store(const KParams& p, HeadArea& H, double* scratch, int K, int t0, int nt) {
  const double* Rg = scratch + SCR_RG;
  Factors& Fo = p.st->f[p.ver ^ 1];
  const int mm = p.m;
  const int k = K - 1;
  const bool split = k4_split(p, K);
  const int E = k - 2;
  constexpr int LC = MMAX + 1;
#pragma unroll 1
  for (int e = t0; e < mm * mm; e += nt) {
    const int j = e / mm, i = e - j * mm;
    double v = 0.0;
    if (split) {
      if (j < E && i < E) continue;   // written by k4_delete_store_early (zeros below the diagonal)
      if (i <= j && j < k) v = (j == E) ? Rg[i] : Rg[LC + i];
    } else if (K >= 1) {
      if (i <= j && j < K - 1) v = Rg[i + j * LDR];
    }
    Fo.Rdel[i + j * MMAX] = v;
  }
  for (int j = t0; j < K - 1; j += nt) {
    Fo.cs[j] = H.cs[j];
    Fo.sn[j] = H.sn[j];
  }
}

// ICWY_DELETE = SMALL (variant, not in the paper, A6b):
// the next QRDelete replaces Q by Q' = Q W (W = the rotations warp 0 is computing, applied
// to columns), so the post-delete Gram is W^T S W with S = T + T^T - I from the P = K-1
// known rows of T (Tw).  Run by warp 1 of CTA 0 concurrently with warp 0's head and
// QRDelete: S is built in its own shared region (leading dimension MMAX+1 against bank
// conflicts) and rotated two-sided as each rotation is published (H.gdone); rotations
// 0..P-2 fix every entry with both indices <= P-2, which are the rows the next step reads.
__device__ void k4_tdel(const KParams& p, HeadArea& H, double* scratch, Factors& Fo, int K) {
  constexpr int LD = MMAX + 1;
  const int lane = threadIdx.x & 31;
  const double* Tw = scratch + SCR_TW;
  double* S = scratch + scr_s(p.m);   // own region (warp 0 rotates Rg meanwhile)
  const int P = K - 1;
  for (int j = 0; j < P; ++j)
    for (int i = j + lane; i < P; i += 32) {
      const double v = (i == j) ? 1.0 : Tw[i + j * MMAX];
      S[i + j * LD] = v;
      S[j + i * LD] = v;
    }
  __syncwarp();
  k3_rotate_sym<LD>(S, P, H.cs, H.sn, &H.gdone);
  const int mm = p.m;
#pragma unroll 1
  for (int j = 0; j < mm; ++j)
    for (int i = lane; i < mm; i += 32)
      Fo.Tdel[i + j * MMAX] = (i == j) ? 1.0 : ((j < i && i < P - 1) ? S[i + j * LD] : 0.0);
  __syncwarp();
}

// K1's spare CTA (small n): the early part of the NEXT QRDelete.  The factor before this
// step's QRAdd is R_cur (k x k: QRDelete(R) at recycle, R at start-up); the next QRDelete
// re-triangularises R_new[:, 1:], whose columns 1..k-2 are R_cur's, so its rotations
// 0..k-3 and R' columns 0..k-3 are those of QRDelete of R_cur's leading (k-1) x (k-1)
// block: computed here (one warp, scratch = this CTA's unused stage memory), finished by K4.
__device__ void k1_delete_pre(const KParams& p, HeadArea& H, double* scratch) {
  // warps 1..7 of the spare CTA (224 threads; warp 0 runs the op head): stage R_cur together,
  // warp 1 runs the serial Givens chain, all seven write the results (one warp's dependent
  // store loop costs ~300 cycles per column at small n)
  const int t = threadIdx.x - 32, nt = NT - 32;
  const int warp = threadIdx.x >> 5;
  const int k = p.k;
  const int mold = k - 1;
  const Factors& F = p.st->f[p.ver];
  const double* Rsrc = p.recycle ? F.Rdel : F.R;
  double* Rs = scratch;
  gather_copy<4>(Rs, Rsrc, mold * mold, t, nt, [mold](int e, int& si, int& di) {
    const int j = e / mold, i = e - j * mold;
    si = i + j * MMAX;
    di = i + j * LDR;
  });
  asm volatile("bar.sync 3, 224;" ::: "memory");
  if (warp == 1) {
    { constexpr int OP = OP_K1; AA_TLW(12); }
    k3_givens_delete<LDR>(Rs, mold, H.cs, H.sn, nullptr);
    { constexpr int OP = OP_K1; AA_TLW(13); }
  }
  asm volatile("bar.sync 3, 224;" ::: "memory");
  SmallState* st = p.st;
  const int E = mold - 1;
#pragma unroll 1
  for (int e = t; e < E * E; e += nt) {
    const int j = e / E, i = e - j * E;
    st->gpre_R[i + j * MMAX] = (i <= j) ? Rs[i + j * LDR] : 0.0;
  }
  for (int j = t; j < E; j += nt) {
    st->gpre_cs[j] = H.cs[j];
    st->gpre_sn[j] = H.sn[j];
  }
  if (warp == 1) { constexpr int OP = OP_K1; AA_TLW(14); }
}

template <int OP>
__device__ void op_head(const KParams& p, HeadArea& H, double* scratch) {
  const int lane = threadIdx.x & 31;
  const double* red0 = p.red;
  const int k = p.k;
  if constexpr (OP == OP_K1) {
    const Factors& F = p.st->f[p.ver];
    // one round of independent loads: scale[j], and at recycle the Givens coefficients of
    // QRDelete(R) precomputed by the previous K4 with the next column's scale folded in
    for (int j = lane; j < p.c_in; j += 32) {
      const double scj = F.scale[j];
      H.sc[j] = scj;
      if (p.recycle && j < p.c_in - 1) {
        const double c = F.cs[j], s = F.sn[j], scn = F.scale[j + 1];
        H.rot[2 * j] = make_double2(c, s * scn);
        H.rot[2 * j + 1] = make_double2(-s, c * scn);
      }
    }
    if (lane == 0) {
      if (p.flags & F_DELETE_ONLY) {
        H.na = 0;
        H.nr = 0;
      } else {
        const int vb = p.vb;
        // stage slot of Delta f (phase A): Q column k at recycle (the slot of the dropped
        // column's input, so the rotated block and Delta f leave in ONE tensor store), the
        // consumed G(x_{i-1}) slot at start-up, vb + 1 for a caller-supplied column
        const int dfs = (p.flags & F_EXT_DF) ? vb + 1 : (p.recycle ? k : vb + 3);
        H.na = k + 2;
        for (int a = 0; a < k; ++a) H.lcol[a] = a;
        H.lcol[k] = vb;          // f_i
        H.lcol[k + 1] = dfs;     // Delta f
        H.nr = 3;
        H.rcol[0] = dfs;
        H.rcol[1] = vb;
        H.rcol[2] = (k >= 1) ? k - 1 : vb;
      }
    }
  } else if constexpr (OP == OP_K2_ICWY) {
    double* Tw = scratch + SCR_TW;                // T' (staged)
    double* v1 = scratch + SCR_V;
    const double* r0s = scratch + SCR_R0;
    const K1Layout L = K1Layout::make(k, p.has_x, p.gram != 0);
    for (int j = lane; j < k; j += 32) v1[j] = r0s[L.off_df + j];
    __syncwarp();
    k3_forward_unit_lower(Tw, v1, k);   // Alg. 4 l.4
    for (int j = lane; j < k; j += 32) H.coef[j] = v1[j] * cur_scale(p, j);
  } else if constexpr (OP == OP_K2_DCGS2) {
    const K1Layout L = K1Layout::make(k, p.has_x, false);
    for (int j = lane; j < k; j += 32) {
      const double sc = cur_scale(p, j);
      H.sc[j] = sc;
      H.coef[j] = (j < k - 1) ? red0[L.off_df + j] * sc : red0[L.off_df + j];
      if (p.reortho && j < k - 1) H.coef2[j] = red0[L.off_x + j] * sc;
    }
  } else if constexpr (OP == OP_K2A_CGS2) {
    const K1Layout L = K1Layout::make(k, false, false);
    for (int j = lane; j < k; j += 32) {
      const double sc = cur_scale(p, j);
      H.sc[j] = sc;
      H.coef[j] = red0[L.off_df + j] * sc;
    }
    if (lane == 0) {
      H.na = k;
      for (int a = 0; a < k; ++a) H.lcol[a] = a;
      H.nr = 1;
      H.rcol[0] = k;
    }
  } else if constexpr (OP == OP_K2B_CGS2) {
    for (int j = lane; j < k; j += 32) H.coef[j] = p.red[LRED + j] * cur_scale(p, j);
  } else if constexpr (OP == OP_K2_MGS) {
    if (lane == 0) {
      const int j = p.mgs_j;
      const K1Layout L = K1Layout::make(k, false, false);
      const double r = (j == 1) ? red0[L.off_df] : p.red[(j - 1) * LRED];
      H.scal[0] = r * cur_scale(p, j - 1);
      H.scal[1] = (j < k) ? cur_scale(p, j) : 1.0;
    }
  } else if constexpr (OP == OP_K4) {
    k4_head(p, H, scratch);
  } else if constexpr (OP == OP_GRAM) {
    for (int j = lane; j < p.c_in; j += 32) H.sc[j] = p.st->f[p.ver].scale[j];
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------- producer
__device__ __forceinline__ uint32_t vec_bytes(const KParams& p, int i, int rows) {
  return ((p.exact_vec >> i) & 1u) ? (((uint32_t)rows * 8u) & ~15u) : (uint32_t)align_up((size_t)rows * 8u, 16);
}

// Copies of one tile: blocks 0..nblk-1 (one 2-D tensor copy each, full box incl. the
// zero-filled rows past n), then vectors; lane 0 of warp w issues copies w, w+NWARP, ...
__device__ void issue_tile_part(const KParams& p, double* stage, uint64_t* bar, long long row0, int rows,
                                int warp) {
  const int TR = p.tr;
  const int ncp = p.nblk + p.nvec;
  uint32_t total = 0;
  for (int c = warp; c < ncp; c += NWARP)
    total += (c < p.nblk) ? (uint32_t)TR * p.blk_ncols[c] * 8u : vec_bytes(p, c - p.nblk, rows);
  mbar_arrive_expect_tx(bar, total);
  for (int c = warp; c < ncp; c += NWARP) {
    if (c < p.nblk) {
      int col0 = 0;
      for (int b = 0; b < c; ++b) col0 += p.blk_ncols[b];
      if (p.tm3d)
        tma_3d_g2s(stage + (size_t)col0 * TR, &p.tm[c], (int)(row0 >> 8), p.blk_gcol[c], bar);
      else
        tma_2d_g2s(stage + (size_t)col0 * TR, &p.tm[c], (int)row0, p.blk_gcol[c], bar);
    } else {
      const int i = c - p.nblk;
      const uint32_t b = vec_bytes(p, i, rows);
      if (b) bulk_g2s(stage + (size_t)(p.vb + i) * TR, p.vec[i] + row0, b, bar);
    }
  }
}

// value of vector i at tile row r (falls back to a plain load for the odd last row of a
// caller buffer that the 16-byte-granular bulk copy could not cover)
__device__ __forceinline__ double ldV(const KParams& p, const double* S, int i, int r, int rows,
                                      long long grow) {
  if ((rows & 1) && r == rows - 1 && ((p.exact_vec >> i) & 1u)) return p.vec[i][grow];
  return S[(size_t)(p.vb + i) * p.tr + r];
}

__device__ __forceinline__ int gram_block_I(int blk) {
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= blk) ++I;
  return I;
}


// Sum the per-warp DMMA Gram accumulators over the 8 warps through shared memory (the
// stage ring is idle after the tile loop), in chunks of blocks, and write this CTA's
// partial words.  mode 0: strict lower, rows < kg-1 -> off_gram, row kg-1 -> off_x (ICWY
// after QRDelete + Alg. 4 l.1); 1: strict lower packed (stand-alone delete); 2: lower incl.
// diagonal packed (loss of orthogonality); 3: mode 0 over the kg-2 columns of Q, then row
// kg-2 (Delta f) -> off_df and df.df, row kg-1 (f_i) -> off_f, df.f and f.f (K1 words 1, 3, 0).
template <int NB8>
__device__ void gram_epilogue(const KParams& p, const double* gc0, const double* gc1, double* buf,
                              double* mypart, int kg, int mode, int off_x, int off_gram, int off_df,
                              int off_f) {
  constexpr int GB = NB8 * (NB8 + 1) / 2;
  constexpr int CH = 8;  // blocks per chunk: 8 warps x 8 blocks x 64 doubles = 32 KB
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b0 = 0; b0 < GB; b0 += CH) {
    __syncthreads();
#pragma unroll
    for (int g = 0; g < GB; ++g)
      if (g >= b0 && g < b0 + CH) {
        buf[((warp * CH) + (g - b0)) * 64 + 2 * lane] = gc0[g];
        buf[((warp * CH) + (g - b0)) * 64 + 2 * lane + 1] = gc1[g];
      }
    __syncthreads();
    const int nb = min(CH, GB - b0);
    for (int e = tid; e < nb * 64; e += NT) {
      const int gl = e / 64, w = e % 64;
      double s = 0.0;
      for (int ww = 0; ww < NWARP; ++ww) s += buf[(ww * CH + gl) * 64 + w];
      const int g = b0 + gl;
      const int I = gram_block_I(g), J = g - I * (I + 1) / 2;
      const int ln = w >> 1, ee = w & 1;
      const int i = 8 * I + (ln >> 2), j = 8 * J + 2 * (ln & 3) + ee;
      if (i >= kg) continue;
      if (mode == 3) {
        const int kq = kg - 2;
        if (j > i) continue;
        int wd = -1;
        if (i < kq) {
          if (j < i) wd = (i == kq - 1) ? off_x + j : off_gram + i * (i - 1) / 2 + j;
        } else if (i == kq) {
          wd = (j < kq) ? off_df + j : 1;
        } else {
          wd = (j < kq) ? off_f + j : (j == kq ? 3 : 0);
        }
        if (wd >= 0) mypart[wd] = s;
      } else if (mode == 2) {
        if (j <= i) mypart[i * (i + 1) / 2 + j] = s;
      } else if (j < i) {
        int wd;
        if (mode == 1) wd = i * (i - 1) / 2 + j;
        else if (i == kg - 1) wd = off_x + j;
        else wd = off_gram + i * (i - 1) / 2 + j;
        mypart[wd] = s;
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------- deterministic sums
// Power-of-two-aligned pairwise tree over values v(0..G-1): node (l, i) = sum of leaves
// [i 2^l, (i+1) 2^l), a node with one missing child equals the other.  The tree depends only
// on the leaf indices, so a rank's sum over an aligned power-of-two range of chunks is a node
// of the global tree (bitwise identical across rank counts).
// One warp: lane l builds the subtree of its aligned block of B leaves (binary counter),
// then 5 shuffle levels pair aligned lane blocks.  Result valid in lane 0.
template <class Load>
__device__ double aligned_tree_sum_warp(int G, Load load) {
  const int lane = threadIdx.x & 31;
  int B = 1;
  while (B * 32 < G) B <<= 1;
  double stk[16];
  int sz[16];
  int top = 0;
  const int base = lane * B;
  for (int i = 0; i < B && base + i < G; ++i) {
    double v = load(base + i);
    int s = 1;
    while (top > 0 && sz[top - 1] == s) {   // merge equal-size (aligned sibling) subtrees
      v = stk[top - 1] + v;
      s <<= 1;
      --top;
    }
    stk[top] = v;
    sz[top] = s;
    ++top;
  }
  bool has = top > 0;
  double acc = 0.0;
  if (has) {
    acc = stk[top - 1];
    for (int e = top - 2; e >= 0; --e) acc = stk[e] + acc;   // missing right parts: left + (right)
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double o = __shfl_down_sync(0xffffffffu, acc, d);
    const bool oh = __shfl_down_sync(0xffffffffu, has ? 1 : 0, d) != 0;
    if ((lane & (2 * d - 1)) == 0) {
      if (has && oh) acc = acc + o;
      else if (oh) acc = o;
      has = has || oh;
    }
  }
  return acc;
}

// the same tree over R <= 8 values held by one thread (the ranks of a fused exchange)
__device__ __forceinline__ double aligned_tree_sum_small(const double* v, int R) {
  double t[MAX_RANKS];
  int n = R;
  for (int q = 0; q < R; ++q) t[q] = v[q];
  while (n > 1) {
    const int h = (n + 1) / 2;
    for (int q = 0; q < h; ++q) t[q] = (2 * q + 1 < n) ? t[2 * q] + t[2 * q + 1] : t[2 * q];
    n = h;
  }
  return t[0];
}

// ---------------------------------------------------------------------------- fused allreduce
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// relaxed system-scope 8-byte accesses: an aligned 8-byte store is single-copy atomic, so
// a word that carries its own sequence tag needs no fence and no separate flag
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* ptr, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(ptr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* ptr) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ptr) : "memory");
  return v;
}

// One-shot allreduce of v[0..cnt) among the node's ranks, run by the LAST CTA of a kernel
// on every rank ("fused local + global reduction"), over
// NVLink peer memory with a low-latency protocol: every fp64 word travels as two 8-byte
// stores, each carrying 32 data bits and the exchange's 32-bit sequence tag, into every
// rank's mailbox [seq parity][source rank][word][half]; a reader spins on the words
// themselves until both halves carry the tag -- no fence, no flag round trip.  The p
// vectors are summed in rank order, the same order on every rank, so all ranks obtain
// bitwise identical sums.  A slot of parity s&1 is rewritten only by exchange s+2, which
// no rank can start before every rank has read exchange s (it needs all of s+1 first).
// The wait is time-bounded (10 s): on timeout a sticky flag is set instead of hanging.
__device__ void fused_exchange(const KParams& p, double* v, int cnt, unsigned long long seq) {
  const int tid = threadIdx.x;
  const int R = p.nranks;
  const int par = (int)(seq & 1ull);
  // 32-bit tag in 1 .. 2^32-1 (never 0, the value of a mailbox word never written)
  const unsigned long long tag = (((seq - 1ull) % 0xffffffffull) + 1ull) << 32;
  for (int i = tid; i < cnt * R; i += NT) {
    const int q = i / cnt, w = i - q * cnt;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v[w]);
    unsigned long long* dst =
        reinterpret_cast<unsigned long long*>(p.pmbox[q]) + ((size_t)(par * R + p.rank) * LRED + w) * 2;
    st_relaxed_sys_u64(dst, tag | (bits & 0xffffffffull));
    st_relaxed_sys_u64(dst + 1, tag | (bits >> 32));
  }
  __syncthreads();   // every v[w] has been read before it is overwritten below
  const unsigned long long* lm = reinterpret_cast<const unsigned long long*>(p.lmbox);
  bool timed_out = false;
  for (int w = tid; w < cnt; w += NT) {
    double s = 0.0;
    double vals[MAX_RANKS];
    for (int q = 0; q < R; ++q) {
      const unsigned long long* src = lm + ((size_t)(par * R + q) * LRED + w) * 2;
      unsigned long long lo, hi;
      unsigned int spins = 0;
      const unsigned long long t0 = global_ns();
      while (true) {
        lo = ld_relaxed_sys_u64(src);
        hi = ld_relaxed_sys_u64(src + 1);
        if ((lo & 0xffffffff00000000ull) == tag && (hi & 0xffffffff00000000ull) == tag) break;
        if ((++spins & 1023u) == 0 && global_ns() - t0 > 10000000000ull) {
          timed_out = true;
          break;
        }
      }
      const double vq = __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
      vals[q] = vq;
      s += vq;   // rank order
    }
    v[w] = (p.det_tpc > 0) ? aligned_tree_sum_small(vals, R) : s;
  }
  if (timed_out) p.st->xchg_timeout = 1;
  __syncthreads();
}

// ---------------------------------------------------------------------------- kernel
// OP: the op; NCW: phase-B columns per warp (0 = no block multi-dot); NB8: 8-column
// groups of the DMMA Gram (0 = no Gram).
template <int OP, int NCW, int NB8>
__global__ void __launch_bounds__(NT, 1) aa_stream_kernel(const __grid_constant__ KParams p) {
  constexpr bool GRAM = NB8 > 0;
  // K1 with the Gram and no block multi-dot (NCW = 0): Delta f and f_i are Gram columns k and
  // k+1, so the one DMMA pass gives T's row, the post-delete Gram, Q^T Delta f, Q^T f_i and the
  // three norms
  constexpr bool GX = (OP == OP_K1) && GRAM && NCW == 0;
  // K1 without a Gram and with 7..22 columns (NCW 2..3; with fewer the split form measured
  // faster -- two CTAs per SM hide it): the block multi-dot is fused into
  // the row-wise pass -- each thread keeps its rows' products with Delta f, f_i and q_{k-1} in
  // registers (per-thread partial sums, reduced across the CTA once at the end), so the rotated
  // columns are never written back to the stage, re-read, or separated from phase A by a
  // barrier
  constexpr bool FUSED = (OP == OP_K1) && !GRAM && NCW >= 2 && NCW <= 3;
  constexpr int KMAX = FUSED ? 8 * NCW - 2 : 1;
  // per-column guards on the fused dots: measured A/B (profiles/r02/k1_fused_variants_ab.txt):
  // guarded is 6 % faster at NCW = 3 (m = 20), unguarded (zeros past k, no selects) 3 %
  // faster at NCW = 2 (m = 10)
  constexpr bool GUARD = (NCW == 3);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  HeadArea& H = *reinterpret_cast<HeadArea*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + head_bytes());
  double* stage0 = reinterpret_cast<double*>(smem_raw + head_bytes() + bar_bytes());
  double* scratch = stage0 + p.scr_off;   // aliases the stage ring unless the host separated it

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // programmatic dependent launch: this grid may be resident before its predecessor on the
  // stream has finished; wait for it (and its memory) before touching anything it wrote,
  // then let the next kernel start launching (it waits the same way)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long n = p.n;          // rows [rbeg, n) are this launch's
  const long long rbeg = p.rbeg;
  const int TR = p.tr, NS = p.stages;
  const size_t stage_words = align_up((size_t)p.nin * TR, 16);
  const long long ntiles = (n > rbeg) ? (n - rbeg + TR - 1) / TR : 0;
  const int k = p.k;
  const int vb = p.vb;

  K4Head hd{};
  // K4's run-time scalars come from the previous kernels' reductions and the previous step's
  // state: thread 0 of every CTA loads them now, so the last CTA's tail has no dependent
  // global loads (small n: the tail is on the step's critical path)
  K4Head tail_hd{};
  double tail_f2 = 0.0, tail_rmin = 0.0;
  if (OP == OP_K4 && tid == 0 && p.chunk_last && !(p.flags & F_DELETE_ONLY)) {
    tail_hd = k4_scalars_head(p);
    tail_f2 = p.red[0];
    tail_rmin = p.st->rratio_min;
  }
  if (blockIdx.x == 0) AA_TL(0);
  // tile CTAs: all, or (K4 / K1 pre_cta) all but CTA 0, which only does the factor precompute
  const int pre = (OP == OP_K4 || OP == OP_K1) ? p.pre_cta : 0;
  long long tb = (long long)blockIdx.x - pre, tg = (long long)gridDim.x - pre;
  long long my_count = (tb >= 0 && ntiles > tb) ? (ntiles - 1 - tb) / tg + 1 : 0;
  if (p.det_tpc > 0) {   // deterministic mode: CTA b streams chunk b's tiles in order
    tb = (long long)blockIdx.x * p.det_tpc;
    tg = 1;
    my_count = (ntiles > tb) ? min((long long)p.det_tpc, ntiles - tb) : 0;
  }
  // the first tiles' TMA loads go out BEFORE the heads when the heads do not use the stage
  // memory (their latency then overlaps the serial K3 work; at small n the head is a large
  // share of a kernel): every op except K4 / K2 ICWY, and those two when the host gave their
  // scratch its own region (p.scr_off > 0)
  const bool early_tma = p.early_tma && (!(OP == OP_K4 || OP == OP_K2_ICWY) || p.scr_off > 0);
  if (early_tma) {
    if (tid == 0) {
      for (int s = 0; s < NS; ++s) mbar_init(&bars[s], NWARP);
      fence_mbar_init();
    }
    __syncthreads();
    if (lane == 0) {
      fence_proxy_async();
      for (int s = 0; s < NS && s < my_count; ++s) {
        const long long t = tb + (long long)s * tg;
        const long long r0 = rbeg + t * TR;
        issue_tile_part(p, stage0 + s * stage_words, &bars[s], r0, (int)min((long long)TR, n - r0), warp);
      }
    }
  }
  if constexpr (OP == OP_K4 || OP == OP_K2_ICWY) {
    if (OP == OP_K4 && tid == 0) {
      H.gdone = 0;
      H.bd = 0;
    }
    stage_small<OP>(p, scratch);
    __syncthreads();
  }
  if (blockIdx.x == 0) AA_TL(1);
  if constexpr (OP == OP_K4) {
    if (!(blockIdx.x == 0 && p.chunk_first)) {
      if (warp == 0) hd = k4_head(p, H, scratch);
    } else if (warp == 0) {
      // the commit CTA: warp 0 forms the new R column, then runs the serial Givens chain of the
      // next QRDelete; warp 1 (released by named barrier 1) solves gamma and writes the scales;
      // warps 3..7 write R and T (barrier 1) and R' and the rotations (barrier 2) in parallel
      hd = k4_rcol(p, H, scratch);
      if (!k4_split(p, hd.K)) {   // full chain: on a copy of R_new
        double* Rw = scratch;
        double* Rg = scratch + SCR_RG;
#pragma unroll 1
        for (int j = 0; j < hd.K; ++j)
          for (int i = lane; i <= j; i += 32) Rg[i + j * LDR] = Rw[i + j * LDR];
      }
      if (lane == 0) {
        H.K4_K = hd.K;
        H.K4_rkk = hd.rkk;
      }
      __syncwarp();
      asm volatile("bar.arrive 1, 224;" ::: "memory");
      AA_TLW(8);
      k4_delete_compute(p, H, scratch, hd.K);
      asm volatile("bar.arrive 2, 192;" ::: "memory");
      AA_TLW(9);
    } else if (warp == 1) {
      asm volatile("bar.sync 1, 224;" ::: "memory");
      K4Head h1{};
      h1.K = H.K4_K;
      h1.rkk = H.K4_rkk;
      k4_gamma(p, H, scratch, h1);
      AA_TLW(10);
      k4_write_factors(p, H, scratch, h1.K, h1.rkk);
      AA_TLW(11);
    } else if (warp >= 3) {
      asm volatile("bar.sync 1, 224;" ::: "memory");
      const int K = H.K4_K;
      const int t3 = tid - 96;
      k4_store_RT(p, scratch, K, t3, NT - 96);
      k4_delete_store_early(p, K, t3, NT - 96);
      if (warp == 3) { AA_TLW(15); }
      asm volatile("bar.sync 2, 192;" ::: "memory");
      k4_delete_store(p, H, scratch, K, t3, NT - 96);
      if (t3 == 0) p.st->f[p.ver ^ 1].has_del = 1;
    } else if (warp == 2 && p.variant == V_ICWY && p.icwy_merged == 2) {
      // ICWY SMALL: the post-delete T, rotated as warp 0 publishes the Givens rotations
      const int K = (p.flags & F_DELETE_ONLY) ? p.k : p.k + 1;
      if (K >= 1) k4_tdel(p, H, scratch, p.st->f[p.ver ^ 1], K);
    }
  } else {
    if (warp == 0) op_head<OP>(p, H, scratch);
    if constexpr (OP == OP_K1) {
      if (p.pre_cta && blockIdx.x == 0 && warp >= 1) k1_delete_pre(p, H, scratch);
    }
  }
  if (!early_tma && tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], NWARP);
    fence_mbar_init();
  }
  __syncthreads();   // the heads' shared-memory results are complete
  if (blockIdx.x == 0) AA_TL(2);
  if (!early_tma && lane == 0) {
    fence_proxy_async();
    for (int s = 0; s < NS && s < my_count; ++s) {
      const long long t = tb + (long long)s * tg;
      const long long r0 = rbeg + t * TR;
      issue_tile_part(p, stage0 + s * stage_words, &bars[s], r0, (int)min((long long)TR, n - r0), warp);
    }
  }

  // K1: CTA 0 carries the lagged ||x_i - x_{i-1}||^2 partial (A15) in its partials; load it now
  double dx2_pref = 0.0;
  if (OP == OP_K1 && tid == 0 && blockIdx.x == 0 && p.chunk_first && !(p.flags & (F_EXT_DF | F_DELETE_ONLY)))
    dx2_pref = p.st->dx2_local;
  // phase-A accumulators (row-wise dots / norms)
  double a0 = 0.0, a1 = 0.0;
  // FUSED K1: per-thread partial dots q_j . Delta f, q_j . f_i, q_j . q_{k-1}; f.f, df.df, df.f
  double fa0[KMAX], fa1[KMAX], fa2[KMAX];
  double fs_ff = 0.0, fs_dd = 0.0, fs_df = 0.0;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) fa0[j] = fa1[j] = fa2[j] = 0.0;
  const bool xrhs = p.has_x && p.gram == 0;
  // phase-B accumulators: this warp's NCW columns x NRB right-hand sides
  constexpr int NRB = (OP == OP_K1) ? 3 : 1;
  constexpr int NCWx = NCW > 0 ? NCW : 1;
  double acc[NCWx][NRB];
  int coff[NCWx], roff[NRB];
#pragma unroll
  for (int c = 0; c < NCWx; ++c) {
#pragma unroll
    for (int b = 0; b < NRB; ++b) acc[c][b] = 0.0;
    const int a = warp + c * NWARP;
    coff[c] = (NCW > 0 && a < H.na) ? H.lcol[a] * TR : 0;
  }
#pragma unroll
  for (int b = 0; b < NRB; ++b) roff[b] = (NCW > 0 && b < H.nr) ? H.rcol[b] * TR : 0;
  // Gram accumulators (fp64 DMMA 8x8 blocks): every warp holds ALL NB8*(NB8+1)/2 lower
  // blocks for its own k-steps (rows r0 = 4*(warp + 8*i) of each tile), so a k-step issues
  // GB independent DMMAs sharing NB8 fragment loads; warps are summed at the end.
  constexpr int GB = GRAM ? NB8 * (NB8 + 1) / 2 : 1;
  double gc0[GB], gc1[GB];
  const bool del_only = p.flags & F_DELETE_ONLY;
  const int kg = (OP == OP_GRAM) ? p.c_in : (del_only ? p.c_in - 1 : k);
  const bool do_gram = GRAM && p.gram != 0 && (OP == OP_GRAM ? kg >= 1 : kg >= 2);
  const int kgx = GX ? k + 2 : kg;   // Gram columns
  int gfrag[NB8 > 0 ? NB8 : 1];
  {
    const int g_r = lane >> 2, g_c = lane & 3;
#pragma unroll
    for (int g = 0; g < GB; ++g) gc0[g] = gc1[g] = 0.0;
#pragma unroll
    for (int X = 0; X < (NB8 > 0 ? NB8 : 1); ++X) {
      const int col = 8 * X + g_r;
      int slot = (col < kg) ? col : -1;   // columns past kgx contribute 0
      if (GX && col == k) slot = H.lcol[k + 1];   // Delta f
      if (GX && col == k + 1) slot = vb;          // f_i
      gfrag[X] = (slot >= 0) ? slot * TR + g_c : -1;
    }
  }

  for (long long it = 0; it < my_count; ++it) {
    const int sidx = (int)(it % NS);
    const uint32_t par = (uint32_t)((it / NS) & 1);
    const long long tile = tb + it * tg;
    const long long row0 = rbeg + tile * TR;
    const int rows = (int)min((long long)TR, n - row0);
    double* S = stage0 + sidx * stage_words;
    mbar_wait(&bars[sidx], par);
    if (blockIdx.x == 0 && it == 0) AA_TL(3);
    // K1 full tiles (AA_K1 TMA-store mode): outputs are written back into the stage and leave
    // with TMA stores after phase A (the tail tile of a launch keeps per-thread stores, so
    // rows outside this launch's range are never written)
    const bool tma_tile = (OP == OP_K1) && !FUSED && p.k1_tmastore && !del_only && !(p.flags & F_EXT_DF) &&
                          rows == TR;
    const int dfs = (OP == OP_K1) ? ((p.flags & F_EXT_DF) ? vb + 1 : (p.recycle ? k : vb + 3)) : 0;
    (void)dfs;

    // ------------------------------------------------------------ phase A (row-wise)
    for (int r = tid; r < TR; r += NT) {
      const long long grow = row0 + r;
      if constexpr (FUSED) {
        if (!del_only) {
          if (r < rows) {
            double f, df;
            if (p.flags & F_EXT_DF) {
              df = ldV(p, S, 0, r, rows, grow);
              f = df;
            } else {
              // Alg. 1 l.3-5: f_i = G(x_i) - x_i, Delta f = f_i - f_{i-1}, Delta g = G(x_i) - G(x_{i-1})
              const double x = ldV(p, S, 0, r, rows, grow);
              const double g = ldV(p, S, 1, r, rows, grow);
              const double fpv = S[(size_t)(vb + 2) * TR + r];
              const double gpv = S[(size_t)(vb + 3) * TR + r];
              f = g - x;
              df = f - fpv;
              p.fp[grow] = f;
              p.gp[grow] = g;
              p.dg_out[grow] = g - gpv;
            }
            double q[KMAX];
            double qlast = 0.0;   // q_{k-1} of this row (no dynamic index into q: it stays in registers)
            if (p.recycle) {
              // QRDelete on Q: the streaming carry form of the Givens rotations (P:111,
              // P:135-136); out_j = column j of Q' for this row, the last carry is dropped
              double carry = S[r] * H.sc[0];
              // running pointers (one add per column instead of a 64-bit index computation)
              double* qg = p.Q + grow;
              const double* sp = S + TR + r;
              const long long ld = p.ld;
#pragma unroll
              for (int j = 0; j < KMAX; ++j) {
                if (!GUARD) q[j] = 0.0;   // unguarded dots below: columns past k contribute exact zeros
                if (j < k) {
                  const double qn = *sp;
                  const double2 a = H.rot[2 * j], b = H.rot[2 * j + 1];
                  const double out = fma(a.x, carry, a.y * qn);
                  carry = fma(b.x, carry, b.y * qn);
                  q[j] = out;
                  qlast = out;
                  *qg = out;
                  qg += ld;
                  sp += TR;
                }
              }
            } else {
#pragma unroll
              for (int j = 0; j < KMAX; ++j) q[j] = (j < k) ? S[(size_t)j * TR + r] * H.sc[j] : 0.0;
              if (k >= 1) qlast = S[(size_t)(k - 1) * TR + r] * H.sc[k - 1];
            }
            p.Q[(size_t)k * p.ld + grow] = df;   // unnormalised new column (lazy scale)
            // Alg. 3-6 pass 1 (Q^T Delta f, Q^T f_i and Q_{0:k-2}^T q_{k-1}) and the norms (the
            // words j >= k, j >= k-1 for the third, are never published)
            if constexpr (GUARD) {
#pragma unroll
              for (int j = 0; j < KMAX; ++j)
                if (j < k) {
                  fa0[j] = fma(q[j], df, fa0[j]);
                  fa1[j] = fma(q[j], f, fa1[j]);
                }
              if (xrhs) {
#pragma unroll
                for (int j = 0; j < KMAX; ++j)
                  if (j < k - 1) fa2[j] = fma(q[j], qlast, fa2[j]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < KMAX; ++j) {
                fa0[j] = fma(q[j], df, fa0[j]);
                fa1[j] = fma(q[j], f, fa1[j]);
              }
              if (xrhs) {
#pragma unroll
                for (int j = 0; j < KMAX; ++j) fa2[j] = fma(q[j], qlast, fa2[j]);
              }
            }
            fs_ff = fma(f, f, fs_ff);
            fs_dd = fma(df, df, fs_dd);
            fs_df = fma(df, f, fs_df);
          }
          continue;
        }
      }
      if constexpr (OP == OP_K1) {
        const int ncols = del_only ? p.c_in : (p.recycle ? p.c_in : k);
        if (r < rows) {
          double f = 0.0, df = 0.0;
          if (!del_only) {
            if (p.flags & F_EXT_DF) {
              df = ldV(p, S, 0, r, rows, grow);
              f = df;
            } else {
              // Alg. 1 l.3-5: f_i = G(x_i) - x_i, Delta f = f_i - f_{i-1}, Delta g = G(x_i) - G(x_{i-1})
              const double x = ldV(p, S, 0, r, rows, grow);
              const double g = ldV(p, S, 1, r, rows, grow);
              const double fpv = S[(size_t)(vb + 2) * TR + r];
              const double gpv = S[(size_t)(vb + 3) * TR + r];
              f = g - x;
              df = f - fpv;
              if (tma_tile) {
                // outputs stay in the stage for the tile's TMA stores: f -> slot vb (x),
                // G(x_i) stays in slot vb + 1, Delta g -> slot vb + 2 (f_{i-1})
                S[(size_t)(vb + 2) * TR + r] = g - gpv;
              } else {
                p.fp[grow] = f;
                p.gp[grow] = g;
                p.dg_out[grow] = g - gpv;
              }
            }
          }
          if (p.recycle) {
            // QRDelete on Q: streaming carry form of the m-1 Givens rotations of adjacent
            // column pairs; the last carry is the dropped column.
            double carry = S[r] * H.sc[0];
            double* Qg = p.Q + grow;
            const long long ld = p.ld;
            if (tma_tile) {
#pragma unroll 4
              for (int j = 0; j < p.c_in - 1; ++j) {
                const double qn = S[(size_t)(j + 1) * TR + r];   // stored (lazily scaled) column
                const double2 a = H.rot[2 * j], b = H.rot[2 * j + 1];
                const double out = fma(a.x, carry, a.y * qn);   // c*carry + s*sc*q
                carry = fma(b.x, carry, b.y * qn);               // -s*carry + c*sc*q
                S[(size_t)j * TR + r] = out;
              }
            } else {
              double* sp = S + r;
#pragma unroll 4
              for (int j = 0; j < p.c_in - 1; ++j) {
                const double qn = sp[TR];
                const double2 a = H.rot[2 * j], b = H.rot[2 * j + 1];
                const double out = fma(a.x, carry, a.y * qn);
                carry = fma(b.x, carry, b.y * qn);
                *sp = out;
                *Qg = out;
                sp += TR;
                Qg += ld;
              }
            }
          } else {
            for (int j = 0; j < ncols; ++j) S[(size_t)j * TR + r] *= H.sc[j];
          }
          if (!del_only) {
            if (!tma_tile) p.Q[(size_t)k * p.ld + grow] = df;  // unnormalised new column (lazy scale)
            S[(size_t)vb * TR + r] = f;
            S[(size_t)dfs * TR + r] = df;
          }
        } else {
          // rows past this launch's range: the tensor copy zero-fills rows past n, but a
          // row-chunked launch (aa_step_host) ends mid-vector, where the staged rows hold the
          // next chunk's data -- zero them so the multi-dot and the Gram see only this range
          for (int j = 0; j < p.c_in; ++j) S[(size_t)j * TR + r] = 0.0;
          if (!del_only) {
            S[(size_t)vb * TR + r] = 0.0;
            S[(size_t)dfs * TR + r] = 0.0;
          }
        }
      } else if constexpr (OP == OP_K2_ICWY || OP == OP_K2B_CGS2) {
        // ICWY: Alg. 4 l.5  Delta f - Q (T^{-1} r);  CGS-2: Alg. 5 l.4  y - Q z
        if (r < rows) {
          double v0 = S[(size_t)k * TR + r], v1 = 0.0;
          int j = 0;
#pragma unroll 2
          for (; j + 1 < k; j += 2) {
            v0 -= H.coef[j] * S[(size_t)j * TR + r];
            v1 -= H.coef[j + 1] * S[(size_t)(j + 1) * TR + r];
          }
          if (j < k) v0 -= H.coef[j] * S[(size_t)j * TR + r];
          const double v = v0 + v1;
          p.Q[(size_t)k * p.ld + grow] = v;
          a0 += v * v;
          a1 += v * S[(size_t)(k + 1) * TR + r];
        }
      } else if constexpr (OP == OP_K2_DCGS2) {
        if (r < rows) {
          // Alg. 6 l.4 (reading A1): q_{k-1} <- q_{k-1} - Q_{0:k-2} s
          double qn = S[(size_t)(k - 1) * TR + r] * H.sc[k - 1];
          double v1 = 0.0;
          if (p.reortho) {
#pragma unroll 4
            for (int j = 0; j < k - 1; ++j) {
              const double qj = S[(size_t)j * TR + r];
              qn -= H.coef2[j] * qj;
              v1 -= H.coef[j] * qj;
            }
            p.Q[(size_t)(k - 1) * p.ld + grow] = qn;
          } else {
#pragma unroll 4
            for (int j = 0; j < k - 1; ++j) v1 -= H.coef[j] * S[(size_t)j * TR + r];
          }
          // Alg. 6 l.7: Delta f <- Delta f - Q_{0:k-1} R_{0:k-1,k}
          const double v = (S[(size_t)k * TR + r] - H.coef[k - 1] * qn) + v1;
          p.Q[(size_t)k * p.ld + grow] = v;
          a0 += v * v;
          a1 += v * S[(size_t)(k + 1) * TR + r];
        }
      } else if constexpr (OP == OP_K2A_CGS2) {
        if (r < rows) {
          double v0 = S[(size_t)k * TR + r], v1 = 0.0;
          int j = 0;
#pragma unroll 2
          for (; j + 1 < k; j += 2) {
            v0 -= H.coef[j] * S[(size_t)j * TR + r];
            v1 -= H.coef[j + 1] * S[(size_t)(j + 1) * TR + r];
          }
          if (j < k) v0 -= H.coef[j] * S[(size_t)j * TR + r];
          const double v = v0 + v1;
          p.Q[(size_t)k * p.ld + grow] = v;  // y (Alg. 5 l.2), in place
          S[(size_t)k * TR + r] = v;
          // phase B dots the STORED columns with y; the lazy scales are applied to the
          // per-CTA partials (z_j = sc_j * sum_r Q_stored[r][j] y[r])
        }
        // rows past n: the tensor copy zero-filled every column
      } else if constexpr (OP == OP_K2_MGS) {
        if (r < rows) {
          // Alg. 3 l.3 (column j-1) then l.2 for column j (or the norm, l.5)
          const double v = S[(size_t)TR + r] - H.scal[0] * S[r];
          p.Q[(size_t)k * p.ld + grow] = v;
          const double w = S[2 * (size_t)TR + r];
          if (p.mgs_j < k) {
            a0 += w * H.scal[1] * v;
          } else {
            a0 += v * v;
            a1 += v * w;
          }
        }
      } else if constexpr (OP == OP_K4) {
        if (r < rows) {
          // Alg. 1 l.7: x_{i+1} = G(x_i) - G_i gamma   [- (1-beta)(f_i - Q Q^T f_i), A13]
          const double g = ldV(p, S, 0, r, rows, grow);
          const double x = ldV(p, S, 1, r, rows, grow);
          double x0 = g, x1 = 0.0;
          int j = 0;
          const bool bd = H.bd != 0;     // breakdown: x_{i+1} = G(x_i) exactly
#pragma unroll 2
          for (; j + 1 <= k && !bd; j += 2) {
            x0 -= H.coef[j] * S[(size_t)j * TR + r];
            x1 -= H.coef[j + 1] * S[(size_t)(j + 1) * TR + r];
          }
          if (j <= k && !bd) x0 -= H.coef[j] * S[(size_t)j * TR + r];
          double xn = x0 + x1;
          if (p.beta_on && !bd) {
            double t = S[(size_t)(vb + 2) * TR + r];
            for (int jj = 0; jj <= k; ++jj) t -= H.coef2[jj] * S[(size_t)(k + 1 + jj) * TR + r];
            xn -= H.scal[0] * t;
          }
          p.x_out[grow] = xn;
          const double d = xn - x;
          a0 += d * d;
        }
      } else if constexpr (OP == OP_GRAM) {
        if (r < rows)
          for (int j = 0; j < p.c_in; ++j) S[(size_t)j * TR + r] *= H.sc[j];
      }
    }

    // ------------------------------------------------------------ phase B (multi-dot)
    if constexpr ((NCW > 0 && !FUSED) || GRAM) {
      if (tma_tile) fence_proxy_async();   // this thread's stage writes -> visible to the TMA stores
      __syncthreads();
      if constexpr (OP == OP_K1) {
        if (tma_tile && tid == 0) {
          // recycle: Q columns 0..k (rotated block + Delta f) in one tensor store; start-up: the
          // new column; then f_i, G(x_i), Delta g
          if (p.recycle) {
            if (p.tm3d) tma_3d_s2g(&p.tm[0], (int)(row0 >> 8), 0, S);
            else tma_2d_s2g(&p.tm[0], (int)row0, 0, S);
          } else {
            bulk_s2g(p.Q + (size_t)k * p.ld + row0, S + (size_t)dfs * TR, (uint32_t)TR * 8u);
          }
          bulk_s2g(p.fp + row0, S + (size_t)vb * TR, (uint32_t)TR * 8u);
          bulk_s2g(p.gp + row0, S + (size_t)(vb + 1) * TR, (uint32_t)TR * 8u);
          bulk_s2g(p.dg_out + row0, S + (size_t)(vb + 2) * TR, (uint32_t)TR * 8u);
          bulk_commit();
        }
      }
      if constexpr (NCW > 0 && !FUSED) {
        if (H.na > 0) {
#pragma unroll 2
          for (int rr = lane; rr < TR; rr += 32) {
            const double* Sr = S + rr;
            double rhs[NRB];
#pragma unroll
            for (int b = 0; b < NRB; ++b) rhs[b] = Sr[roff[b]];
#pragma unroll
            for (int c = 0; c < NCW; ++c) {
              const double v = Sr[coff[c]];
#pragma unroll
              for (int b = 0; b < NRB; ++b) acc[c][b] = fma(v, rhs[b], acc[c][b]);
            }
          }
        }
      }
      if constexpr (GRAM) {
        if (do_gram) {
          for (int r0 = 4 * warp; r0 < TR; r0 += 4 * NWARP) {
            const double* Sr = S + r0;
            double fr[NB8];
#pragma unroll
            for (int X = 0; X < NB8; ++X) fr[X] = gfrag[X] >= 0 ? Sr[gfrag[X]] : 0.0;
#pragma unroll
            for (int I = 0; I < NB8; ++I)
#pragma unroll
              for (int J = 0; J <= I; ++J) dmma_8x8x4(gc0[I * (I + 1) / 2 + J], gc1[I * (I + 1) / 2 + J], fr[I], fr[J]);
          }
        }
      }
    }
    // the stage may be refilled only after the TMA stores have read it
    if (tma_tile && tid == 0) bulk_wait_read0();
    __syncthreads();
    if (lane == 0 && it + NS < my_count) {
      fence_proxy_async();
      const long long t2 = tb + (it + NS) * tg;
      const long long r2 = rbeg + t2 * TR;
      issue_tile_part(p, S, &bars[sidx], r2, (int)min((long long)TR, n - r2), warp);
    }
  }

  // the K1 TMA stores are complete before this CTA's results are published
  if (OP == OP_K1 && p.k1_tmastore && tid == 0) bulk_wait0();
  if (blockIdx.x == 0) AA_TL(4);
  // ------------------------------------------------------------ per-CTA partials
  double* mypart = p.part + (size_t)blockIdx.x * LRED;
  if constexpr (FUSED) {
    const K1Layout L = K1Layout::make(k, p.has_x, p.gram != 0);
    if (!del_only) {
      // the per-thread partials summed over the CTA in a fixed order: every thread writes its
      // NV values to shared memory (the stage ring is idle after the tile loop; row t of an
      // odd-strided table), then thread v sums column v over the 256 rows in four interleaved
      // chains combined as ((c0 + c1) + (c2 + c3)) -- no shuffles (MIO-bound at small n)
      constexpr int NV = 3 * KMAX + 3;
      constexpr int NVP = NV | 1;
      double* wbuf = stage0;
      if (my_count == 0) {   // (the spare CTA of small n: no rows, its partials are exact zeros)
        for (int v = tid; v < L.off_gram; v += NT)
          if (v != 2) mypart[v] = 0.0;
        if (tid == 0) mypart[2] = dx2_pref;
      } else {
      __syncthreads();
      {
        double* row = wbuf + (size_t)tid * NVP;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          row[j] = fa0[j];
          row[KMAX + j] = fa1[j];
          row[2 * KMAX + j] = fa2[j];
        }
        row[3 * KMAX] = fs_ff;
        row[3 * KMAX + 1] = fs_dd;
        row[3 * KMAX + 2] = fs_df;
      }
      __syncthreads();
      for (int v = tid; v < NV; v += NT) {
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll 4
        for (int t = 0; t < NT; t += 4) {
          c0 += wbuf[(size_t)t * NVP + v];
          c1 += wbuf[(size_t)(t + 1) * NVP + v];
          c2 += wbuf[(size_t)(t + 2) * NVP + v];
          c3 += wbuf[(size_t)(t + 3) * NVP + v];
        }
        const double sum = (c0 + c1) + (c2 + c3);
        int wd = -1;
        if (v < KMAX) wd = (v < k) ? L.off_df + v : -1;
        else if (v < 2 * KMAX) wd = (v - KMAX < k) ? L.off_f + (v - KMAX) : -1;
        else if (v < 3 * KMAX) wd = (xrhs && v - 2 * KMAX < k - 1) ? L.off_x + (v - 2 * KMAX) : -1;
        else if (v == 3 * KMAX) wd = 0;       // f.f
        else if (v == 3 * KMAX + 1) wd = 1;   // df.df
        else wd = 3;                          // df.f
        if (wd >= 0) mypart[wd] = sum;
      }
      if (tid == 0) mypart[2] = dx2_pref;
      }
    }
  } else if constexpr (OP == OP_K1) {
    const K1Layout L = K1Layout::make(k, p.has_x, p.gram != 0);
    if (!del_only) {
      // all NCW x NRB butterflies level by level (independent shuffles in flight together)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < NCWx; ++c)
#pragma unroll
          for (int b = 0; b < NRB; ++b) acc[c][b] += __shfl_xor_sync(0xffffffffu, acc[c][b], o);
#pragma unroll
      for (int c = 0; c < NCWx; ++c) {
        const int a = warp + c * NWARP;
        if (NCW > 0 && a < H.na) {
#pragma unroll
          for (int b = 0; b < NRB; ++b) {
            const double v = acc[c][b];
            if (lane == 0) {
              int w = -1;
              if (a < k) {
                if (b == 0) w = L.off_df + a;
                else if (b == 1) w = L.off_f + a;
                else if (p.has_x && p.gram == 0 && a < k - 1) w = L.off_x + a;
              } else if (a == k) {
                if (b == 1) w = 0;  // f.f
              } else {
                if (b == 0) w = 1;       // df.df
                else if (b == 1) w = 3;  // df.f
              }
              if (w >= 0) mypart[w] = v;
            }
          }
        }
      }
      if (tid == 0) mypart[2] = dx2_pref;
    }
    if constexpr (GRAM) {
      if (do_gram)
        gram_epilogue<NB8>(p, gc0, gc1, stage0, mypart, kgx, GX ? 3 : (del_only ? 1 : 0), L.off_x, L.off_gram,
                           L.off_df, L.off_f);
    }
  } else if constexpr (OP == OP_K2A_CGS2) {
#pragma unroll
    for (int c = 0; c < NCWx; ++c) {
      const int a = warp + c * NWARP;
      if (NCW > 0 && a < H.na) {
        const double v = warp_sum(acc[c][0]);
        if (lane == 0) mypart[a] = v * H.sc[a];   // lazy scale of column a (lcol[a] = a)
      }
    }
  } else if constexpr (OP == OP_GRAM) {
    if constexpr (GRAM) {
      if (do_gram) gram_epilogue<NB8>(p, gc0, gc1, stage0, mypart, kg, 2, 0, 0, 0, 0);
    }
  } else {
    // row-wise accumulators: block reduction
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    if (lane == 0) {
      H.redw[warp][0] = a0;
      H.redw[warp][1] = a1;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int w = 0; w < NWARP; ++w) {
        s0 += H.redw[w][0];
        s1 += H.redw[w][1];
      }
      mypart[0] = s0;
      if (p.words > 1) mypart[1] = s1;
    }
  }

  if (blockIdx.x == 0) AA_TL(5);
  // ------------------------------------------------------------ cross-CTA reduction
  if (gridDim.x > 1) {
    // the barrier orders every thread's partial stores before thread 0's ticket, an
    // acquire-release atomic at GPU scope: its release half publishes them (cumulatively),
    // its acquire half orders the last CTA's reads of the others' partials (through L2,
    // __ldcg, after the next barrier) -- no separate fences
    __syncthreads();
    if (tid == 0) {
      unsigned int t;
      asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(&p.st->counter) : "memory");
      H.is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!H.is_last) return;
  } else {
    __syncthreads();   // one CTA: its own partials are visible after the barrier
  }
  AA_TL(6);   // last CTA
  double* outv = (OP == OP_K4) ? reinterpret_cast<double*>(H.scal) + 4 : p.red + (size_t)p.red_slot * LRED;
  if (p.det_tpc > 0) {
    // deterministic mode: the chunk partials (one per CTA) in the aligned tree, one warp per word
    const int G = (int)gridDim.x;
    for (int w = warp; w < p.words; w += NWARP) {
      const double sum = aligned_tree_sum_warp(G, [&](int b) { return __ldcg(p.part + (size_t)b * LRED + w); });
      if (lane == 0) outv[w] = sum;
    }
  } else
  {
    // K lanes per word (a power of two: as many as the words leave, at most a warp): lane q of a
    // word's group sums the CTAs b = q, q + K, ... in order (independent loads in flight), then
    // a fixed butterfly across the group -- a fixed order for a given grid, so results stay
    // bitwise reproducible; one thread walking all CTAs serially costs a full L2 latency per
    // few CTAs (296 CTAs at n >= 1.5e6: ~20 us per launch)
    const int words = p.words;
    const int G = (int)gridDim.x;
    int K = 32;
    while (K > 1 && K * words > NT) K >>= 1;
    const int q = tid & (K - 1), grp = tid / K, ngrp = NT / K;
    const int rounds = (words + ngrp - 1) / ngrp;
    for (int rd = 0; rd < rounds; ++rd) {
      const int w = grp + rd * ngrp;
      const bool valid = w < words;
      double s = 0.0;
      if (valid) {
#pragma unroll 8
        for (int b = q; b < G; b += K) s += __ldcg(p.part + (size_t)b * LRED + w);
      }
      for (int o = K >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (valid && q == 0) {
        // row-chunked launches (aa_step_host) add to the previous chunks' sums, in chunk order
        if (!p.chunk_first) s += (OP == OP_K4) ? (w == 0 ? p.st->dx2_acc : 0.0) : outv[w];
        outv[w] = s;
      }
    }
  }
  __syncthreads();
  if constexpr (OP != OP_K4) {
    if (p.nxchg > 0) {
      // sequence numbers from the device counter (stream order: the previous kernel's last
      // CTA has advanced it before this grid passed griddepcontrol.wait)
      if (tid == 0) {
        H.xbase = *p.xseq;
        *p.xseq = H.xbase + (unsigned long long)p.nxchg;
      }
      __syncthreads();
      for (int e = 0; e < p.nxchg; ++e) fused_exchange(p, outv + p.xoff[e], p.xcnt[e], H.xbase + 1ull + e);
    }
  }
  if constexpr (OP == OP_K4) {
    if (tid == 0 && !p.chunk_last) p.st->dx2_acc = outv[0];
    // run-time scalars (the factors were written by CTA 0 from its head)
    if (tid == 0 && p.chunk_last && !(p.flags & F_DELETE_ONLY)) {
      SmallState* st = p.st;
      hd = tail_hd;
      st->last_rkk = hd.rkk;
      const double dfn = sqrt(hd.df2);
      const double ratio = dfn > 0.0 ? hd.rkk / dfn : 0.0;
      if (ratio < tail_rmin) st->rratio_min = ratio;
      if (!(hd.rkk > p.eps_a * dfn)) {   // reading A12: this step's column is dependent
        st->breakdown = 1;
        st->breakdown_count += 1;
        if (p.bd_host) {   // the mapped pinned word aa_step polls (without blocking)
          *reinterpret_cast<volatile int*>(p.bd_host) = 1;
          __threadfence_system();
        }
      }
      if (!(p.flags & F_EXT_DF)) {
        st->f2 = tail_f2;
        st->dx2_local = outv[0];
      }
    }
  }
  // every CTA has taken its ticket; the reset is ordered before the next launch by the
  // kernel boundary
  if (tid == 0 && gridDim.x > 1) p.st->counter = 0u;
  AA_TL(7);
}

// aa_test_exchange: `iters` back-to-back one-shot exchanges of `words` words by one CTA,
// timed on the device with %globaltimer (per-exchange latency)
__global__ void __launch_bounds__(NT, 1) aa_xchg_bench_kernel(const __grid_constant__ KParams p, int words,
                                                               int iters, unsigned long long* out_ns) {
  __shared__ unsigned long long base;
  double* v = p.red + (size_t)(NSLOT - 2) * LRED;
  for (int w = threadIdx.x; w < words; w += NT) v[w] = (double)(p.rank + 1) * 1e-3 + (double)w;
  if (threadIdx.x == 0) {
    base = *p.xseq;
    *p.xseq = base + (unsigned long long)iters;
  }
  __syncthreads();
  const unsigned long long t0 = global_ns();
  for (int it = 0; it < iters; ++it) {
    fused_exchange(p, v, words, base + 1ull + (unsigned long long)it);
    for (int w = threadIdx.x; w < words; w += NT) v[w] *= 1e-3;   // keep the values bounded
    __syncthreads();
  }
  const unsigned long long t1 = global_ns();
  if (threadIdx.x == 0) *out_ns = t1 - t0;
}

// deterministic mode over NCCL: v[w] = aligned tree over ranks of gathered[q * cnt + w]
__global__ void aa_det_rank_sum_kernel(double* v, const double* gathered, int cnt, int R) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < cnt; w += gridDim.x * blockDim.x) {
    double t[MAX_RANKS];
    for (int q = 0; q < R; ++q) t[q] = gathered[(size_t)q * cnt + w];
    v[w] = aligned_tree_sum_small(t, R);
  }
}

// counter-based SplitMix64 uniform generator (aa_testing.h), bitwise equal to
// aa_inputs.uniform: u = (z >> 11) * 2^-53, value = lo + (hi - lo) * u without FMA.
__global__ void aa_fill_uniform_kernel(double* out, long long n, unsigned long long base,
                                       double lo, double width) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = base + (unsigned long long)i + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const double u = (double)(z >> 11) * 0x1.0p-53;
    out[i] = __dadd_rn(lo, __dmul_rn(width, u));
  }
}

// aa_init: f_0 = G(x_0) - x_0, keep G(x_0), x_1 = G(x_0)  (Alg. 1 l.1)
__global__ void aa_init_kernel(const double* __restrict__ x0, const double* gx0, double* x1,
                               double* fp, double* gp, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = gx0[i];
    fp[i] = g - x0[i];
    gp[i] = g;
    x1[i] = g;
  }
}

// normalised copy of the active Q columns (aa_get_q)
__global__ void aa_copy_q_kernel(const double* Q, long long ld, const SmallState* st, int ver, int mi,
                                 double* out, long long n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n * mi;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long j = idx / n, i = idx % n;
    out[idx] = Q[j * ld + i] * st->f[ver].scale[j];
  }
}

}  // namespace aa
