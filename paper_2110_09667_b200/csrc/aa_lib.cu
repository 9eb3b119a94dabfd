// aa_lib.cu — libaa host side: the C ABI of include/aa.h and include/aa_testing.h,
// the per-variant schedule of kernels and allreduces (one ncclAllReduce per global
// reduction), and the reduction ledger.  P:n = PAPER.md line n.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "../../include/aa.h"
#include "../../include/aa_testing.h"
#include "aa_kernels.cuh"

using namespace aa;

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(lib, "ncclCommInitRank");
  api.AllReduce = (decltype(api.AllReduce))dlsym(lib, "ncclAllReduce");
  api.AllGather = (decltype(api.AllGather))dlsym(lib, "ncclAllGather");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(lib, "ncclCommDestroy");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(lib, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
  return api;
}
}  // namespace

// ------------------------------------------------------------------ handle
struct TimedEv {
  int cls;
  cudaEvent_t a, b;
};

struct aa_ctx {
  int64_t n = 0, ld = 0, n_global = 0;
  int m = 0, variant = 0, rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int device = 0, sms = 148;
  double *Q = nullptr, *DG = nullptr, *fp = nullptr, *gp = nullptr;
  SmallState* st = nullptr;
  double *red = nullptr, *part = nullptr;
  double *hx = nullptr, *hg = nullptr, *hxn = nullptr;  // staging for aa_step_host
  bool hxn_valid = false;   // hxn holds the x_{i+1} the last aa_step_host returned
  int* bd_host = nullptr;   // mapped pinned breakdown word (written by K4, polled by aa_step)
  // AA_OPT_DETERMINISTIC: one partial slot per DET_ROWS chunk, and the all-gather buffer of the
  // NCCL path (ranks summed in the aligned tree by aa_det_rank_sum_kernel)
  int det = 0;
  // K1 form for 7..22 columns: 0 fused row pass + dots (FUSED), 1 split row pass + block
  // multi-dot; chosen per (device, m, n) by timing both at aa_init (k1_form_trial)
  int k1_split = 0;
  double* part_det = nullptr;
  double* xgather = nullptr;
  int* bd_dev = nullptr;    // its device alias
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  // window bookkeeping (host; depends only on i, m_i)
  int64_t iter = 0;
  int mi = 0, dg_head = 0;
  int ver = 0;  // factor version read by the next step (K4 writes ver ^ 1)
  int max_tr_blocks = 512;  // tallest tile for kernels with column blocks
  // fused one-shot NVLink allreduce (AA_OPT_FUSED_ALLREDUCE)
  int fused = 0;
  void* xbuf = nullptr;                 // local [flags 4 KB][mailbox 2 x nranks x LRED]
  void* peer_base[MAX_RANKS] = {};
  unsigned long long* tl = nullptr;   // test-only phase timeline (aa_test_timeline)
  bool inited = false;
  int failed = AA_OK;
  // options
  double beta = 1.0, eps_a = -1.0;
  int icwy_merged = 0, dcgs2_cond = 3, dcgs2_rscale = 0, profile = 0;
  int conv_norm = 0;   // AA_OPT_CONV_NORM: 0 lagged, 1 immediate, 2 off
  cudaStream_t cstream = nullptr;                     // aa_step_host copy stream (lazy)
  cudaEvent_t chunk_evH[8] = {}, chunk_evK[8] = {};
  // ledger
  int64_t logical[5] = {0, 0, 0, 0, 0}, logical_last[5] = {0, 0, 0, 0, 0};
  int64_t ar_total = 0;
  int ar_last = 0, sp_last = 0;
  int64_t launches = 0;
  std::vector<TimedEv> evs;
  std::map<std::tuple<int, int, int>, CUtensorMap> tmaps;  // (buffer, box cols, box rows)
  double t_ms[5] = {0, 0, 0, 0, 0};
  int64_t t_cnt[5] = {0, 0, 0, 0, 0};
};

namespace {

int fail(aa_ctx* c, int code) {
  if (c && c->failed == AA_OK) c->failed = code;
  return code;
}

#define CUDA_TRY(c, expr)                                                                    \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      fprintf(stderr, "libaa: CUDA error %s at %s:%d: %s\n", cudaGetErrorString(_e), __FILE__, \
              __LINE__, #expr);                                                              \
      return fail(c, AA_ERR_CUDA);                                                           \
    }                                                                                        \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

double* qcol(aa_ctx* c, int j) { return c->Q + (size_t)j * c->ld; }
double* dgcol(aa_ctx* c, int slot) { return c->DG + (size_t)slot * c->ld; }

// Tile rows / stage count: the largest tile that keeps >= 3 stages within ~200 KB of
// shared memory (tools/stream_bench.cu: ~7 TB/s at 252-256 rows, 3-4 stages, 1 CTA/SM).
// Kernels with a DMMA Gram take TR in {252,124,60,28} (bank skew), the others
// TR in {256,128,64,32} (every 2-D box lands 128-byte aligned).
// Tile rows TR and stage count NS of one launch.  Two CTAs per SM with a 2-stage ring
// each when registers allow (<= 128 per thread): the largest TR <= max_tr whose two stages
// fit in ~104 KB.  Otherwise one CTA with >= 3 stages in ~200 KB.  Kernels with a DMMA
// Gram take TR in {252,124,60,28} (bank skew), vector-only kernels up to 1024 rows
// (1-D copies of 8 KB), the rest TR in {256,128,64,32} (2-D boxes 128-byte aligned).
// Measured on B200 (tools/tune_tiles.sh, config 2, m = 20): see DESIGN.md §7.
bool choose_tile(int nin, bool skew, bool vec_only, size_t budget, int min_stages, int max_stages, int max_tr,
                 int* tr, int* stages) {
  static const int trs_s[] = {252, 124, 60, 28};
  static const int trs_p[] = {1024, 512, 256, 128, 64, 32};
  static const int trs_v[] = {1024, 512, 256, 128, 64, 32};
  const int* trs = skew ? trs_s : (vec_only ? trs_v : trs_p);
  const int nt = skew ? 4 : 6;
  for (int t = 0; t < nt; ++t) {
    if (trs[t] > max_tr) continue;
    const size_t sb = align_up((size_t)nin * trs[t], 16) * sizeof(double);
    const int s = (int)std::min<size_t>((size_t)max_stages, budget / sb);
    if (s >= min_stages) {
      *tr = trs[t];
      *stages = s;
      return true;
    }
  }
  *tr = trs[nt - 1];
  *stages = 2;
  return false;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

// 2-D tensor map over a column-major n x m buffer (Q or the Delta G ring), box = tr rows
// x ncols columns; rows past n read as zero.  Cached per (buffer, ncols, tr).
const CUtensorMap* get_map(aa_ctx* c, int which, int ncols, int tr) {
  auto key = std::make_tuple(which, ncols, tr);
  auto it = c->tmaps.find(key);
  if (it != c->tmaps.end()) return &it->second;
  auto fn = encode_fn();
  if (!fn) return nullptr;
  CUtensorMap m;
  void* base = which == 0 ? (void*)c->Q : (void*)c->DG;
  CUresult r;
  if (tr % 256 == 0) {
    // 3-D view {256 rows, ld/256 row blocks, m columns}: a box of tr/256 row blocks; the
    // padding rows [n, ld) are zero (never written), row blocks past ld are zero-filled
    cuuint64_t gdim[3] = {256, (cuuint64_t)(c->ld / 256), (cuuint64_t)c->m};
    cuuint64_t gstr[2] = {256 * sizeof(double), (cuuint64_t)(c->ld * sizeof(double))};
    cuuint32_t box[3] = {256, (cuuint32_t)(tr / 256), (cuuint32_t)ncols};
    cuuint32_t es[3] = {1, 1, 1};
    r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t gdim[2] = {(cuuint64_t)c->n, (cuuint64_t)c->m};
    cuuint64_t gstr[1] = {(cuuint64_t)(c->ld * sizeof(double))};
    cuuint32_t box[2] = {(cuuint32_t)tr, (cuuint32_t)ncols};
    cuuint32_t es[2] = {1, 1};
    r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "libaa: cuTensorMapEncodeTiled failed (%d) for %d cols x %d rows\n", (int)r, ncols, tr);
    return nullptr;
  }
  return &(c->tmaps[key] = m);
}

// Column-block / vector description of a kernel's inputs (before the tile is chosen).
struct Inputs {
  int nblk = 0, nvec = 0;
  int blk_which[NBLK_MAX], blk_gcol[NBLK_MAX], blk_ncols[NBLK_MAX];
  const double* vec[NVEC_MAX];
  unsigned exact = 0;
  void block(int which, int gcol, int ncols) {
    if (ncols <= 0) return;
    blk_which[nblk] = which;
    blk_gcol[nblk] = gcol;
    blk_ncols[nblk] = ncols;
    ++nblk;
  }
  void vector(const double* v, bool is_exact) {
    if (is_exact) exact |= 1u << nvec;
    vec[nvec++] = v;
  }
  int ncols() const {
    int s = 0;
    for (int b = 0; b < nblk; ++b) s += blk_ncols[b];
    return s;
  }
};

struct EvScope {
  aa_ctx* c;
  int cls;
  cudaEvent_t a = nullptr;
  EvScope(aa_ctx* c_, int cls_) : c(c_), cls(cls_) {
    if (c->profile) {
      cudaEventCreate(&a);
      cudaEventRecord(a, c->stream);
    }
  }
  ~EvScope() {
    if (c->profile) {
      cudaEvent_t b;
      cudaEventCreate(&b);
      cudaEventRecord(b, c->stream);
      c->evs.push_back({cls, a, b});
    }
  }
};

// Launch one instantiation.  The tile (TR rows x stages) is chosen here, knowing the
// kernel's register count: when registers allow two 256-thread CTAs per SM (<= 128 per
// thread) the stage ring is sized for ~110 KB per CTA so two CTAs share each SM (twice
// the warps to hide the fp64 / shared-memory latencies of phases A and B); otherwise one
// CTA gets ~200 KB.
template <int OP, int NCW, int G>
int launch_inst(aa_ctx* c, KParams& p, size_t /*unused*/, int cls) {
  static int regs = -1;
  if (regs < 0) {
    cudaFuncAttributes fa;
    CUDA_TRY(c, cudaFuncGetAttributes(&fa, aa_stream_kernel<OP, NCW, G>));
    regs = fa.numRegs;
  }
  // deterministic mode: tiles of a multiple of 256 rows dividing DET_ROWS (so every thread sees
  // the same rows of a chunk in the same order whatever the tile), no bank-skewed Gram tiles
  const bool skew = (G > 0) && !c->det;
  const bool vec_only = (p.nblk == 0 && p.nin > 0);
  const int nin = std::max(p.nin, 1);
  // Tile policy (tools/tune_tiles.sh sweeps, config 2, m in {5,10,20,50}):
  // the tallest tile (<= 512 rows for column-block kernels via 3-D tensor maps; 252 with a
  // DMMA Gram; 1024 for vector-only kernels) whose 2-stage ring fits one CTA's shared
  // memory; then as many extra stages (<= 4) as fit while two CTAs share an SM (when the
  // registers allow) -- small tiles (few columns) need them to keep bytes in flight.
  int tr = 0, stages = 0;
  bool k1_two = false;
  // (the Gram instances too when they fit: m = 10 K1 0.70 -> 0.72, m = 20 0.76 -> 0.77 of peak)
  if (OP == OP_K1 && nin < 20 && regs <= 128)
    // K1 with few columns: keep two CTAs per SM (16 warps hide the rotation chain); the Gram
    // instances with a third stage when it still fits (ICWY m = 5: K1 2.46 -> 2.27 ms, m = 10
    // equal; profiles/r02/icwy_smallm_tiles.txt)
    k1_two = choose_tile(nin, skew, vec_only, 104 * 1024, 2, G > 0 ? 3 : 2, c->max_tr_blocks, &tr, &stages) &&
             tr >= (skew ? 252 : 256);
  // CGS-2's K2a (phase B dots the y that phase A just produced, so a tile's two phases
  // serialise): two CTAs per SM overlap them -- the tallest tile, up to 1024 rows, whose
  // 2-stage ring lets two CTAs share an SM (sweeps: m = 20 256 rows, K2 5.34 -> 5.05 ms;
  // m = 5 1024 rows, 1.97 -> 1.74 ms)
  bool k2a_two = false;
  if (OP == OP_K2A_CGS2 && !skew && regs <= 128)
    k2a_two = choose_tile(nin, skew, vec_only, 104 * 1024, 2, 2, 1024, &tr, &stages) && tr >= 256;
  // the projection kernels (K2 ICWY / DCGS-2, CGS-2's K2b) stream best with tiles up to 1024
  // rows when few columns let a 2-stage ring fit (m = 5 / 10: K2 3-6 % faster; m >= 20 falls
  // back to 512 rows by itself); K1 and K4 keep 512
  const bool tall = vec_only || OP == OP_K2_ICWY || OP == OP_K2_DCGS2 || OP == OP_K2B_CGS2;
  // K1 keeps 2 stages here: the fused-dot form at m = 10 took 3 on an earlier build and box
  // (K1 3.74 -> 3.67 ms, profiles/r02/k1_tiles.txt), but on the final build 2 measured faster
  // in both repetitions (3.54 -> 3.37 ms, profiles/r02/tiles_final_ab.txt); the ICWY Gram K1
  // with up to 6 stages of 252-row tiles was slower (m = 10 0.69 -> 0.50, m = 20 0.77 -> 0.59)
  const int k1_max_stages = 2;
  if (!k1_two && !k2a_two)
    choose_tile(nin, skew, vec_only, 220 * 1024, 2, k1_max_stages, tall ? 1024 : c->max_tr_blocks, &tr, &stages);
  // (MGS's one-axpy-one-dot K2 keeps 2: with 4 its 1024-row tiles measured 8 % slower,
  // m = 10 K2 4.63 -> 4.24 ms, m = 20 9.80 -> 9.02 ms, profiles/r02/tiles_final_ab.txt)
  if (OP != OP_K1 && OP != OP_K2_MGS) {
    const size_t sb = align_up((size_t)nin * tr, 16) * sizeof(double);
    const size_t budget = (regs <= 128 && 2 * sb <= 104 * 1024) ? 104 * 1024 : 0;
    if (budget) stages = (int)std::max<size_t>(2, std::min<size_t>(4, budget / sb));
  }
  // small n: while the tiles would cover at most half the SMs, halve a column-block kernel's tile (down to 256
  // rows) so more SMs stream the vectors (n = 1000, m = 20: DCGS-2 32.5 -> 29.6 us per step)
  {
    const long long nrows = p.n - p.rbeg;
    while (!skew && !vec_only && tr >= 512 && tr % 256 == 0 && ((nrows + tr - 1) / tr) * 2 <= c->sms) tr /= 2;
  }
  if (c->det && tr < 256) {   // (few columns may pick taller tiles; never shorter than 256 rows)
    tr = 256;
    stages = 2;
  }
  // tuning override (tools only): AA_TILE="<op>:<tr>:<stages>[,<op>:<tr>:<stages>...]", read once
  static const char* const tile_override = getenv("AA_TILE");
  if (const char* ov = tile_override) {
    const char* q = ov;
    while (*q) {
      int o, t, s, used = 0;
      if (sscanf(q, "%d:%d:%d%n", &o, &t, &s, &used) == 3 && used > 0) {
        if (o == OP && t >= 4 && s >= 1 && s <= MAXSTAGES) {
          tr = skew ? (t / 4) * 4 : t;
          stages = s;
        }
        q += used;
        if (*q == ',') ++q;
      } else {
        break;
      }
    }
  }
  p.tr = tr;
  p.stages = stages;
  p.tm3d = (tr % 256 == 0) ? 1 : 0;
  for (int b = 0; b < p.nblk; ++b) {
    const CUtensorMap* m = get_map(c, p.blk_which[b], p.blk_ncols[b], tr);
    if (!m) return fail(c, AA_ERR_CUDA);
    p.tm[b] = *m;
  }
  const size_t stage_bytes = (size_t)stages * align_up((size_t)nin * tr, 16) * sizeof(double);
  size_t scr = (OP == OP_K4) ? scratch_bytes_k4(p.m, p.variant == V_ICWY && p.icwy_merged == 2) : scratch_bytes();
  if (OP == OP_K1 && G == 0 && NCW >= 2 && NCW <= 3) scr = std::max(scr, fused_k1_table_bytes(NCW));
  // the head scratch gets its own region after the stages when that fits without costing
  // occupancy (then the first TMA loads can be issued before the heads run)
  size_t smem = head_bytes() + bar_bytes() + std::max(stage_bytes, scr);
  static const bool early_off = getenv("AA_NO_EARLY_TMA") && atoi(getenv("AA_NO_EARLY_TMA")) != 0;
  p.early_tma = early_off ? 0 : 1;
  p.scr_off = 0;
  if ((OP == OP_K4 || OP == OP_K2_ICWY) && !early_off) {
    const size_t sep = head_bytes() + bar_bytes() + stage_bytes + scr;
    constexpr size_t kMaxSmem = 227 * 1024, kTwoPerSm = 110 * 1024;
    if (sep <= kMaxSmem && (smem > kTwoPerSm || sep <= kTwoPerSm)) {
      p.scr_off = (long long)(stage_bytes / sizeof(double));
      smem = sep;
    }
  }
  // per-device state of this instance (function attributes are set per device)
  constexpr int kMaxDev = 16;
  const int dev = (c->device >= 0 && c->device < kMaxDev) ? c->device : 0;
  static size_t attr_set[kMaxDev] = {};
  if (smem > attr_set[dev]) {
    CUDA_TRY(c, cudaFuncSetAttribute(aa_stream_kernel<OP, NCW, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 110 * 1024)));
    attr_set[dev] = std::max<size_t>(smem, 110 * 1024);
  }
  // resident CTAs per SM for this instance and shared-memory size (cached: the query costs
  // host time on every launch otherwise, which matters at small n)
  static size_t occ_smem[kMaxDev][8];
  static int occ_val[kMaxDev][8], occ_n[kMaxDev] = {};
  int per_sm = 0;
  for (int i = 0; i < occ_n[dev]; ++i)
    if (occ_smem[dev][i] == smem) per_sm = occ_val[dev][i];
  if (per_sm == 0) {
    CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, aa_stream_kernel<OP, NCW, G>, NT, smem));
    per_sm = std::max(1, std::min(per_sm, 2));
    if (occ_n[dev] < 8) {
      occ_smem[dev][occ_n[dev]] = smem;
      occ_val[dev][occ_n[dev]++] = per_sm;
    }
  }
  const long long ntiles = (p.n - p.rbeg + p.tr - 1) / p.tr;
  long long grid = std::min<long long>(ntiles, (long long)c->sms * per_sm);
  if (grid < 1) grid = 1;
  p.det_tpc = 0;
  if (c->det && p.n > 0) {   // one CTA per DET_ROWS chunk (n_local is a multiple of DET_ROWS)
    p.det_tpc = (int)(DET_ROWS / p.tr);
    p.part = c->part_det;
    p.k1_pre = 0;
    grid = (p.n - p.rbeg) / DET_ROWS;
  }
  // K4 when the tiles do not fill the GPU: one extra CTA (CTA 0) writes the next factor
  // version and precomputes the next QRDelete while the others run gamma + the x update,
  // so that serial work leaves the kernel's critical path
  p.pre_cta = 0;
  if (OP == OP_K4 && !c->det && ntiles >= 1 && ntiles + 1 <= (long long)c->sms * per_sm) {
    p.pre_cta = 1;
    grid = ntiles + 1;
  } else if (OP == OP_K4 && !c->det && ntiles <= 32 * (long long)c->sms * per_sm && grid >= 2) {
    // mid n: CTA 0 still only commits (its ~3 us of serial head work would otherwise delay its
    // share of the tiles, the kernel's tail); the other CTAs take every tile
    p.pre_cta = 1;
  }
  // K1 when the tiles do not fill the GPU: one extra CTA (CTA 0) computes the early rotations of
  // the next QRDelete (k1_delete_pre) while the others stream; K4 then only finishes them
  if (OP == OP_K1) {
    if (p.k1_pre && ntiles >= 1 && ntiles + 1 <= (long long)c->sms * per_sm) {
      p.pre_cta = 1;
      grid = ntiles + 1;
    } else {
      p.k1_pre = 0;
    }
  }
  {
    EvScope ev(c, cls);
    // programmatic dependent launch (griddepcontrol in the kernel): the launch and CTA
    // ramp-up overlap the predecessor's tail; AA_NO_PDL=1 disables it (A/B measurements)
    static const bool pdl = !(getenv("AA_NO_PDL") && atoi(getenv("AA_NO_PDL")) != 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_TRY(c, cudaLaunchKernelEx(&cfg, aa_stream_kernel<OP, NCW, G>, p));
  }
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  return AA_OK;
}

#define AA_NCW_CASES(OP, G)                                \
  switch (ncw) {                                           \
    case 1: return launch_inst<OP, 1, G>(c, p, smem, cls); \
    case 2: return launch_inst<OP, 2, G>(c, p, smem, cls); \
    case 3: return launch_inst<OP, 3, G>(c, p, smem, cls); \
    case 4: return launch_inst<OP, 4, G>(c, p, smem, cls); \
    case 5: return launch_inst<OP, 5, G>(c, p, smem, cls); \
    case 6: return launch_inst<OP, 6, G>(c, p, smem, cls); \
    case 7: return launch_inst<OP, 7, G>(c, p, smem, cls); \
    case 8: return launch_inst<OP, 8, G>(c, p, smem, cls); \
    default: return launch_inst<OP, 9, G>(c, p, smem, cls); \
  }
// K1 with the DMMA Gram: NB8 = ceil(k/8) and NCW = ceil((k+2)/8) in {NB8, NB8+1}
#define AA_K1_GRAM_CASE(NB)                                                        \
  case NB:                                                                         \
    if (ncw == NB) return launch_inst<OP_K1, NB, NB>(c, p, smem, cls);             \
    return launch_inst<OP_K1, (NB < 9 ? NB + 1 : 9), NB>(c, p, smem, cls);

template <int OP>
int launch_op(aa_ctx* c, KParams& p, const Inputs& in, int cls) {
  const bool gram = (OP == OP_GRAM) || (OP == OP_K1 && p.gram != 0);
  (void)gram;
  const int nin = in.ncols() + in.nvec;
  p.nin = nin;
  p.vb = in.ncols();
  p.nblk = in.nblk;
  p.nvec = in.nvec;
  p.exact_vec = in.exact;
  for (int b = 0; b < in.nblk; ++b) {
    p.blk_which[b] = in.blk_which[b];
    p.blk_gcol[b] = in.blk_gcol[b];
    p.blk_ncols[b] = in.blk_ncols[b];
  }
  for (int i = 0; i < in.nvec; ++i) p.vec[i] = in.vec[i];
  const size_t smem = 0;
  p.st = c->st;
  p.tl = c->tl;
  p.ver = c->ver;
  p.red = c->red;
  p.part = c->part;
  p.Q = c->Q;
  p.ld = c->ld;
  p.fp = c->fp;
  p.gp = c->gp;
  if constexpr (OP == OP_K1) {
    int ncw = (p.flags & F_DELETE_ONLY) ? 1 : (p.k + 2 + NWARP - 1) / NWARP;
    // AA_K1_NOFUSE=1 (A/B only): the split row pass + block multi-dot instead of the fused one
    // (an NCW = 4 instance covers up to 30 columns, unused warps' columns are skipped)
    static const bool nofuse = getenv("AA_K1_NOFUSE") && atoi(getenv("AA_K1_NOFUSE")) != 0;
    if ((nofuse || c->k1_split) && !gram && (ncw == 2 || ncw == 3)) ncw = 4;
    if (gram) {
      const int kg = (p.flags & F_DELETE_ONLY) ? p.c_in - 1 : p.k;
      const int nb8 = (kg + 7) / 8;
      if (p.flags & F_DELETE_ONLY) {
        switch (nb8) {
          case 1: return launch_inst<OP_K1, 1, 1>(c, p, smem, cls);
          case 2: return launch_inst<OP_K1, 1, 2>(c, p, smem, cls);
          case 3: return launch_inst<OP_K1, 1, 3>(c, p, smem, cls);
          case 4: return launch_inst<OP_K1, 1, 4>(c, p, smem, cls);
          case 5: return launch_inst<OP_K1, 1, 5>(c, p, smem, cls);
          case 6: return launch_inst<OP_K1, 1, 6>(c, p, smem, cls);
          case 7: return launch_inst<OP_K1, 1, 7>(c, p, smem, cls);
          default: return launch_inst<OP_K1, 1, 8>(c, p, smem, cls);
        }
      }
      // Delta f and f_i as Gram columns k, k+1 when they fit the k columns' 8-column blocks
      // (k mod 8 in 1..6; AA_GRAM_MULTIDOT=1 keeps the block multi-dot, A/B only)
      static const bool gram_md = getenv("AA_GRAM_MULTIDOT") && atoi(getenv("AA_GRAM_MULTIDOT")) != 0;
      if (!gram_md && (p.k + 2 + 7) / 8 == nb8) {
        switch (nb8) {
          case 1: return launch_inst<OP_K1, 0, 1>(c, p, smem, cls);
          case 2: return launch_inst<OP_K1, 0, 2>(c, p, smem, cls);
          case 3: return launch_inst<OP_K1, 0, 3>(c, p, smem, cls);
          case 4: return launch_inst<OP_K1, 0, 4>(c, p, smem, cls);
          case 5: return launch_inst<OP_K1, 0, 5>(c, p, smem, cls);
          case 6: return launch_inst<OP_K1, 0, 6>(c, p, smem, cls);
          case 7: return launch_inst<OP_K1, 0, 7>(c, p, smem, cls);
          default: return launch_inst<OP_K1, 0, 8>(c, p, smem, cls);
        }
      }
      switch (nb8) {
        AA_K1_GRAM_CASE(1)
        AA_K1_GRAM_CASE(2)
        AA_K1_GRAM_CASE(3)
        AA_K1_GRAM_CASE(4)
        AA_K1_GRAM_CASE(5)
        AA_K1_GRAM_CASE(6)
        AA_K1_GRAM_CASE(7)
        default:
          if (ncw == 8) return launch_inst<OP_K1, 8, 8>(c, p, smem, cls);
          return launch_inst<OP_K1, 9, 8>(c, p, smem, cls);
      }
    } else {
      AA_NCW_CASES(OP_K1, 0)
    }
  } else if constexpr (OP == OP_K2A_CGS2) {
    const int ncw = std::max(1, (p.k + NWARP - 1) / NWARP);
    AA_NCW_CASES(OP_K2A_CGS2, 0)
  } else if constexpr (OP == OP_GRAM) {
    switch ((p.c_in + 7) / 8) {
      case 1: return launch_inst<OP_GRAM, 0, 1>(c, p, smem, cls);
      case 2: return launch_inst<OP_GRAM, 0, 2>(c, p, smem, cls);
      case 3: return launch_inst<OP_GRAM, 0, 3>(c, p, smem, cls);
      case 4: return launch_inst<OP_GRAM, 0, 4>(c, p, smem, cls);
      case 5: return launch_inst<OP_GRAM, 0, 5>(c, p, smem, cls);
      case 6: return launch_inst<OP_GRAM, 0, 6>(c, p, smem, cls);
      case 7: return launch_inst<OP_GRAM, 0, 7>(c, p, smem, cls);
      default: return launch_inst<OP_GRAM, 0, 8>(c, p, smem, cls);
    }
  } else {
    return launch_inst<OP, 0, 0>(c, p, smem, cls);
  }
}

#define RET_IF_(x)              \
  do {                          \
    int _s = (x);               \
    if (_s != AA_OK) return _s; \
  } while (0)

int allreduce(aa_ctx* c, double* buf, size_t count) {
  if (c->nranks == 1 || count == 0) return AA_OK;
  EvScope ev(c, 3);
  if (c->det) {
    // deterministic: all-gather the rank vectors, every rank sums them in the aligned tree
    ncclResult_t r = nccl().AllGather(buf, c->xgather, count, kNcclFloat64, c->comm, c->stream);
    if (r != 0) {
      fprintf(stderr, "libaa: ncclAllGather failed: %s\n", nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
      return fail(c, AA_ERR_NCCL);
    }
    aa_det_rank_sum_kernel<<<(unsigned)std::max<size_t>(1, (count + 255) / 256), 256, 0, c->stream>>>(
        buf, c->xgather, (int)count, c->nranks);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    c->ar_last++;
    c->ar_total++;
    return AA_OK;
  }
  ncclResult_t r = nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm, c->stream);
  if (r != 0) {
    fprintf(stderr, "libaa: ncclAllReduce failed: %s\n",
            nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
    return fail(c, AA_ERR_NCCL);
  }
  c->ar_last++;
  c->ar_total++;
  return AA_OK;
}

constexpr size_t kFlagBytes = 4096;

// Plan the reduction(s) at the end of the kernel q: ranges [o0, o0+n0) and [o1, o1+n1) of
// its reduction slot, each ONE global reduction (n = 0: none).  Fused mode: the kernel's
// last CTA exchanges them over NVLink; otherwise post_ar() issues ncclAllReduce after it.
void plan_ar(aa_ctx* c, KParams& q, int o0, int n0, int o1, int n1) {
  q.nxchg = 0;
  if (!(c->fused && c->nranks > 1)) return;
  const int offs[2] = {o0, o1}, cnts[2] = {n0, n1};
  q.nranks = c->nranks;
  q.rank = c->rank;
  q.xseq = reinterpret_cast<unsigned long long*>(c->xbuf);   // header word 0 of the local buffer
  for (int e = 0; e < 2; ++e)
    if (cnts[e] > 0) {
      q.xoff[q.nxchg] = offs[e];
      q.xcnt[q.nxchg] = cnts[e];
      ++q.nxchg;
    }
  for (int r = 0; r < c->nranks; ++r) q.pmbox[r] = (double*)((char*)c->peer_base[r] + kFlagBytes);
  q.lmbox = (double*)((char*)c->xbuf + kFlagBytes);
  c->ar_last += q.nxchg;
  c->ar_total += q.nxchg;
}

int post_ar(aa_ctx* c, double* slot, int o0, int n0, int o1, int n1) {
  c->sp_last += (n0 > 0) + (n1 > 0);
  if (c->fused || c->nranks == 1) return AA_OK;
  if (n0 > 0) RET_IF_(allreduce(c, slot + o0, (size_t)n0));
  if (n1 > 0) RET_IF_(allreduce(c, slot + o1, (size_t)n1));
  return AA_OK;
}

KParams base_params(aa_ctx* c) {
  KParams p;
  memset(&p, 0, sizeof(p));
  p.variant = c->variant;
  p.m = c->m;
  p.n = c->n;
  p.beta = c->beta;
  p.eps_a = c->eps_a;
  p.icwy_merged = c->icwy_merged;
  p.rscale = c->dcgs2_rscale;
  p.rbeg = 0;
  p.chunk_first = 1;
  p.chunk_last = 1;
  p.bd_host = c->bd_dev;
  return p;
}

// aa_step_host at large n: the PCIe copies are split into row chunks on a copy stream so
// that K1 starts on the first chunk while the rest is still in flight, and x_{i+1} goes back
// chunk by chunk behind K4.  Chunk boundaries are multiples of 1024 rows.
constexpr int kMaxChunks = 8;
constexpr int64_t kChunkMinRows = 4 << 20;
struct ChunkPlan {
  int nc = 0;
  int64_t b[kMaxChunks + 1];
  cudaStream_t cs = nullptr;
  cudaEvent_t* evH = nullptr;   // chunk c of x_i, G(x_i) is on the device
  cudaEvent_t* evK = nullptr;   // K4 has written chunk c of x_{i+1}
  const double* dev_xn = nullptr;
  double* host_xn = nullptr;
};

#define RET_IF(x)            \
  do {                       \
    int _s = (x);            \
    if (_s != AA_OK) return _s; \
  } while (0)

// One QRAdd (with the fused QRDelete when the window is full) and, unless
// commit_only, the LSP solve and the x update.  mode: 0 = aa_step, 1 = aa_test_qradd.
int run_step(aa_ctx* c, const double* x, const double* g, double* xn, const double* vext,
             const ChunkPlan* cp = nullptr) {
  const bool ext = vext != nullptr;
  const int V = c->variant;
  const bool recycle = (c->mi == c->m);
  const int k = recycle ? c->m - 1 : c->mi;
  const int c_in = recycle ? c->m : k;
  int dg_slot;
  if (recycle) {
    dg_slot = c->dg_head;
    c->dg_head = (c->dg_head + 1) % c->m;
  } else {
    dg_slot = (c->dg_head + c->mi) % c->m;
  }
  const bool reortho = (V == V_DCGS2) && k >= 2 && (k + 1 > c->dcgs2_cond);
  const bool has_x = (V == V_ICWY && k >= 2) || (V == V_DCGS2 && reortho);
  // ICWY T update after QRDelete: the paper's Gram rebuild, unless SMALL (precomputed by K4)
  const int gram = (V == V_ICWY && recycle && k >= 2 && c->icwy_merged != 2) ? 1 : 0;
  const K1Layout L = K1Layout::make(k, has_x, gram != 0);
  c->ar_last = 0;
  c->sp_last = 0;
  for (int i = 0; i < 5; ++i) c->logical_last[i] = 0;

  KParams p = base_params(c);
  p.red_words0 = L.words;
  p.k = k;
  p.c_in = c_in;
  p.recycle = recycle ? 1 : 0;
  p.has_x = has_x ? 1 : 0;
  p.gram = gram;
  p.reortho = reortho ? 1 : 0;
  p.beta_on = (c->beta != 1.0 && !ext) ? 1 : 0;
  p.flags = ext ? F_EXT_DF : 0;

  // ---------------- K1: prologue + QRDelete rotation + pass-1 multi-dot
  int k1_ar[4];
  int k1_pre = 0;   // K1's spare CTA computed the early rotations of the next QRDelete
  {
    KParams q = p;
    q.op = OP_K1;
    Inputs in;
    in.block(0, 0, c_in);                 // Q_0 .. Q_{c_in-1}
    if (ext) {
      in.vector(vext, true);              // Delta f supplied by the caller
      in.vector(vext, true);
    } else {
      in.vector(x, true);
      in.vector(g, true);
      in.vector(c->fp, false);
      in.vector(c->gp, false);
    }
    q.dg_out = dgcol(c, dg_slot);
    q.words = L.words;
    q.red_slot = 0;
    // K1 output path: per-thread coalesced stores (default) or TMA stores from the stage
    // (AA_K1_STORE=1).  Measured A/B on B200 (profiles/r02/k1_store_ab/): equal at m = 20 and 50,
    // 6-8 % slower at m = 5 / 10 (two CTAs per SM), so the stores stay per-thread.
    static const int k1_store = getenv("AA_K1_STORE") ? atoi(getenv("AA_K1_STORE")) : 0;
    q.k1_tmastore = ext ? 0 : k1_store;
    // the ICWY correction-matrix update after QRDelete is its own reduction
    if (gram && L.n_gram > 0 && !c->icwy_merged) {
      k1_ar[0] = L.off_gram; k1_ar[1] = L.n_gram; k1_ar[2] = 0; k1_ar[3] = L.off_gram;
    } else {
      k1_ar[0] = 0; k1_ar[1] = L.words; k1_ar[2] = 0; k1_ar[3] = 0;
    }
    if (!cp) {
      plan_ar(c, q, k1_ar[0], k1_ar[1], k1_ar[2], k1_ar[3]);
      q.k1_pre = (k >= 3) ? 1 : 0;   // launch_inst keeps it only if a spare CTA exists
      RET_IF(launch_op<OP_K1>(c, q, in, 0));
      k1_pre = q.k1_pre;
    } else {
      // row chunks: each launch waits only for its own chunk's copies; the reduction slot
      // accumulates over the chunks (in order); only the last one exchanges
      for (int ci = 0; ci < cp->nc; ++ci) {
        KParams qc = q;
        qc.rbeg = cp->b[ci];
        qc.n = cp->b[ci + 1];
        qc.chunk_first = (ci == 0);
        qc.chunk_last = (ci == cp->nc - 1);
        if (qc.chunk_last) plan_ar(c, qc, k1_ar[0], k1_ar[1], k1_ar[2], k1_ar[3]);
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, cp->evH[ci], 0));
        RET_IF(launch_op<OP_K1>(c, qc, in, 0));
      }
    }
  }
  RET_IF(post_ar(c, c->red, k1_ar[0], k1_ar[1], k1_ar[2], k1_ar[3]));
  // ---------------- K2: the rest of QRAdd
  int final_slot = 0;
  if (k >= 1) {
    KParams q = p;
    if (V == V_ICWY || V == V_DCGS2) {
      q.op = (V == V_ICWY) ? OP_K2_ICWY : OP_K2_DCGS2;
      Inputs in;
      in.block(0, 0, k + 1);              // Q_0 .. Q_{k-1}, Delta f (slot k)
      in.vector(c->fp, false);            // f_i
      q.words = 2;
      q.red_slot = 1;
      plan_ar(c, q, 0, 2, 0, 0);
      if (V == V_ICWY) RET_IF(launch_op<OP_K2_ICWY>(c, q, in, 1));
      else RET_IF(launch_op<OP_K2_DCGS2>(c, q, in, 1));
      RET_IF(post_ar(c, c->red + LRED, 0, 2, 0, 0));
      final_slot = 1;
    } else if (V == V_CGS2) {
      q.op = OP_K2A_CGS2;
      Inputs in;
      in.block(0, 0, k + 1);
      q.words = k;
      q.red_slot = 1;
      plan_ar(c, q, 0, k, 0, 0);
      RET_IF(launch_op<OP_K2A_CGS2>(c, q, in, 1));
      RET_IF(post_ar(c, c->red + LRED, 0, k, 0, 0));
      KParams q2 = p;
      q2.op = OP_K2B_CGS2;
      Inputs in2;
      in2.block(0, 0, k + 1);
      in2.vector(c->fp, false);
      q2.words = 2;
      q2.red_slot = 2;
      plan_ar(c, q2, 0, 2, 0, 0);
      RET_IF(launch_op<OP_K2B_CGS2>(c, q2, in2, 1));
      RET_IF(post_ar(c, c->red + 2 * LRED, 0, 2, 0, 0));
      final_slot = 2;
    } else {  // MGS: k dependent passes
      for (int j = 1; j <= k; ++j) {
        KParams q2 = p;
        q2.op = OP_K2_MGS;
        q2.mgs_j = j;
        Inputs in;
        in.vector(qcol(c, j - 1), false);
        in.vector(qcol(c, k), false);
        in.vector((j < k) ? qcol(c, j) : c->fp, false);
        q2.words = (j < k) ? 1 : 2;
        q2.red_slot = j;
        plan_ar(c, q2, 0, q2.words, 0, 0);
        RET_IF(launch_op<OP_K2_MGS>(c, q2, in, 1));
        RET_IF(post_ar(c, c->red + (size_t)j * LRED, 0, q2.words, 0, 0));
      }
      final_slot = k;
    }
  }
  // ---------------- K4: gamma + x update + commit
  {
    KParams q = p;
    q.op = OP_K4;
    q.k1_pre = k1_pre;
    q.final_slot = final_slot;
    q.words = 1;
    Inputs in;
    if (ext) {
      q.n = 0;
      q.flags |= F_COMMIT_ONLY;
    } else {
      // the Delta G window (oldest first) is a ring: at most two contiguous slot ranges
      const int first = c->dg_head, cnt = k + 1;
      const int c1 = std::min(cnt, c->m - first);
      in.block(1, first, c1);
      in.block(1, 0, cnt - c1);
      if (q.beta_on) in.block(0, 0, k + 1);
      in.vector(g, true);
      in.vector(x, true);
      if (q.beta_on) in.vector(c->fp, false);
      q.x_out = xn;
    }
    if (!cp || ext) {
      RET_IF(launch_op<OP_K4>(c, q, in, 2));
    } else {
      // row chunks: x_{i+1} chunk c goes back to the host as soon as K4 has written it
      for (int ci = 0; ci < cp->nc; ++ci) {
        KParams qc = q;
        qc.rbeg = cp->b[ci];
        qc.n = cp->b[ci + 1];
        qc.chunk_first = (ci == 0);
        qc.chunk_last = (ci == cp->nc - 1);
        RET_IF(launch_op<OP_K4>(c, qc, in, 2));
        CUDA_TRY(c, cudaEventRecord(cp->evK[ci], c->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(cp->cs, cp->evK[ci], 0));
        const size_t off = (size_t)cp->b[ci], cnt = (size_t)(cp->b[ci + 1] - cp->b[ci]);
        CUDA_TRY(c, cudaMemcpyAsync(cp->host_xn + off, cp->dev_xn + off, cnt * sizeof(double),
                                    cudaMemcpyDeviceToHost, cp->cs));
      }
    }
  }
  // CONV_NORM = IMMEDIATE: ||x_{i+1} - x_i||^2 summed over ranks now (Alg. 1 l.8 every step)
  if (!ext && c->conv_norm == 1 && c->nranks > 1) {
    double* d2 = &c->st->dx2_global;
    CUDA_TRY(c, cudaMemcpyAsync(d2, &c->st->dx2_local, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    RET_IF(allreduce(c, d2, 1));
    c->sp_last++;
  }
  c->ver ^= 1;
  c->mi = k + 1;
  // ---------------- ledger (paper's logical counts)
  int add;
  if (k == 0) add = 1;
  else if (V == V_MGS) add = k + 1;
  else if (V == V_CGS2) add = 3;
  else add = 2;
  c->logical_last[AA_PH_QRADD] = add;
  c->logical_last[AA_PH_QRDELETE] = (V == V_ICWY && recycle && c->icwy_merged != 2) ? 1 : 0;
  if (!ext) {
    c->logical_last[AA_PH_LSP_RHS] = 1;
    c->logical_last[AA_PH_NORM] = (c->conv_norm == 2) ? 0 : 1;
  }
  for (int i = 0; i < 5; ++i) c->logical[i] += c->logical_last[i];
  // the library asserts its schedule against the paper's count: the physical
  // global reductions of this step are QRAdd's (the printed formula), plus ICWY's delete
  // reduction when it is issued on its own and is non-empty (A6), plus the convergence norm
  // when CONV_NORM = IMMEDIATE on several ranks; the LSP right-hand side and the lagged norm
  // ride in these (A14, A15)
  {
    const int want = add + ((V == V_ICWY && gram && L.n_gram > 0 && !c->icwy_merged) ? 1 : 0) +
                     ((!ext && c->conv_norm == 1 && c->nranks > 1) ? 1 : 0);
    if (c->sp_last != want) {
      fprintf(stderr, "libaa: schedule issued %d global reductions, the paper's count is %d (variant %d, k %d)\n",
              c->sp_last, want, V, k);
      return fail(c, AA_ERR_STATE);
    }
  }
  return AA_OK;
}

// aa_step on the handle's staging buffers with the row-chunked K1 / K4 of aa_step_host
int aa_step_chunked(aa_ctx* h, const ChunkPlan* cp) {
  int rc;
  {
    EvScope ev(h, 4);
    rc = run_step(h, h->hx, h->hg, h->hxn, nullptr, cp);
  }
  if (rc == AA_OK) h->iter++;
  return rc;
}

int check_handle(aa_handle_t h) {
  if (!h) return AA_ERR_ARG;
  if (h->failed != AA_OK) return h->failed;
  return AA_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* aa_status_string(int s) {
  switch (s) {
    case AA_OK: return "ok";
    case AA_ERR_ARG: return "invalid argument";
    case AA_ERR_STATE: return "invalid state for this call";
    case AA_ERR_CUDA: return "CUDA error";
    case AA_ERR_NCCL: return "NCCL error or NCCL unavailable";
    case AA_ERR_NOMEM: return "device allocation failed";
    case AA_ERR_BREAKDOWN: return "QR breakdown (new column numerically dependent)";
    default: return "unknown status";
  }
}

int aa_comm_unique_id(void* id128) {
  if (!id128) return AA_ERR_ARG;
  if (!nccl().ok) return AA_ERR_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != 0) return AA_ERR_NCCL;
  memcpy(id128, &id, sizeof(id));
  return AA_OK;
}

static int create_impl(aa_handle_t* out, int64_t n_local, int m, int qr_variant, int rank, int nranks,
                       const void* id128, void* borrowed_comm, void* cuda_stream) {
  if (!out || n_local < 1 || m < 1 || m > MMAX || qr_variant < 0 || qr_variant > 3 || nranks < 1 ||
      rank < 0 || rank >= nranks || (nranks > 1 && !id128 && !borrowed_comm))
    return AA_ERR_ARG;
  *out = nullptr;
  aa_ctx* c = new aa_ctx();
  c->n = n_local;
  c->ld = (n_local + 255) / 256 * 256;
  c->n_global = n_local * nranks;
  c->m = m;
  c->variant = qr_variant;
  c->rank = rank;
  c->nranks = nranks;
  auto bail = [&](int code) {
    aa_destroy(c);
    return code;
  };
  if (cudaGetDevice(&c->device) != cudaSuccess) return bail(AA_ERR_CUDA);
  if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess)
    return bail(AA_ERR_CUDA);
  // NULL = the CUDA legacy default stream (what torch reports as stream 0)
  c->stream = (cudaStream_t)cuda_stream;
  c->own_stream = false;
  const size_t vbytes = (size_t)c->ld * sizeof(double);
  if (cudaHostAlloc(&c->bd_host, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->bd_dev), c->bd_host, 0) != cudaSuccess) {
    cudaGetLastError();
    c->bd_host = nullptr;
    return bail(AA_ERR_NOMEM);
  }
  *reinterpret_cast<volatile int*>(c->bd_host) = 0;
  if (cudaMalloc(&c->Q, vbytes * m) != cudaSuccess || cudaMalloc(&c->DG, vbytes * m) != cudaSuccess ||
      cudaMalloc(&c->fp, vbytes) != cudaSuccess || cudaMalloc(&c->gp, vbytes) != cudaSuccess ||
      cudaMalloc(&c->st, sizeof(SmallState)) != cudaSuccess ||
      cudaMalloc(&c->red, sizeof(double) * LRED * NSLOT) != cudaSuccess ||
      cudaMalloc(&c->part, sizeof(double) * LRED * 2 * c->sms) != cudaSuccess) {
    cudaGetLastError();
    return bail(AA_ERR_NOMEM);
  }
  // zero the padded rows once (they are read, never used, by the bulk copies)
  if (cudaMemset(c->Q, 0, vbytes * m) != cudaSuccess || cudaMemset(c->DG, 0, vbytes * m) != cudaSuccess ||
      cudaMemset(c->fp, 0, vbytes) != cudaSuccess || cudaMemset(c->gp, 0, vbytes) != cudaSuccess ||
      cudaMemset(c->red, 0, sizeof(double) * LRED * NSLOT) != cudaSuccess ||
      cudaMemset(c->st, 0, sizeof(SmallState)) != cudaSuccess)
    return bail(AA_ERR_CUDA);
  if (nranks > 1 && borrowed_comm) {
    if (!nccl().ok) {
      fprintf(stderr, "libaa: libnccl.so.2 could not be loaded (dlopen)\n");
      return bail(AA_ERR_NCCL);
    }
    c->comm = (ncclComm_t)borrowed_comm;
    c->own_comm = false;
  } else if (nranks > 1) {
    if (!nccl().ok) {
      fprintf(stderr, "libaa: libnccl.so.2 could not be loaded (dlopen)\n");
      return bail(AA_ERR_NCCL);
    }
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    const ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
    if (r != 0) {
      fprintf(stderr, "libaa: ncclCommInitRank(rank %d of %d) failed: %d %s\n", rank, nranks, (int)r,
              nccl().GetErrorString ? nccl().GetErrorString(r) : "");
      c->comm = nullptr;
      return bail(AA_ERR_NCCL);
    }
    c->own_comm = true;
  }
  if (nranks > 1) {
    // n_global = sum of the ranks' n_local (collective, once): the default breakdown threshold
    // eps_a = 10 eps sqrt(n_global) must be the same on every rank (reading A12), including
    // uneven shards
    double* tmp = c->red + (size_t)(NSLOT - 1) * LRED;
    double nl = (double)n_local, ng = 0.0;
    if (cudaMemcpy(tmp, &nl, sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) return bail(AA_ERR_CUDA);
    if (nccl().AllReduce(tmp, tmp, 1, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0) return bail(AA_ERR_NCCL);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess ||
        cudaMemcpy(&ng, tmp, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return bail(AA_ERR_CUDA);
    c->n_global = (int64_t)ng;
  }
  *out = c;
  return AA_OK;
}

// Fused-allreduce setup (collective): one device buffer per rank [header][mailbox], its
// CUDA IPC handle all-gathered over the handle's NCCL communicator, peers' buffers
// opened with cudaIpcOpenMemHandle (NVLink P2P within the node).  Every rank takes part in
// both collectives whatever happened locally (a rank that failed sends a dummy handle and a
// "failed" mark), and one allreduce of the failure count decides for all: every rank enables
// the fused exchange, or every rank keeps ncclAllReduce (no rank is left waiting in a
// collective its peers skipped, and no rank exchanges with a peer that is not listening).
static int fused_setup(aa_ctx* c) {
  // Any failure here leaves the handle usable with ncclAllReduce (not sticky).
  if (c->nranks > MAX_RANKS || !nccl().AllGather) return AA_ERR_ARG;
  // mailbox: [seq parity][source rank][LRED words][2 tagged halves] of 8 bytes (low-latency protocol)
  const size_t bytes = kFlagBytes + (size_t)2 * c->nranks * LRED * 2 * sizeof(unsigned long long);
  struct Entry {
    cudaIpcMemHandle_t h;
    int ok;
    int pad[15];
  };
  static_assert(sizeof(Entry) * MAX_RANKS <= sizeof(double) * LRED, "handle exchange fits one slot");
  // the exchange buffer is a reduction slot allocated at aa_create (no allocation that could fail here)
  char* dh = reinterpret_cast<char*>(c->red + (size_t)(NSLOT - 1) * LRED);
  double* dflag = c->red + (size_t)(NSLOT - 2) * LRED;
  Entry mine;
  memset(&mine, 0, sizeof(mine));
  mine.ok = cudaMalloc(&c->xbuf, bytes) == cudaSuccess && cudaMemset(c->xbuf, 0, bytes) == cudaSuccess &&
            cudaIpcGetMemHandle(&mine.h, c->xbuf) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  if (!mine.ok) cudaGetLastError();
  std::vector<Entry> all(c->nranks);
  auto release = [&]() {
    for (int r = 0; r < MAX_RANKS; ++r) {
      if (c->peer_base[r] && c->peer_base[r] != c->xbuf) cudaIpcCloseMemHandle(c->peer_base[r]);
      c->peer_base[r] = nullptr;
    }
    if (c->xbuf) cudaFree(c->xbuf);
    c->xbuf = nullptr;
    cudaGetLastError();
  };
  if (cudaMemcpy(dh + sizeof(Entry) * c->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice) != cudaSuccess ||
      nccl().AllGather(dh + sizeof(Entry) * c->rank, dh, sizeof(Entry), 0 /*ncclInt8*/, c->comm, c->stream) != 0 ||
      cudaStreamSynchronize(c->stream) != cudaSuccess ||
      cudaMemcpy(all.data(), dh, sizeof(Entry) * c->nranks, cudaMemcpyDeviceToHost) != cudaSuccess) {
    // the communicator or the device itself failed: peers see the same NCCL failure
    release();
    fprintf(stderr, "libaa: fused NVLink allreduce set-up failed in the handle exchange\n");
    return AA_ERR_NCCL;
  }
  bool ok = true;
  for (int r = 0; r < c->nranks; ++r) ok = ok && all[r].ok;
  for (int r = 0; r < c->nranks && ok; ++r) {
    if (r == c->rank) {
      c->peer_base[r] = c->xbuf;
    } else if (cudaIpcOpenMemHandle(&c->peer_base[r], all[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      c->peer_base[r] = nullptr;
      cudaGetLastError();
      ok = false;
    }
  }
  // agree: the number of ranks that could not open every peer
  double fails = ok ? 0.0 : 1.0;
  if (cudaMemcpy(dflag, &fails, sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      nccl().AllReduce(dflag, dflag, 1, kNcclFloat64, kNcclSum, c->comm, c->stream) != 0 ||
      cudaStreamSynchronize(c->stream) != cudaSuccess ||
      cudaMemcpy(&fails, dflag, sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
    release();
    return AA_ERR_NCCL;
  }
  if (fails > 0.0) {
    release();
    fprintf(stderr, "libaa: fused NVLink allreduce unavailable on %g rank(s); every rank keeps ncclAllReduce\n",
            fails);
    return AA_ERR_CUDA;
  }
  return AA_OK;
}

int aa_create(aa_handle_t* out, int64_t n_local, int m, int qr_variant, int rank, int nranks,
              const void* id128, void* cuda_stream) {
  return create_impl(out, n_local, m, qr_variant, rank, nranks, id128, nullptr, cuda_stream);
}

int aa_create_with_comm(aa_handle_t* out, int64_t n_local, int m, int qr_variant, int rank, int nranks,
                        void* nccl_comm, void* cuda_stream) {
  if (nranks > 1 && !nccl_comm) return AA_ERR_ARG;
  return create_impl(out, n_local, m, qr_variant, rank, nranks, nullptr, nccl_comm, cuda_stream);
}

int aa_set_option(aa_handle_t h, int opt, double val) {
  RET_IF(check_handle(h));
  switch (opt) {
    case AA_OPT_DAMPING_BETA:
      if (!(val > 0.0 && val <= 1.0)) return AA_ERR_ARG;
      h->beta = val;
      return AA_OK;
    case AA_OPT_ICWY_DELETE:
      if (val != 0.0 && val != 1.0 && val != 2.0) return AA_ERR_ARG;
      // SMALL needs the post-delete T precomputed by the previous K4: choose it before aa_init
      if (val == 2.0 && h->icwy_merged != 2 && h->inited) return AA_ERR_STATE;
      h->icwy_merged = (int)val;
      return AA_OK;
    case AA_OPT_DCGS2_COND:
      if (val != 2.0 && val != 3.0) return AA_ERR_ARG;
      h->dcgs2_cond = (int)val;
      return AA_OK;
    case AA_OPT_DCGS2_RSCALE:
      if (val != 0.0 && val != 1.0) return AA_ERR_ARG;
      h->dcgs2_rscale = (int)val;
      return AA_OK;
    case AA_OPT_BREAKDOWN_EPS:
      if (!(val >= 0.0)) return AA_ERR_ARG;
      h->eps_a = val;
      return AA_OK;
    case AA_OPT_PROFILE:
      h->profile = val != 0.0;
      return AA_OK;
    case AA_OPT_N_GLOBAL:
      if (!(val >= 1.0)) return AA_ERR_ARG;
      h->n_global = (int64_t)val;
      return AA_OK;
    case AA_OPT_FUSED_ALLREDUCE:
      if (val != 0.0 && val != 1.0) return AA_ERR_ARG;
      if (val == 1.0 && h->nranks > 1 && !h->xbuf) {
        const int rc = fused_setup(h);   // collective; on failure NCCL stays in use
        if (rc != AA_OK) return rc;
      }
      h->fused = (int)val;
      return AA_OK;
    case AA_OPT_CONV_NORM:
      if (val != 0.0 && val != 1.0 && val != 2.0) return AA_ERR_ARG;
      h->conv_norm = (int)val;
      return AA_OK;
    case AA_OPT_DETERMINISTIC:
      if (val != 0.0 && val != 1.0) return AA_ERR_ARG;
      if (val == 1.0 && !h->det) {
        // every rank's rows in whole DET_ROWS chunks (so chunks sit at the same global rows for
        // every rank count); the chunk partials and the all-gather buffer are allocated here
        if (h->n % DET_ROWS != 0) return AA_ERR_ARG;
        const size_t chunks = (size_t)(h->n / DET_ROWS);
        if (cudaMalloc(&h->part_det, sizeof(double) * LRED * chunks) != cudaSuccess ||
            (h->nranks > 1 && cudaMalloc(&h->xgather, sizeof(double) * LRED * h->nranks) != cudaSuccess)) {
          cudaGetLastError();
          cudaFree(h->part_det);
          h->part_det = nullptr;
          return AA_ERR_NOMEM;
        }
      }
      h->det = (int)val;
      return AA_OK;
    default:
      return AA_ERR_ARG;
  }
}

static void init_small(SmallState* hs, bool keep_scalars, const SmallState* old) {
  memset(hs, 0, sizeof(SmallState));
  for (int v = 0; v < 2; ++v)
    for (int j = 0; j < MMAX; ++j) hs->f[v].scale[j] = 1.0;
  hs->rratio_min = DBL_MAX;
  if (keep_scalars && old) {
    hs->dx2_local = old->dx2_local;
    hs->f2 = old->f2;
    hs->breakdown_count = old->breakdown_count;
  }
}

static int reset_small(aa_ctx* c) {
  SmallState* hs = new SmallState();
  init_small(hs, false, nullptr);
  cudaError_t e = cudaMemcpyAsync(c->st, hs, sizeof(SmallState), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  delete hs;
  if (e != cudaSuccess) return fail(c, AA_ERR_CUDA);
  c->ver = 0;
  return AA_OK;
}

// K1's two forms for 7..22 columns: the fused row pass (dots in registers,
// the default) and the split one (rotated tile back to shared memory, block multi-dot).  Which
// is faster depends on the B200: same-build A/Bs at the bench's configuration gave fused 6.06
// vs split 6.72-6.85 ms on three runs of one box type, 6.42 vs 6.11 ms on another
// (profiles/r02/k1_fused_vs_split_ab*.txt, k1_form_ab.txt), and a short timing trial on the
// handle's own buffers (AA_K1_FORM=auto: both forms, three launches each, at aa_init) picked
// the split form on the box where the fused one is 11 % faster in sustained runs -- the
// power-capped clocks of a long run are not those of a short burst.  So the fused form is the
// default; AA_K1_FORM=split|auto selects otherwise.  Both forms give results inside the same
// tolerances; the choice only changes the summation order of pass 1.
static int k1_form_trial(aa_ctx* c) {
  c->k1_split = 0;
  const char* env = getenv("AA_K1_FORM");
  if (env && !strcmp(env, "split")) c->k1_split = 1;
  if (!env || strcmp(env, "auto")) return AA_OK;
  const int k = c->m - 1;
  const int ncw = (k + 2 + NWARP - 1) / NWARP;
  if (c->det || ncw < 2 || ncw > 3 || c->n < (1 << 20)) return AA_OK;
  static std::map<std::tuple<int, int, int64_t>, int> cache;
  const auto key = std::make_tuple(c->device, c->m, c->n);
  auto it = cache.find(key);
  if (it != cache.end()) {
    c->k1_split = it->second;
    return AA_OK;
  }
  // a recycle-shaped K1 on the handle's own buffers, made representative: distinct vectors
  // (Delta G slots 1..4 as x, G(x), f_{i-1}, G(x_{i-1})), uniform data in Q and those slots,
  // nonzero rotations (the handle is empty: aa_init resets everything the trial touches)
  for (int j = 0; j < c->m; ++j) {
    aa_fill_uniform_kernel<<<c->sms * 8, 256, 0, c->stream>>>(qcol(c, j), c->n, 1000ull * j, -1.0, 2.0);
    aa_fill_uniform_kernel<<<c->sms * 8, 256, 0, c->stream>>>(dgcol(c, j), c->n, 777ull * j + 5, -1.0, 2.0);
  }
  {
    double cs[MMAX], sn[MMAX];
    for (int j = 0; j < MMAX; ++j) {
      cs[j] = 0.6;
      sn[j] = 0.8;
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->st->f[0].cs, cs, sizeof(cs), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->st->f[0].sn, sn, sizeof(sn), cudaMemcpyHostToDevice, c->stream));
  }
  KParams p = base_params(c);
  const K1Layout L = K1Layout::make(k, true, false);
  p.red_words0 = L.words;
  p.k = k;
  p.c_in = c->m;
  p.recycle = 1;
  p.has_x = 1;
  p.reortho = 1;
  p.op = OP_K1;
  p.dg_out = dgcol(c, 0);
  p.words = L.words;
  p.red_slot = 0;
  Inputs in;
  in.block(0, 0, c->m);
  for (int v = 1; v <= 4; ++v) in.vector(dgcol(c, v), false);
  cudaEvent_t e0, e1;
  CUDA_TRY(c, cudaEventCreate(&e0));
  CUDA_TRY(c, cudaEventCreate(&e1));
  float best[2] = {1e30f, 1e30f};
  for (int rep = 0; rep < 4; ++rep)
    for (int form = 0; form < 2; ++form) {
      c->k1_split = form;
      KParams q = p;
      CUDA_TRY(c, cudaEventRecord(e0, c->stream));
      RET_IF(launch_op<OP_K1>(c, q, in, 0));
      CUDA_TRY(c, cudaEventRecord(e1, c->stream));
      CUDA_TRY(c, cudaEventSynchronize(e1));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best[form]) best[form] = ms;   // rep 0 warms both forms up
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c->k1_split = (best[1] < best[0]) ? 1 : 0;
  cache[key] = c->k1_split;
  return AA_OK;
}

int aa_init(aa_handle_t h, const double* x0, const double* gx0, double* x1_out) {
  RET_IF(check_handle(h));
  if (!x0 || !gx0 || !x1_out) return AA_ERR_ARG;
  RET_IF(reset_small(h));
  RET_IF(k1_form_trial(h));
  RET_IF(reset_small(h));   // the trial used the reduction slots and the factor scratch
  *reinterpret_cast<volatile int*>(h->bd_host) = 0;
  if (h->eps_a < 0.0) h->eps_a = 10.0 * DBL_EPSILON * sqrt((double)h->n_global);
  const int grid = h->sms * 4;
  aa_init_kernel<<<grid, 256, 0, h->stream>>>(x0, gx0, x1_out, h->fp, h->gp, h->n);
  h->launches++;
  CUDA_TRY(h, cudaGetLastError());
  h->iter = 0;
  h->mi = 0;
  h->dg_head = 0;
  h->hxn_valid = false;
  h->inited = true;
  return AA_OK;
}

int aa_step(aa_handle_t h, const double* x_i, const double* gx_i, double* x_next) {
  RET_IF(check_handle(h));
  if (!h->inited) return AA_ERR_STATE;
  h->hxn_valid = false;   // (aa_step_host sets it again after its own call)
  // a breakdown seen by an earlier step (mapped pinned word, polled without blocking):
  // refuse until aa_reset.  One rank only: ranks could see the word at different times and
  // must not diverge in their collective call sequences; with nranks > 1 the breakdown is
  // surfaced by aa_stats (collective, after a synchronisation), and steps enqueued before
  // that degrade to gamma = 0 on every rank alike.
  if (h->nranks == 1 && *reinterpret_cast<volatile int*>(h->bd_host)) return AA_ERR_BREAKDOWN;
  if (!x_i || !gx_i || !x_next || !aligned16(x_i) || !aligned16(gx_i) || !aligned16(x_next))
    return AA_ERR_ARG;
  int rc;
  {
    EvScope ev(h, 4);
    rc = run_step(h, x_i, gx_i, x_next, nullptr);
  }
  if (rc == AA_OK) h->iter++;
  return rc;
}

int aa_step_host(aa_handle_t h, const double* x_i, const double* gx_i, double* x_next) {
  RET_IF(check_handle(h));
  if (!h->inited) return AA_ERR_STATE;
  if (!gx_i || !x_next) return AA_ERR_ARG;
  // the breakdown poll of aa_step, before anything changes: after aa_reset the caller retries
  // the same call (x_i = NULL still finds its device copy)
  if (h->nranks == 1 && *reinterpret_cast<volatile int*>(h->bd_host)) return AA_ERR_BREAKDOWN;
  // x_i = NULL: the x_{i+1} the previous aa_step_host returned, still on the device (the
  // staging buffers swap roles; only G(x_i) crosses PCIe on the way in)
  if (!x_i && !h->hxn_valid) return AA_ERR_STATE;
  const bool reuse_x = (x_i == nullptr);
  if (reuse_x) std::swap(h->hx, h->hxn);
  h->hxn_valid = false;
  const size_t vb = (size_t)h->n * sizeof(double);
  if (!h->hx || !h->hg || !h->hxn) {
    if ((!h->hx && cudaMalloc(&h->hx, vb) != cudaSuccess) || (!h->hg && cudaMalloc(&h->hg, vb) != cudaSuccess) ||
        (!h->hxn && cudaMalloc(&h->hxn, vb) != cudaSuccess)) {
      cudaGetLastError();
      // all or nothing: a later call retries the allocation (not sticky)
      cudaFree(h->hx);
      cudaFree(h->hg);
      cudaFree(h->hxn);
      h->hx = h->hg = h->hxn = nullptr;
      return AA_ERR_NOMEM;
    }
  }
  if (h->n < kChunkMinRows || h->mi == 0 || h->det) {
    if (!reuse_x) CUDA_TRY(h, cudaMemcpyAsync(h->hx, x_i, vb, cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(h, cudaMemcpyAsync(h->hg, gx_i, vb, cudaMemcpyHostToDevice, h->stream));
    RET_IF(aa_step(h, h->hx, h->hg, h->hxn));
    CUDA_TRY(h, cudaMemcpyAsync(x_next, h->hxn, vb, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    h->hxn_valid = true;
    return AA_OK;
  }
  // large n: chunked copies overlapped with K1 (uploads) and K4 (downloads)
  if (!h->cstream) {
    CUDA_TRY(h, cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < kMaxChunks; ++i) {
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->chunk_evH[i], cudaEventDisableTiming));
      CUDA_TRY(h, cudaEventCreateWithFlags(&h->chunk_evK[i], cudaEventDisableTiming));
    }
  }
  ChunkPlan cp;
  cp.nc = kMaxChunks;
  for (int i = 0; i <= cp.nc; ++i) cp.b[i] = (i == cp.nc) ? h->n : ((h->n * i / cp.nc) / 1024) * 1024;
  cp.cs = h->cstream;
  cp.evH = h->chunk_evH;
  cp.evK = h->chunk_evK;
  cp.dev_xn = h->hxn;
  cp.host_xn = x_next;
  // the copy stream must not overwrite the staging buffers before earlier work on the
  // handle's stream has finished with them
  CUDA_TRY(h, cudaEventRecord(h->chunk_evK[0], h->stream));
  CUDA_TRY(h, cudaStreamWaitEvent(h->cstream, h->chunk_evK[0], 0));
  for (int ci = 0; ci < cp.nc; ++ci) {
    const size_t off = (size_t)cp.b[ci], cnt = (size_t)(cp.b[ci + 1] - cp.b[ci]);
    if (!reuse_x)
      CUDA_TRY(h, cudaMemcpyAsync(h->hx + off, x_i + off, cnt * sizeof(double), cudaMemcpyHostToDevice, h->cstream));
    CUDA_TRY(h, cudaMemcpyAsync(h->hg + off, gx_i + off, cnt * sizeof(double), cudaMemcpyHostToDevice, h->cstream));
    CUDA_TRY(h, cudaEventRecord(h->chunk_evH[ci], h->cstream));
  }
  RET_IF(aa_step_chunked(h, &cp));
  CUDA_TRY(h, cudaStreamSynchronize(h->cstream));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->hxn_valid = true;
  return AA_OK;
}

int aa_delete_oldest(aa_handle_t h) {
  RET_IF(check_handle(h));
  if (!h->inited || h->mi == 0) return AA_ERR_STATE;
  const int V = h->variant;
  const int k = h->mi - 1;  // retained columns
  const int gram = (V == V_ICWY && k >= 2) ? 1 : 0;
  const int words = gram ? k * (k - 1) / 2 : 0;
  for (int i = 0; i < 5; ++i) h->logical_last[i] = 0;
  h->ar_last = 0;
  h->sp_last = 0;
  KParams p = base_params(h);
  p.red_words0 = words;
  p.k = k;
  p.c_in = h->mi;
  p.recycle = 1;
  p.gram = gram;
  p.flags = F_DELETE_ONLY;
  {
    KParams q = p;
    q.op = OP_K1;
    Inputs in;
    in.block(0, 0, h->mi);
    q.words = words;
    q.red_slot = 0;
    plan_ar(h, q, 0, V == V_ICWY ? words : 0, 0, 0);
    RET_IF(launch_op<OP_K1>(h, q, in, 0));
  }
  if (V == V_ICWY) RET_IF(post_ar(h, h->red, 0, words, 0, 0));
  {
    KParams q = p;
    q.op = OP_K4;
    q.n = 0;
    q.words = 1;
    q.flags |= F_COMMIT_ONLY;
    RET_IF(launch_op<OP_K4>(h, q, Inputs(), 2));
  }
  h->ver ^= 1;
  h->mi = k;
  h->dg_head = (h->dg_head + 1) % h->m;
  h->logical_last[AA_PH_QRDELETE] = (V == V_ICWY) ? 1 : 0;
  h->logical[AA_PH_QRDELETE] += h->logical_last[AA_PH_QRDELETE];
  return AA_OK;
}

int aa_test_qradd(aa_handle_t h, const double* v) {
  RET_IF(check_handle(h));
  if (!h->inited) return AA_ERR_STATE;
  if (!v || !aligned16(v)) return AA_ERR_ARG;
  return run_step(h, nullptr, nullptr, nullptr, v);
}

int aa_stats(aa_handle_t h, struct aa_stats* out, int flags) {
  if (!h || !out) return AA_ERR_ARG;
  memset(out, 0, sizeof(*out));
  out->loo = -1.0;
  out->iter = h->iter;
  out->m_i = h->mi;
  out->sync_points_last = h->sp_last;
  out->allreduce_last = h->ar_last;
  out->allreduce_total = h->ar_total;
  for (int i = 0; i < 5; ++i) {
    out->logical_sync[i] = h->logical[i];
    out->logical_sync_last[i] = h->logical_last[i];
  }
  struct {
    double dx2 = 0.0, f2 = 0.0, rmin = 0.0;
    int bd = 0, bdc = 0;
  } hs;
  int status = h->failed;
  if (status == AA_OK) {
    // only the scalar tail of SmallState (the factors stay on the device)
    constexpr size_t off = offsetof(SmallState, dx2_local);
    unsigned char tail[sizeof(SmallState) - off];
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy(tail, reinterpret_cast<unsigned char*>(h->st) + off, sizeof(tail), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      fprintf(stderr, "libaa: CUDA error %s in aa_stats\n", cudaGetErrorString(e));
      status = fail(h, AA_ERR_CUDA);
    } else {
      auto fld = [&](size_t o) { return tail + (o - off); };
      double dx2l, dx2g;
      int xto;
      memcpy(&dx2l, fld(offsetof(SmallState, dx2_local)), sizeof(double));
      memcpy(&dx2g, fld(offsetof(SmallState, dx2_global)), sizeof(double));
      memcpy(&hs.f2, fld(offsetof(SmallState, f2)), sizeof(double));
      memcpy(&hs.rmin, fld(offsetof(SmallState, rratio_min)), sizeof(double));
      memcpy(&hs.bd, fld(offsetof(SmallState, breakdown)), sizeof(int));
      memcpy(&hs.bdc, fld(offsetof(SmallState, breakdown_count)), sizeof(int));
      memcpy(&xto, fld(offsetof(SmallState, xchg_timeout)), sizeof(int));
      hs.dx2 = (h->conv_norm == 1 && h->nranks > 1) ? dx2g : dx2l;
      if (xto) {
        fprintf(stderr, "libaa: fused peer exchange timed out\n");
        status = fail(h, AA_ERR_NCCL);
      }
    }
  }
  // collective (nranks > 1): every rank contributes {lagged ||dx||^2 partial, error flag} to ONE
  // allreduce, so the ranks agree on the outcome and none is left waiting in a collective its
  // peers skipped; a rank whose communicator itself failed cannot take part
  bool peer_failed = false;
  if (h->nranks > 1 && h->comm && nccl().ok && !(h->failed == AA_ERR_NCCL && !h->fused)) {
    double* tmp = h->red + (size_t)(NSLOT - 1) * LRED;
    double v[2] = {(h->conv_norm == 0 && status == AA_OK) ? hs.dx2 : 0.0, status != AA_OK ? 1.0 : 0.0};
    cudaError_t e = cudaMemcpyAsync(tmp, v, sizeof(v), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess && nccl().AllReduce(tmp, tmp, 2, kNcclFloat64, kNcclSum, h->comm, h->stream) != 0) {
      status = fail(h, AA_ERR_NCCL);
      return status;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(v, tmp, sizeof(v), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return fail(h, AA_ERR_CUDA);
    if (h->conv_norm == 0) hs.dx2 = v[0];
    peer_failed = v[1] > 0.0;
  }
  if (status != AA_OK) return status;
  if (peer_failed) {
    fprintf(stderr, "libaa: a peer rank's handle failed\n");
    return fail(h, AA_ERR_NCCL);
  }
  out->f_norm = sqrt(hs.f2);
  out->dx_norm = (h->conv_norm == 2) ? -1.0 : sqrt(hs.dx2);
  out->r_ratio_min = hs.rmin;
  out->breakdown = hs.bd;
  out->breakdown_count = hs.bdc;
  if ((flags & AA_STATS_LOO) && h->mi >= 1) {
    KParams p = base_params(h);
    p.op = OP_GRAM;
    p.gram = 2;
    p.c_in = h->mi;
    Inputs in;
    in.block(0, 0, h->mi);
    const int words = h->mi * (h->mi + 1) / 2;
    p.words = words;
    p.red_slot = NSLOT - 1;
    RET_IF(launch_op<OP_GRAM>(h, p, in, 1));
    double* gbuf = h->red + (size_t)(NSLOT - 1) * LRED;
    if (h->nranks > 1) {
      ncclResult_t r = nccl().AllReduce(gbuf, gbuf, words, kNcclFloat64, kNcclSum, h->comm, h->stream);
      if (r != 0) return fail(h, AA_ERR_NCCL);
    }
    std::vector<double> gh(words);
    CUDA_TRY(h, cudaMemcpyAsync(gh.data(), gbuf, sizeof(double) * words, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    double s = 0.0;
    for (int i = 0; i < h->mi; ++i)
      for (int j = 0; j <= i; ++j) {
        const double g = gh[i * (i + 1) / 2 + j];
        s += (i == j) ? (1.0 - g) * (1.0 - g) : 2.0 * g * g;
      }
    out->loo = sqrt(s);
  }
  if (flags & AA_STATS_RESET) {
    for (int i = 0; i < 5; ++i) h->logical[i] = 0;
    h->ar_total = 0;
  }
  return hs.bd ? AA_ERR_BREAKDOWN : AA_OK;
}

int aa_reset(aa_handle_t h) {
  RET_IF(check_handle(h));
  if (!h->inited) return AA_ERR_STATE;
  // empty the window; f_{i-1} and G(x_{i-1}) are kept, so the next aa_step takes the
  // i = 1 branch of Alg. 2 with Delta f = f_i - f_{i-1}
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  h->mi = 0;
  h->dg_head = 0;
  SmallState* old = new SmallState();
  SmallState* hs = new SmallState();
  cudaError_t e = cudaMemcpy(old, h->st, sizeof(SmallState), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) {
    init_small(hs, true, old);   // keep ||dx||^2 / ||f||^2 of the last step
    e = cudaMemcpy(h->st, hs, sizeof(SmallState), cudaMemcpyHostToDevice);
  }
  delete old;
  delete hs;
  if (e != cudaSuccess) return fail(h, AA_ERR_CUDA);
  *reinterpret_cast<volatile int*>(h->bd_host) = 0;
  h->ver = 0;
  return AA_OK;
}

int aa_destroy(aa_handle_t h) {
  if (!h) return AA_ERR_ARG;
  cudaStreamSynchronize(h->stream);
  for (auto& e : h->evs) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (int r = 0; r < MAX_RANKS; ++r)
    if (h->peer_base[r] && h->peer_base[r] != h->xbuf) cudaIpcCloseMemHandle(h->peer_base[r]);
  cudaFree(h->xbuf);
  cudaFree(h->tl);
  if (h->cstream) {
    cudaStreamDestroy(h->cstream);
    for (int i = 0; i < 8; ++i) {
      cudaEventDestroy(h->chunk_evH[i]);
      cudaEventDestroy(h->chunk_evK[i]);
    }
  }
  if (h->comm && h->own_comm && nccl().ok) nccl().CommDestroy(h->comm);
  cudaFree(h->Q);
  cudaFree(h->DG);
  cudaFree(h->fp);
  cudaFree(h->gp);
  cudaFree(h->st);
  cudaFree(h->red);
  cudaFree(h->part);
  cudaFree(h->hx);
  cudaFree(h->hg);
  cudaFree(h->hxn);
  cudaFree(h->part_det);
  cudaFree(h->xgather);
  if (h->bd_host) cudaFreeHost(h->bd_host);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return AA_OK;
}

// ------------------------------------------------------------------ testing hooks
int aa_get_small(aa_handle_t h, double* R, double* T, double* gamma, double* scale) {
  RET_IF(check_handle(h));
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  SmallState* hs = new SmallState();
  cudaError_t e = cudaMemcpy(hs, h->st, sizeof(SmallState), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    delete hs;
    return fail(h, AA_ERR_CUDA);
  }
  const int m = h->m;
  const Factors& F = hs->f[h->ver];
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) {
      if (R) R[i + j * m] = F.R[i + j * MMAX];
      if (T) T[i + j * m] = F.T[i + j * MMAX];
    }
  if (gamma)
    for (int j = 0; j < h->mi; ++j) gamma[j] = F.gamma[j];
  if (scale)
    for (int j = 0; j < m; ++j) scale[j] = F.scale[j];
  delete hs;
  return AA_OK;
}

int aa_get_q(aa_handle_t h, double* q_out) {
  RET_IF(check_handle(h));
  if (!q_out) return AA_ERR_ARG;
  if (h->mi == 0) return AA_OK;
  aa_copy_q_kernel<<<h->sms * 4, 256, 0, h->stream>>>(h->Q, h->ld, h->st, h->ver, h->mi, q_out, h->n);
  h->launches++;
  CUDA_TRY(h, cudaGetLastError());
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  return AA_OK;
}

int aa_timings(aa_handle_t h, double* ms_out5, int64_t* counts5, int reset) {
  if (!h) return AA_ERR_ARG;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  for (auto& e : h->evs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    h->t_ms[e.cls] += ms;
    h->t_cnt[e.cls]++;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  h->evs.clear();
  for (int i = 0; i < 5; ++i) {
    if (ms_out5) ms_out5[i] = h->t_ms[i];
    if (counts5) counts5[i] = h->t_cnt[i];
    if (reset) {
      h->t_ms[i] = 0;
      h->t_cnt[i] = 0;
    }
  }
  return AA_OK;
}

int64_t aa_kernel_launches(aa_handle_t h) { return h ? h->launches : -1; }

int aa_test_timeline(aa_handle_t h, int enable, uint64_t* out384) {
  if (!h) return AA_ERR_ARG;
  if (enable && !h->tl) {
    CUDA_TRY(h, cudaMalloc(&h->tl, 384 * sizeof(unsigned long long)));
    CUDA_TRY(h, cudaMemset(h->tl, 0, 384 * sizeof(unsigned long long)));
  }
  if (!enable && h->tl) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    cudaFree(h->tl);
    h->tl = nullptr;
  }
  if (out384 && h->tl) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    CUDA_TRY(h, cudaMemcpy(out384, h->tl, 384 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  }
  return AA_OK;
}

int aa_test_exchange(aa_handle_t h, int words, int iters, double* us_fused, double* us_nccl) {
  RET_IF(check_handle(h));
  if (words < 1 || words > LRED || iters < 1) return AA_ERR_ARG;
  if (us_fused) *us_fused = -1.0;
  if (us_nccl) *us_nccl = -1.0;
  if (h->nranks == 1) return AA_OK;
  double* slot = h->red + (size_t)(NSLOT - 2) * LRED;
  if (us_fused && h->fused && h->xbuf) {
    KParams q = base_params(h);
    q.red = h->red;
    q.st = h->st;
    q.nranks = h->nranks;
    q.rank = h->rank;
    q.xseq = reinterpret_cast<unsigned long long*>(h->xbuf);
    for (int r = 0; r < h->nranks; ++r) q.pmbox[r] = (double*)((char*)h->peer_base[r] + kFlagBytes);
    q.lmbox = (double*)((char*)h->xbuf + kFlagBytes);
    unsigned long long* dns = nullptr;
    CUDA_TRY(h, cudaMalloc(&dns, sizeof(unsigned long long)));
    aa_xchg_bench_kernel<<<1, NT, 0, h->stream>>>(q, words, iters, dns);
    h->launches++;
    unsigned long long ns = 0;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&ns, dns, sizeof(ns), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(dns);
    CUDA_TRY(h, e);
    *us_fused = (double)ns * 1e-3 / iters;
  }
  if (us_nccl && h->comm && nccl().ok) {
    cudaEvent_t a, b;
    CUDA_TRY(h, cudaEventCreate(&a));
    CUDA_TRY(h, cudaEventCreate(&b));
    // one untimed call (lazy connection set-up), then iters back to back
    if (nccl().AllReduce(slot, slot, (size_t)words, kNcclFloat64, kNcclSum, h->comm, h->stream) != 0)
      return fail(h, AA_ERR_NCCL);
    CUDA_TRY(h, cudaEventRecord(a, h->stream));
    for (int it = 0; it < iters; ++it)
      if (nccl().AllReduce(slot, slot, (size_t)words, kNcclFloat64, kNcclSum, h->comm, h->stream) != 0)
        return fail(h, AA_ERR_NCCL);
    CUDA_TRY(h, cudaEventRecord(b, h->stream));
    CUDA_TRY(h, cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us_nccl = (double)ms * 1e3 / iters;
  }
  return AA_OK;
}

int aa_fill_uniform(double* out, int64_t n, int64_t offset, uint64_t seed, uint64_t stream, double lo,
                    double hi, void* cuda_stream) {
  if (!out || n < 0) return AA_ERR_ARG;
  if (n == 0) return AA_OK;
  const unsigned long long base = seed + stream * (1ull << 48) + (unsigned long long)offset;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return AA_ERR_CUDA;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  aa_fill_uniform_kernel<<<sms * 8, 256, 0, (cudaStream_t)cuda_stream>>>(out, n, base, lo, hi - lo);
  if (cudaGetLastError() != cudaSuccess) return AA_ERR_CUDA;
  return AA_OK;
}

int aa_build_info(char* buf, int len) {
  if (!buf || len <= 0) return AA_ERR_ARG;
  snprintf(buf, (size_t)len,
           "libaa sm_100a; NT=%d MMAX=%d LRED=%d MAXSTAGES=%d; TMA bulk staging, fp64 DMMA Gram", NT, MMAX,
           LRED, MAXSTAGES);
  return AA_OK;
}

}  // extern "C"
