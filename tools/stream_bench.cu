// stream_bench.cu — microbenchmark of multi-column streaming strategies on B200 (sm_100a).
// Reads `nin` fp64 columns of length n (column-major, ld = n padded), writes one output column
// (sum of inputs), reports GB/s of (nin + 1) * 8 * n bytes.  Used to pick libaa's engine design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(smem_u32(bar)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Strategy A: TMA 1D bulk per column per tile (libaa round-1 engine).
__global__ void __launch_bounds__(256) k_tma(const double* __restrict__ X, long long ld, int nin, long long n, int TR, int NS, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  double* st = (double*)(sm + 128);
  const int STR = TR + 4;
  const size_t sw = (size_t)nin * STR;
  long long ntiles = (n + TR - 1) / TR;
  long long cnt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](int s, long long t) {
    long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    uint32_t b = (rows * 8 + 15) & ~15;
    mbar_expect(&bars[s], b * nin);
    for (int i = 0; i < nin; ++i) bulk(st + s * sw + (size_t)i * STR, X + i * ld + r0, b, &bars[s]);
  };
  if (threadIdx.x == 0) for (int s = 0; s < NS && s < cnt; ++s) issue(s, blockIdx.x + (long long)s * gridDim.x);
  for (long long it = 0; it < cnt; ++it) {
    int s = it % NS; long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    mbar_wait(&bars[s], (it / NS) & 1);
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      double a = 0; const double* S = st + s * sw;
      for (int i = 0; i < nin; ++i) a += S[(size_t)i * STR + r];
      out[r0 + r] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0 && it + NS < cnt) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s, blockIdx.x + (it + NS) * gridDim.x); }
  }
}

// Strategy B: TMA with a dedicated producer warp and full/empty mbarriers (no CTA barrier).
__global__ void __launch_bounds__(288) k_tma_ws(const double* __restrict__ X, long long ld, int nin, long long n, int TR, int NS, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 16;
  double* st = (double*)(sm + 256);
  const int STR = TR + 4;
  const size_t sw = (size_t)nin * STR;
  long long ntiles = (n + TR - 1) / TR;
  long long cnt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (warp == 8) {
    if ((threadIdx.x & 31) == 0) {
      for (long long it = 0; it < cnt; ++it) {
        int s = it % NS;
        if (it >= NS) mbar_wait(&empty[s], ((it / NS) - 1) & 1);
        long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
        uint32_t b = (rows * 8 + 15) & ~15;
        mbar_expect(&full[s], b * nin);
        for (int i = 0; i < nin; ++i) bulk(st + s * sw + (size_t)i * STR, X + i * ld + r0, b, &full[s]);
      }
    }
    return;
  }
  for (long long it = 0; it < cnt; ++it) {
    int s = it % NS; long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    mbar_wait(&full[s], (it / NS) & 1);
    const double* S = st + s * sw;
    for (int r = threadIdx.x; r < rows; r += 256) {
      double a = 0;
      for (int i = 0; i < nin; ++i) a += S[(size_t)i * STR + r];
      out[r0 + r] = a;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
  }
}


// Strategy D: 1D bulk copies issued by lane 0 of EVERY warp (columns split over warps).
__global__ void __launch_bounds__(256) k_tma_mw(const double* __restrict__ X, long long ld, int nin, long long n, int TR, int NS, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  double* st = (double*)(sm + 128);
  const int STR = TR + 4;
  const size_t sw = (size_t)nin * STR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long ntiles = (n + TR - 1) / TR;
  long long cnt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 8); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](int s, long long t) {
    long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    uint32_t b = (rows * 8 + 15) & ~15;
    int c0 = warp * nin / 8, c1 = (warp + 1) * nin / 8;
    mbar_expect(&bars[s], b * (c1 - c0));
    for (int i = c0; i < c1; ++i) bulk(st + s * sw + (size_t)i * STR, X + i * ld + r0, b, &bars[s]);
  };
  if (lane == 0) for (int s = 0; s < NS && s < cnt; ++s) issue(s, blockIdx.x + (long long)s * gridDim.x);
  for (long long it = 0; it < cnt; ++it) {
    int s = it % NS; long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    mbar_wait(&bars[s], (it / NS) & 1);
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      double a = 0; const double* S = st + s * sw;
      for (int i = 0; i < nin; ++i) a += S[(size_t)i * STR + r];
      out[r0 + r] = a;
    }
    __syncthreads();
    if (lane == 0 && it + NS < cnt) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s, blockIdx.x + (it + NS) * gridDim.x); }
  }
}

// Strategy E: one 2D tensor-map TMA per tile (box TR x nin).
__global__ void __launch_bounds__(256) k_tma2d(const __grid_constant__ CUtensorMap tm, int nin, long long n, int TR, int NS, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  double* st = (double*)(sm + 128);
  const size_t sw = (size_t)nin * TR;
  long long ntiles = (n + TR - 1) / TR;
  long long cnt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](int s, long long t) {
    int r0 = (int)(t * TR);
    mbar_expect(&bars[s], (uint32_t)(TR * nin * 8));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(st + s * sw)), "l"(&tm), "r"(r0), "r"(0), "r"(smem_u32(&bars[s])) : "memory");
  };
  if (threadIdx.x == 0) for (int s = 0; s < NS && s < cnt; ++s) issue(s, blockIdx.x + (long long)s * gridDim.x);
  for (long long it = 0; it < cnt; ++it) {
    int s = it % NS; long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR; int rows = (int)min((long long)TR, n - r0);
    mbar_wait(&bars[s], (it / NS) & 1);
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
      double a = 0; const double* S = st + s * sw;
      for (int i = 0; i < nin; ++i) a += S[(size_t)i * TR + r];
      out[r0 + r] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0 && it + NS < cnt) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s, blockIdx.x + (it + NS) * gridDim.x); }
  }
}

// Strategy C: plain LDG.128 (2 rows per thread), grid-stride, columns unrolled by 8.
__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ X, long long ld, int nin, long long n, double* out) {
  long long npair = n / 2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npair; p += (long long)gridDim.x * blockDim.x) {
    double2 a = make_double2(0, 0);
    int i = 0;
    for (; i + 8 <= nin; i += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(X + (i + u) * ld) + p);
#pragma unroll
      for (int u = 0; u < 8; ++u) { a.x += v[u].x; a.y += v[u].y; }
    }
    for (; i < nin; ++i) { double2 v = __ldcs(reinterpret_cast<const double2*>(X + i * ld) + p); a.x += v.x; a.y += v.y; }
    reinterpret_cast<double2*>(out)[p] = a;
  }
}


int main(int argc, char** argv) {
  long long n = 20000000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int maxin = 64;
  long long ld = (n + 255) / 256 * 256;
  double *X, *out;
  CK(cudaMalloc(&X, sizeof(double) * ld * maxin));
  CK(cudaMalloc(&out, sizeof(double) * ld));
  CK(cudaMemset(X, 0, sizeof(double) * ld * maxin));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(k_tma_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(k_tma2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  auto report = [&](const char* name, int nin, float ms, const char* extra) {
    double gb = (nin + 1) * 8.0 * n / 1e9;
    printf("%-10s nin=%2d %-28s %8.3f ms %7.0f GB/s\n", name, nin, extra, ms, gb / (ms * 1e-3));
  };
  int nins[] = {4, 8, 22, 24, 54};
  for (int nin : nins) {
    for (int TR : {64, 128, 256}) {
      for (int NS : {2, 3, 4}) {
        for (int cps : {1, 2}) {
          size_t smem = 128 + (size_t)NS * nin * (TR + 4) * 8;
          if (smem * cps > 225 * 1024) continue;
          float ms;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_tma_mw<<<sms * cps, 256, smem>>>(X, ld, nin, n, TR, NS, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
          }
          cudaEventElapsedTime(&ms, e0, e1);
          char ex[64]; snprintf(ex, 64, "TR=%d NS=%d cps=%d", TR, NS, cps);
          report("tma_mw", nin, ms, ex);
          if (nin > 256) continue;
          CUtensorMap tm;
          cuuint64_t gdim[2] = {(cuuint64_t)n, (cuuint64_t)nin};
          cuuint64_t gstr[1] = {(cuuint64_t)(ld * 8)};
          cuuint32_t box[2] = {(cuuint32_t)TR, (cuuint32_t)nin};
          cuuint32_t es[2] = {1, 1};
          CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) { printf("encode failed %d (nin=%d TR=%d)\n", (int)r, nin, TR); continue; }
          size_t smem2 = 128 + (size_t)NS * nin * TR * 8;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_tma2d<<<sms * cps, 256, smem2>>>(tm, nin, n, TR, NS, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
          }
          cudaEventElapsedTime(&ms, e0, e1);
          report("tma2d", nin, ms, ex);
        }
      }
    }
  }
  return 0;
}
