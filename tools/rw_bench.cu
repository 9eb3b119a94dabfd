// rw_bench.cu — K1-shaped streaming: read NIN columns, write NOUT columns (fp64), B200.
// Compares direct STG stores against TMA bulk stores (cp.async.bulk.global.shared::cta),
// 1 vs 2 CTAs per SM.  GB/s counts (NIN + NOUT) * 8 * n bytes.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) { asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(su(b)), "r"(par) : "memory"); }
__device__ __forceinline__ void bulk_ld(void* d, const void* s, uint32_t n, uint64_t* b) { asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void bulk_st(void* g, const void* s, uint32_t n) { asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"(su(s)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// mode 0: STG from registers; mode 1: write results into the stage, TMA bulk store per column
__global__ void __launch_bounds__(256) k_rw(const double* __restrict__ X, double* Y, long long ld, int nin, int nout,
                                            long long n, int TR, int NS, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  double* st = (double*)(sm + 128);
  const size_t sw = (size_t)(nin + nout) * TR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long ntiles = (n + TR - 1) / TR;
  long long cnt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 8); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](int s, long long t) {
    long long r0 = t * TR;
    int c0 = warp * nin / 8, c1 = (warp + 1) * nin / 8;
    mbar_expect(&bars[s], TR * 8 * (c1 - c0));
    for (int i = c0; i < c1; ++i) bulk_ld(st + s * sw + (size_t)i * TR, X + i * ld + r0, TR * 8, &bars[s]);
  };
  if (lane == 0) for (int s = 0; s < NS && s < cnt; ++s) issue(s, blockIdx.x + (long long)s * gridDim.x);
  for (long long it = 0; it < cnt; ++it) {
    int s = it % NS; long long t = blockIdx.x + it * gridDim.x; long long r0 = t * TR;
    mbar_wait(&bars[s], (it / NS) & 1);
    double* S = st + s * sw;
    for (int r = threadIdx.x; r < TR; r += 256) {
      double carry = S[r];
      for (int j = 0; j < nout; ++j) {
        double q = S[(size_t)((j + 1) % nin) * TR + r];
        double o = fma(0.6, carry, 0.8 * q);
        carry = fma(-0.8, carry, 0.6 * q);
        if (mode == 0) Y[(size_t)j * ld + r0 + r] = o;
        else S[(size_t)(nin + j) * TR + r] = o;
      }
    }
    __syncthreads();
    if (mode == 1) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int j = warp; j < nout; j += 8) bulk_st(Y + (size_t)j * ld + r0, S + (size_t)(nin + j) * TR, TR * 8);
        bulk_commit();
        bulk_wait_read0();   // the stage may be reloaded only after the stores have read it
      }
      __syncthreads();
    }
    if (lane == 0 && it + NS < cnt) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(s, blockIdx.x + (it + NS) * gridDim.x); }
  }
}

int main() {
  long long n = 20000000;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  long long ld = (n + 1023) / 1024 * 1024;
  double *X, *Y;
  CK(cudaMalloc(&X, sizeof(double) * ld * 64));
  CK(cudaMalloc(&Y, sizeof(double) * ld * 64));
  CK(cudaMemset(X, 0, sizeof(double) * ld * 64));
  CK(cudaFuncSetAttribute(k_rw, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int nin, nout; } cfgs[] = {{24, 23}, {4, 1}, {21, 2}, {54, 53}};
  for (auto c : cfgs) {
    for (int mode = 0; mode < 2; ++mode)
      for (int TR : {64, 128, 256}) for (int NS : {2, 3, 4}) for (int cps : {1, 2}) {
        size_t smem = 128 + (size_t)NS * (c.nin + c.nout) * TR * 8;
        if (smem * cps > 226 * 1024 || smem > 225 * 1024) continue;
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          k_rw<<<sms * cps, 256, smem>>>(X, Y, ld, c.nin, c.nout, n, TR, NS, mode);
          cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
          cudaEventElapsedTime(&ms, e0, e1);
        }
        double gb = (c.nin + c.nout) * 8.0 * n / 1e9;
        printf("nin=%2d nout=%2d %s TR=%3d NS=%d cps=%d  %7.3f ms %6.0f GB/s\n", c.nin, c.nout, mode ? "tmaST" : "stg  ", TR, NS, cps, ms, gb / (ms * 1e-3));
      }
  }
  return 0;
}
