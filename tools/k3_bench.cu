// The K3 routines of aa_device.cuh in isolation (one working warp, shared memory), to
// compare with their cost inside the K4 kernel (tools/timeline_probe.py).  Launch shapes:
// 32 threads / small smem, 256 threads (warps 1..7 parked at a barrier), + 220 KB smem.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2110_09667_b200/csrc/aa_device.cuh"
using namespace aa;
__global__ void k3(double* cs, double* sn, double* g, long long* cyc, int K, const double* Rin) {
  extern __shared__ double smem[];
  double *R = smem, *W = R + MMAX * LDR, *c = W + MMAX * LDR, *gam = c + MMAX;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int j = 0; j < MMAX; ++j)
      for (int i = lane; i < MMAX; i += 32)
        R[i + j * LDR] = Rin ? Rin[i + j * MMAX] : ((i <= j) ? 1.0 / (1 + i + j) + (i == j) : 0.0);
    for (int i = lane; i < MMAX; i += 32) c[i] = 1.0 + i;
    __syncwarp();
    long long t0 = clock64();
    double* scs0 = gam + MMAX;
    double* ssn0 = scs0 + MMAX;
    k3_givens_delete<LDR>(R, K, scs0, ssn0);   // in place (as K4)
    long long t1 = clock64();
    k3_back_subst<LDR>(R, c, gam, K);
    long long t2 = clock64();
    k3_forward_unit_lower(W, c, K);
    long long t3 = clock64();
    // symmetric two-sided rotation (ICWY SMALL T update) on W viewed with LD = LDR
    for (int j = 0; j < K; ++j)
      for (int i = lane; i < K; i += 32) W[i + j * LDR] = (i == j) ? 1.0 : 0.01 * (1 + ((i + j) % 7));
    __syncwarp();
    double* scs = scs0;
    double* ssn = ssn0;
    for (int i = lane; i < K; i += 32) { cs[i] = scs[i]; sn[i] = ssn[i]; }
    __syncwarp();
    long long t4 = clock64();
    k3_rotate_sym<LDR>(W, K - 1, scs, ssn);
    long long t5 = clock64();
    if (lane < K) g[lane] = gam[lane] + c[lane];
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t5 - t4; }
  }
  __syncthreads();
}
int main(int argc, char** argv) {
  double *cs, *sn, *g; long long* c;
  double* Rin = nullptr;
  int Kfile = 0;
  if (argc > 2) {   // R (MMAX x MMAX fp64, column-major) from a file, and its K
    static double h[MMAX * MMAX];
    FILE* f = fopen(argv[1], "rb");
    if (!f || fread(h, sizeof(double), MMAX * MMAX, f) != MMAX * MMAX) { printf("bad R file\n"); return 1; }
    fclose(f);
    Kfile = atoi(argv[2]);
    cudaMalloc(&Rin, sizeof(h));
    cudaMemcpy(Rin, h, sizeof(h), cudaMemcpyHostToDevice);
  }
  cudaMalloc(&cs, 512); cudaMalloc(&sn, 512); cudaMalloc(&g, 512); cudaMalloc(&c, 64);  // 4 counters
  const int small = (2 * MMAX * LDR + 4 * MMAX) * 8, big = 220 * 1024;
  cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  struct { int thr, sm; const char* name; } shapes[] = {{32, small, "32thr/66KB"}, {256, small, "256thr/66KB"}, {256, big, "256thr/220KB"}};
  for (auto s : shapes)
    for (int K : {5, 20, 50}) {
      if (Kfile && K != 20) continue;
      if (Kfile) K = Kfile;
      long long h[4];
      for (int r = 0; r < 2; ++r) {
        k3<<<1, s.thr, s.sm>>>(cs, sn, g, c, K, Rin);
        cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
      }
      printf("%-13s K=%d cycles: givens %lld (%.0f/step)  back_subst %lld  fwd %lld  rotate_sym %lld  [%s]\n", s.name,
             K, h[0], h[0] / (double)(K - 1), h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
