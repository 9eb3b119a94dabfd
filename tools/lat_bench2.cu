// Per-iteration cost of the primitives of the serial K3 loops (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double S[64 * 65];
  const int lane = threadIdx.x;
  for (int i = lane; i < 64 * 65; i += 32) S[i] = 1.0 + i * 1e-6;
  __syncwarp();
  double x = 1.0 + lane * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(__shfl_sync(0xffffffffu, x, i & 31), 0.999999, 1e-7);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) y = rsqrt(fma(y, y, 1.0));
  long long t2 = clock64();
  // pass: two loads, 4 fp ops, two stores, syncwarp (k3_rotate_sym's inner pattern, P <= 32)
  const double c = 0.8, s = 0.6;
  for (int j = 0; j < iters; ++j) {
    const int col = j & 31;
    const double a = S[lane + col * 65], b = S[lane + (col + 1) * 65];
    S[lane + col * 65] = c * a + s * b;
    S[lane + (col + 1) * 65] = -s * a + c * b;
    __syncwarp();
  }
  long long t3 = clock64();
  for (int j = 0; j < iters; ++j) {
    const int col = j & 31;
    const double a = S[lane + col * 65], b = S[lane + (col + 1) * 65];
    S[lane + col * 65] = c * a + s * b;
    S[lane + (col + 1) * 65] = -s * a + c * b;
  }
  long long t4 = clock64();
  for (int j = 0; j < iters; ++j) __syncwarp();
  long long t5 = clock64();
  out[lane] = x + y + S[lane];
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  const int it = 1000;
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(o, c, it);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("cycles/iter: shfl+dfma %.1f  rsqrt(fma) %.1f  smem pass+syncwarp %.1f  smem pass %.1f  syncwarp %.1f\n",
           h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it);
  }
  return 0;
}
