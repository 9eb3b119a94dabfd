// Dependent-latency microbenchmark (one warp): DFMA chain, 1/x, sqrt, shared round trip,
// and the Givens step of k3_givens_delete in isolation.  Prints cycles per dependent op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double seed, int iters) {
  __shared__ double sm[64 * 64];
  const int lane = threadIdx.x;
  double x = seed + lane * 1e-3;
  for (int i = lane; i < 64 * 64; i += 32) sm[i] = 1.0 + i * 1e-6;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) y = 1.0 / (y + 1.0);
  long long t2 = clock64();
  double z = y + 2.0;
  for (int i = 0; i < iters; ++i) z = sqrt(z + 1.0);
  long long t3 = clock64();
  double w = z;
  for (int i = 0; i < iters; ++i) { sm[lane * 64] = w; __syncwarp(); w = sm[((lane + 1) & 31) * 64] * 1.0000001; __syncwarp(); }
  long long t4 = clock64();
  double u = w;
  for (int i = 0; i < iters; ++i) { sm[lane] = u; __syncwarp(); u = sm[(lane + 1) & 31] * 1.0000001; __syncwarp(); }
  long long t5 = clock64();
  out[lane] = x + y + z + w + u;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  const int it = 1000;
  for (int r = 0; r < 3; ++r) {
    lat<<<1, 32>>>(o, c, 0.5, it);
    long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
    printf("cycles/op: dfma %.1f  rcp %.1f  sqrt %.1f  sts+lds(conflict32) %.1f  sts+lds %.1f\n",
           h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it);
  }
  return 0;
}
