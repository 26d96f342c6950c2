// Microbenchmark: streaming kernel reading R vectors and writing one vector,
// with the written range cold in L2 vs hot in L2 (is a write miss expensive?).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* __restrict__ in, long n, int R, double* out, int fence) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    double s = 0;
    for (int r = 0; r < R; ++r) s += in[r * n + i];
    out[i] = s;
  }
  if (fence) __threadfence();
}
__global__ void touch(double* p, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) p[i] = 0.0;
}
int main() {
  long n = 2L << 20; int R = 6;
  double *in, *outs, *flush;
  cudaMalloc(&in, R * n * 8); cudaMalloc(&outs, 40 * n * 8); cudaMalloc(&flush, 64L << 20);
  cudaMemset(in, 0, R * n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int fence = 0; fence < 2; ++fence)
  for (int mode = 0; mode < 3; ++mode) {
    float tot = 0; int reps = 20;
    for (int rep = 0; rep < reps; ++rep) {
      double* out = outs + (long)(rep % 40) * n;
      if (mode == 1) touch<<<592, 256>>>(out, n);          // out hot in L2
      if (mode == 2) out = outs;                          // same buffer every rep (hot)
      cudaEventRecord(a);
      k<<<592, 256>>>(in, n, R, out, fence);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
    }
    printf("fence=%d mode=%s  %.2f us\n", fence, mode == 0 ? "cold-out" : mode == 1 ? "touched-out" : "same-out", 1e3 * tot / reps);
  }
}
