// Diagnostic: are CUDA's sincos() results bitwise equal to sin() and cos()
// for the proxy-circle angles t = 2 pi s / ns (s < ns <= 2048)?
#include <cstdio>
__global__ void k(int* bad, int* total) {
  const double kPi = 3.14159265358979323846;
  for (int ns = 64; ns <= 2048; ns *= 2)
    for (int s = threadIdx.x + blockIdx.x * blockDim.x; s < ns; s += blockDim.x * gridDim.x) {
      const double t = 2.0 * kPi * double(s) / double(ns);
      double a, b;
      sincos(t, &a, &b);
      atomicAdd(total, 1);
      if (a != sin(t) || b != cos(t)) atomicAdd(bad, 1);
    }
}
int main() {
  int *d, h[2];
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  k<<<8, 256>>>(d, d + 1);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("sincos differs from sin/cos on %d of %d angles\n", h[0], h[1]);
  return 0;
}
