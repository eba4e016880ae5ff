// Diagnostic: dependent-chain latencies (cycles) of the operations on the
// CPQR engines' per-step critical path, one warp (and one CTA of 512 for
// the barriers).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/lat_micro.cu -o scripts/lat_micro
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double x = x0 + threadIdx.x * 1e-12, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-300;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  // div chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  // LDS dependent (pointer chase through smem index)
  int k = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < n; ++i) k = int(sm[k]) & 7;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  // __syncthreads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  // __syncthreads_or
  int f = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f += __syncthreads_or(f + i == -5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = (t1 - t0) / n;
  // any_sync
  t0 = clock64();
  for (int i = 0; i < n; ++i) f += __any_sync(0xffffffffu, f == i);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / n;
  out[threadIdx.x] = x + k + f;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const char* names[] = {"dfma", "dadd", "dsqrt", "ddiv", "shfl.f64", "lds-chase", "syncthreads(512)", "syncthreads_or(512)", "any_sync"};
  for (int bs : {32, 512}) {
    lat<<<1, bs>>>(out, cyc, 0.5, 2000);
    cudaDeviceSynchronize();
    printf("block %d:", bs);
    for (int i = 0; i < 9; ++i) printf(" %s=%lld", names[i], cyc[i]);
    printf("\n");
  }
  return 0;
}
