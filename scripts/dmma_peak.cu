// FP64 tensor-core (DMMA) and FP64 FMA peak probes for the roofline
// denominators (MEASURED_PEAKS.json carries no FP64 figure).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_peak.cu -o dmma_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8, iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    dmma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 8*8*4 FMA = 512 flop per warp instruction
    const double flops = double(blocks) * (threads / 32) * iters * 8 * 512.0;
    const double dmma_tf = flops / (ms * 1e-3) / 1e12;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f2 = double(blocks) * threads * iters * 8 * 2.0;
    const double dfma_tf = f2 / (ms * 1e-3) / 1e12;
    if (rep == 1)
      printf("{\"fp64_dmma_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f, \"sms\": %d}\n", dmma_tf, dfma_tf, sms);
  }
  return 0;
}
