// FP64 tensor-pipe ceiling on this GPU: every warp issues independent m8n8k4 DMMAs (8 accumulator
// chains) from registers, no memory traffic.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// dmma_peak.cu -o dmma_peak && ./dmma_peak
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double *o;
  cudaMalloc(&o, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    k<<<sms, warps * 32>>>(o, 100);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * sms;
    printf("warps/SM %2d: %.1f TFLOP/s FP64 (m8n8k4 DMMA)\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
