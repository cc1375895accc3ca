// Legacy warp-level MMA ceilings on this GPU (register-only, 8 independent accumulator chains per warp):
// FP64 m8n8k4 DMMA and TF32 m16n8k8.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32(float *out, int iters) {
  float acc[8][4] = {};
  unsigned a0 = 0x3f800000u + threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = 0x3f000000u, b1 = b0 ^ 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.0f) out[0] = s;
}
__global__ void f64(double *out, int iters) {
  double acc[8][2] = {};
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
  float *o;
  cudaMalloc(&o, 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 8; warps <= 32; warps *= 2) {
    float ms;
    tf32<<<sms, warps * 32>>>(o, 100);
    cudaEventRecord(e0);
    tf32<<<sms, warps * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("warps/SM %2d: TF32 m16n8k8 mma.sync %.1f TFLOP/s\n", warps,
           2.0 * 16 * 8 * 8 * 8.0 * iters * warps * sms / (ms * 1e-3) / 1e12);
    f64<<<sms, warps * 32>>>((double *)o, 100);
    cudaEventRecord(e0);
    f64<<<sms, warps * 32>>>((double *)o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("warps/SM %2d: FP64 m8n8k4 DMMA %.1f TFLOP/s\n", warps,
           2.0 * 8 * 8 * 4 * 8.0 * iters * warps * sms / (ms * 1e-3) / 1e12);
  }
  return 0;
}
