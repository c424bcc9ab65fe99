// Micro-benchmark (measurement only): fp64 peak on B200 via DMMA.8x8x4 (mma.sync
// m8n8k4 f64) vs scalar DFMA, register-resident operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2] = {};
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double acc[16];
  for (int j = 0; j < 16; j++) acc[j] = j;
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 16; j++) acc[j] = fma(acc[j], b, a);
  }
  double s = 0;
  for (int j = 0; j < 16; j++) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocksPerSM : {4, 8}) {
    const int grid = sms * blocksPerSM, threads = 256, iters = 4096;
    dmma_loop<<<grid, threads>>>(out, 16);
    cudaEventRecord(a); dmma_loop<<<grid, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (grid * threads / 32.0);
    printf("DMMA  grid %d: %.2f TFLOP/s\n", grid, flops / (ms * 1e-3) / 1e12);
    dfma_loop<<<grid, threads>>>(out, 16);
    cudaEventRecord(a); dfma_loop<<<grid, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 16 * iters * (double)grid * threads;
    printf("DFMA  grid %d: %.2f TFLOP/s\n", grid, flops / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
